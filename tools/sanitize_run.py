"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
C1 hump (N = 2, PP + TVB), C4 dam break (N = 3, 3 MRAB levels, graphs), N = 4 and N = 5 (DMMA K1), FP32, a Dirichlet
vortex and an in-process 2-rank partition.  Exits non-zero on any solver error.
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1403_1661_b200 as P  # noqa: E402
import swe_inputs as si  # noqa: E402


def run(w, steps, dt, L=1, prm=None, bnd=False):
    m = w.mesh
    x, y = P.nodes(m.vx, m.vy, m.etov, w.N)
    B, h, hu, hv = w.fields(x, y)
    s = P.Solver(m.vx, m.vy, m.etov, B, w.N, w.g, vper=m.vper, vbc=m.vbc, params=dict(w.params, **(prm or {})))
    if bnd:
        s.set_boundary_state(*w.exact(x, y, 0.0))
    s.set_state(h, hu, hv)
    for _ in range(steps):
        s.step(dt, L)
    st = s.get_state()
    s.info()
    s.close()
    return st


w = si.c1_lake(N=2, n=8, hump=True)
run(w, 4, si.dt_for(w.mesh, 2, w.g, 1.0, 0.0, 0.2), prm=dict(tvb_M=0.1))
w = si.c4_dambreak(N=3, base=10)
run(w, 10, si.dt_for(w.mesh, 3, w.g, 1.875, 13.0, 0.2), L=3)  # 10 macro steps: past the ramp, graphs replayed
run(w, 3, si.dt_for(w.mesh, 3, w.g, 1.875, 13.0, 0.2), L=3, prm=dict(precision=32))
w4 = si.c4_dambreak(N=4, base=10)
run(w4, 3, si.dt_for(w4.mesh, 4, w4.g, 1.875, 13.0, 0.2), L=3)
w5 = si.c4_dambreak(N=5, base=10)
run(w5, 3, si.dt_for(w5.mesh, 5, w5.g, 1.875, 13.0, 0.2), L=3)
wd = si.c2_vortex_dirichlet(2, 8)
run(wd, 4, si.dt_for(wd.mesh, 2, wd.g, 1.0, 0.0, 0.1, u_max=2.0), bnd=True)
# in-process 2-rank partition (halo pack / unpack kernels)
m = w.mesh
x, y = P.nodes(m.vx, m.vy, m.etov, 3)
B, h, hu, hv = w.fields(x, y)
v = m.etov
owner = (m.vx[v].mean(1) > np.median(m.vx[v].mean(1))).astype(np.int32)
parts = [P.Solver(m.vx, m.vy, m.etov, B, 3, w.g, params=w.params, rank=r, nranks=2, owner=owner) for r in range(2)]
P.link_group(parts)
for s in parts:
    s.set_state(h, hu, hv)
for _ in range(3):
    P.step_group(parts, si.dt_for(m, 3, w.g, 1.875, 13.0, 0.2), 3)
print("sanitize runs ok")
