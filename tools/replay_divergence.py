"""Locate the first macro step where the GPU and the decision-replaying oracle part by more than 1e-12
(A23 norm) and print the elements involved with their logged decisions.
    python tools/replay_divergence.py lake|thacker [M] [nsteps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1403_1661_b200 as P  # noqa: E402
import swe_inputs as si  # noqa: E402
from tests.common import make_oracle, parity_rel  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "lake"
M = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
nsteps = int(sys.argv[3]) if len(sys.argv) > 3 else 100
if case == "lake":
    w = si.c8_oscillating_lake(2, 16)
    dt = si.dt_for(w.mesh, w.N, w.g, 0.2, 0.0, 0.2, u_max=0.5)
else:
    w = si.c3_thacker(N=2, n=40)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)
o, d = make_oracle(w, tvb_M=M)
m = w.mesh
prm = dict(w.params, tvb_M=M, record_decisions=1)
s = P.Solver(m.vx, m.vy, m.etov, d["B"], w.N, w.g, vper=m.vper, params=prm, vbc=m.vbc)
s.set_state(d["h"], d["hu"], d["hv"])
states = []
for k in range(nsteps):
    s.step(dt, 1)
    states.append(s.get_state())
log = s.decisions()
o.set_replay(log)
o.set_state(d["h"], d["hu"], d["hv"])
print("params", w.params, "M", M, "records", log.shape)
for k in range(nsteps):
    assert o.step(dt, 1) == 0
    go = o.get_state()
    rel = parity_rel(states[k], go, w.g)
    if max(rel) > 1e-12:
        hs = np.abs(go[0]).max()
        err = np.max([np.abs(states[k][f] - go[f]).max(axis=1) for f in range(3)], axis=0)
        bad = np.argsort(-err)[:8]
        print(f"step {k}: rel {rel}, info {o.info()}")
        for e in bad:
            print(f"  elem {e} err {err[e]:.3e} gpu h {states[k][0][e]} orc h {go[0][e]} log {log[k + 1][e]}"
                  f" prev {log[k][e]} means_h {states[k][0][e].mean():.6e}")
        break
else:
    print("no divergence", o.info())
