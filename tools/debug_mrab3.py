import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1403_1661_b200 as P
import swe_inputs as si
import oracle
from tests.common import make_oracle
w = si.c4_dambreak(N=3, base=5)
w.bathymetry = (lambda B0: (lambda x, y: B0(x, y) - 4.0))(w.bathymetry)
w.initial = lambda x, y: (0.1 * np.exp(-((x - 20.0) ** 2 + (y - 15.0) ** 2) / 8.0) - w.bathymetry(x, y), np.zeros_like(x), np.zeros_like(x))
dt = si.dt_for(w.mesh, w.N, w.g, 4.2, 13.0, 0.2)
o, d = make_oracle(w, tvb_M=1e6)
prm = dict(w.params); prm["tvb_M"] = 1e6
m = w.mesh
s = P.Solver(m.vx, m.vy, m.etov, d["B"], w.N, w.g, params=prm)
s.set_state(d["h"], d["hu"], d["hv"]); o.set_state(d["h"], d["hu"], d["hv"])
Q0 = o.get_state(); R0 = o.rhs(*Q0)
o.step(dt, 2); s.step(dt, 2)
lev = o.levels(); go, gs = o.get_state(), s.get_state()
bad = np.abs(gs[0] - go[0]).max(1) > 1e-13
Rg = [(a - b) / (2 * dt) for a, b in zip(gs, Q0)]
o1, _ = make_oracle(w, tvb_M=1e6); o1.set_state(d["h"], d["hu"], d["hv"]); o1.step(dt, 1); Qdt = o1.get_state()
def mix(Qa, Qb):  # level-1 from Qa, level-2 from Qb
    return [np.where((lev == 1)[:, None], a, b) for a, b in zip(Qa, Qb)]
cands = {"A: all t=0": R0, "B: lev1 at dt": o.rhs(*mix(Qdt, Q0)), "C: lev1 at 2dt": o.rhs(*mix(go, Q0)),
         "D: all at dt": o.rhs(*Qdt)}
for k, R in cands.items():
    print(k, [float(np.abs(Rg[f][bad] - R[f][bad]).max()) for f in range(3)])
print("level-2 elements, all: max|Rg-R0|", [float(np.abs(Rg[f][lev == 2] - R0[f][lev == 2]).max()) for f in range(3)])
o2, _ = make_oracle(w, tvb_M=1e6); o2.set_state(d["h"], d["hu"], d["hv"]); o2.step(dt, 1); E = o2.get_state(); o2.step(dt, 1); F = o2.get_state()
sel = lev == 2
for name, S in [("E: L1 1 step", E), ("F: L1 2 steps", F), ("oracle L2", go)]:
    print(name, [float(np.abs(gs[f][sel] - S[f][sel]).max()) for f in range(3)])
print("level counts gpu", s.info()["level_count"], "oracle", np.bincount(lev))
print("gpu levels equal", np.array_equal(s.levels(), lev))
