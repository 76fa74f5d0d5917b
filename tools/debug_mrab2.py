import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1403_1661_b200 as P
import swe_inputs as si
from tests.common import make_oracle
w = si.c4_dambreak(N=3, base=5)
w.bathymetry = (lambda B0: (lambda x, y: B0(x, y) - 4.0))(w.bathymetry)
w.initial = lambda x, y: (0.1 * np.exp(-((x - 20.0) ** 2 + (y - 15.0) ** 2) / 8.0) - w.bathymetry(x, y), np.zeros_like(x), np.zeros_like(x))
dt = si.dt_for(w.mesh, w.N, w.g, 4.2, 13.0, 0.2)
o, d = make_oracle(w, tvb_M=1e6)
prm = dict(w.params); prm["tvb_M"] = 1e6
m = w.mesh
for variant in ["getstate_first", "no_getstate"]:
    s = P.Solver(m.vx, m.vy, m.etov, d["B"], w.N, w.g, params=prm)
    s.set_state(d["h"], d["hu"], d["hv"])
    if variant == "getstate_first":
        s.get_state()
    o.set_state(d["h"], d["hu"], d["hv"])
    Q0 = o.get_state(); R0 = o.rhs(*Q0)
    o.step(dt, 2); s.step(dt, 2)
    lev = o.levels()
    go, gs = o.get_state(), s.get_state()
    err = np.abs(gs[0] - go[0]).max(1)
    print(variant, "max err", err.max(), "levels of bad", np.bincount(lev[err > 1e-13], minlength=3))
    e = int(np.argmax(err))
    for f in range(2):
        print(" field", f, "gpu-Q0", (gs[f][e] - Q0[f][e])[:4], "orc-Q0", (go[f][e] - Q0[f][e])[:4], "2dtR0", (2 * dt * R0[f][e])[:4], "dtR0", (dt*R0[f][e])[:4])
