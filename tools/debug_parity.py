"""Step-by-step GPU vs oracle divergence tracer (debug tool, needs a GPU).

  python tools/debug_parity.py {thacker|dambreak|tvb} [nsteps]
Prints, per step, the parity norm and the limiter counters of both codes; at the
first step above 1e-12 it dumps the worst element of each field."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1403_1661_b200 as P  # noqa: E402
import swe_inputs as si  # noqa: E402
from tests.common import make_oracle, parity_rel  # noqa: E402


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "thacker"
    nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    over = {}
    L = 1
    if case == "thacker":
        w = si.c3_thacker(N=2, n=40)
        dt = si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)
    elif case == "dambreak":
        w = si.c4_dambreak(N=3, base=5)
        dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
        L = int(os.environ.get("L", "1"))
    elif case == "smoothmrab":
        w = si.c4_dambreak(N=3, base=5)
        w.bathymetry = (lambda B0: (lambda x, y: B0(x, y) - 4.0))(w.bathymetry)
        w.initial = lambda x, y: (0.1 * np.exp(-((x - 20.0) ** 2 + (y - 15.0) ** 2) / 8.0) - w.bathymetry(x, y),
                                  np.zeros_like(x), np.zeros_like(x))
        dt = si.dt_for(w.mesh, w.N, w.g, 4.2, 13.0, 0.2)
        L = int(os.environ.get("L", "3"))
        over = {"tvb_M": 1e6}
    else:
        w = si.c1_lake(N=2, hump=True, n=16)
        dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2)
        over = {"tvb_M": 0.1}
    for k, v in os.environ.items():
        if k.startswith("P_"):
            over[k[2:]] = float(v) if "." in v or "e" in v else int(v)
    o, d = make_oracle(w, **over)
    prm = dict(w.params)
    prm.update(over)
    m = w.mesh
    s = P.Solver(m.vx, m.vy, m.etov, d["B"], w.N, w.g, vper=m.vper, params=prm)
    o.set_state(d["h"], d["hu"], d["hv"])
    s.set_state(d["h"], d["hu"], d["hv"])
    rel = parity_rel(s.get_state(), o.get_state(), w.g)
    print("init", rel, o.info()["n_pp"], s.info()["n_pp"], o.info()["n_dry"], s.info()["n_dry"])
    for k in range(nsteps):
        assert o.step(dt, L) == 0
        s.step(dt, L)
        go, gs = o.get_state(), s.get_state()
        rel = parity_rel(gs, go, w.g)
        io, ig = o.info(), s.info()
        print(k, ["%.1e" % r for r in rel], "pp", io["n_pp"], ig["n_pp"], "dry", io["n_dry"], ig["n_dry"], "tvb",
              io["n_tvb"], ig["n_tvb"], "inj %.3e %.3e" % (io["injected_mass"], ig["injected_mass"]))
        if case == "smoothmrab" and k == 0:
            lev = o.levels()
            e2e, e2f = o.connectivity()
            err = np.abs(gs[0] - go[0]).max(1)
            worst = np.argsort(-err)[:12]
            for e in worst:
                nbl = [int(lev[n]) if n != e else -1 for n in e2e[e]]
                print("   worst elem", e, "lev", lev[e], "err %.2e" % err[e], "nbr levels", nbl,
                      "x %.2f y %.2f" % (d["x"][e].mean(), d["y"][e].mean()))
            print("   n_err>1e-13:", int((err > 1e-13).sum()), "of", len(err), "levels of those",
                  np.bincount(lev[err > 1e-13]))
        if case == "smoothmrab":
            lev = o.levels()
            for l in sorted(set(lev.tolist())):
                sel = lev == l
                print("   level", l, "max|dh|", np.abs(gs[0][sel] - go[0][sel]).max(), "max|dhu|",
                      np.abs(gs[1][sel] - go[1][sel]).max())
        if max(rel) > 1e-12 and case != "smoothmrab":
            for f in range(3):
                diff = np.abs(gs[f] - go[f])
                e = int(np.argmax(diff.max(1)))
                print(" field", f, "elem", e, "x", d["x"][e].mean(), "y", d["y"][e].mean())
                print("   orc", go[0][e], go[1][e])
                print("   gpu", gs[0][e], gs[1][e])
            break


if __name__ == "__main__":
    main()
