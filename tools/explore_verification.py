import time, math, numpy as np, oracle, swe_inputs as si
from tests.common import make_oracle
oracle.set_threads(0)

def l2err(o, w, t, field=0, region=None):
    x, y = o.nodes()
    ex = w.exact(x, y, t)
    st = o.get_state()
    Mw = oracle.refel(w.N)["wmean"]  # int l_i on the reference triangle (weights of the nodal quadrature proxy)
    # element areas
    v = w.mesh.etov; X=w.mesh.vx[v]; Y=w.mesh.vy[v]
    A = 0.5*np.abs((X[:,1]-X[:,0])*(Y[:,2]-Y[:,0])-(X[:,2]-X[:,0])*(Y[:,1]-Y[:,0]))
    err = (st[field]-ex[field])**2
    wts = (A/2.0)[:,None]*Mw[None,:]
    if region is not None:
        sel = region(x, y)
        return math.sqrt((wts*err*sel).sum())
    return math.sqrt((wts*err).sum())

def run(w, t_end, t0=0.0, dtf=0.2, umax=0.0, hmax=1.0):
    o, d = make_oracle(w)
    o.set_state(d["h"], d["hu"], d["hv"])
    dt = si.dt_for(w.mesh, w.N, w.g, hmax, 0.0, dtf, u_max=umax)
    n = int(math.ceil((t_end - t0) / dt)); dt = (t_end - t0) / n
    t1=time.time()
    for _ in range(n): assert o.step(dt, 1) == 0
    return o, n, time.time()-t1

for N in (1, 2, 3):
    errs=[]
    for (nr, nth) in [(2, 12), (4, 24), (8, 48)]:
        w = si.c6_couette(N, nr, nth)
        o, n, el = run(w, 1.0, umax=0.1)
        errs.append(l2err(o, w, 1.0, 0)); 
        print("couette N", N, nr, nth, "K", w.mesh.K, "steps", n, "err h", errs[-1], "t", round(el,2), flush=True)
    print("  EOC", [math.log(errs[i]/errs[i+1], 2) for i in range(len(errs)-1)])
for N in (1, 2):
    errs=[]; loc=[]
    for n_ in (2, 4, 8):
        w = si.c7_rarefaction(N, n_)
        o, n, el = run(w, 3.0, t0=2.0, umax=2.0)
        errs.append(l2err(o, w, 3.0, 0)); loc.append(l2err(o, w, 3.0, 0, region=lambda x,y: (x>18)&(x<24)))
        print("rare N", N, n_, "K", w.mesh.K, "steps", n, "err", errs[-1], "loc", loc[-1], "t", round(el,2), "min h", o.get_state()[0].min(), flush=True)
    print("  EOC glob", [math.log(errs[i]/errs[i+1], 2) for i in range(len(errs)-1)], "loc", [math.log(loc[i]/loc[i+1], 2) for i in range(len(loc)-1)])
for N in (1, 2):
    errs=[]
    for n_ in (8, 16, 32):
        w = si.c8_oscillating_lake(N, n_)
        o, n, el = run(w, 0.1, umax=0.5, hmax=0.2)
        errs.append(l2err(o, w, 0.1, 0, region=lambda x,y: x*x+y*y < 0.4))
        i = o.info()
        print("lake N", N, n_, "K", w.mesh.K, "steps", n, "err", errs[-1], "t", round(el,2), "mass", i["mass"], "inj", i["injected_mass"], "minh", i["min_h"], flush=True)
    print("  EOC", [math.log(errs[i]/errs[i+1], 2) for i in range(len(errs)-1)])
