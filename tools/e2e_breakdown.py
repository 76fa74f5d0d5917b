"""Wall-clock breakdown of the e2e path on C5 (set_state, first step with binning, steady steps,
swe_get_info, final swe_get_state into pinned memory)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_1661_b200 as P  # noqa: E402
import swe_inputs as si  # noqa: E402

w = si.c5_tsunami(P=1)
m = w.mesh
x, y = P.nodes(m.vx, m.vy, m.etov, 3)
B, h, hu, hv = w.fields(x, y)
del x, y
s = P.Solver(m.vx, m.vy, m.etov, B, 3, w.g, params=w.params)
dt = si.dt_for(m, 3, w.g, 4001.0, w.params["a_floor"], w.dt_factor)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
hh, hhu, hhv = pin(h), pin(hu), pin(hv)
oh, ohu, ohv = pin(np.zeros_like(h)), pin(np.zeros_like(h)), pin(np.zeros_like(h))
s.set_state(hh, hhu, hhv)
for _ in range(4):
    s.step(dt, 4)
torch.cuda.synchronize()


def t(f, n=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("set_state (H2D + speeds)   %.1f ms" % t(lambda: s.set_state(hh, hhu, hhv)))
print("first step (bin+limit+step) %.1f ms" % t(lambda: s.step(dt, 4)))
print("steady step                %.1f ms" % t(lambda: s.step(dt, 4), 5))
print("swe_get_info               %.1f ms" % t(lambda: s.info(), 5))
print("get_state_into (pinned)    %.1f ms" % t(lambda: s.get_state_into(oh, ohu, ohv)))
print("get_state_into again       %.1f ms" % t(lambda: s.get_state_into(oh, ohu, ohv)))
print("set_state again            %.1f ms" % t(lambda: s.set_state(hh, hhu, hhv)))
print("first step again           %.1f ms" % t(lambda: s.step(dt, 4)))
# raw PCIe reference: one 565 MB field each way through torch
a = torch.from_numpy(hh)
d = torch.empty(a.shape, dtype=a.dtype, device="cuda")
print("torch H2D one field        %.1f ms (%.1f GB/s)" % (t(lambda: d.copy_(a, non_blocking=True)), 0))
o = torch.from_numpy(oh)
print("torch D2H one field        %.1f ms" % t(lambda: o.copy_(d, non_blocking=True)))
