"""Full-size checks in bench.py's launch configuration (C5: 7,056,640 triangles, N = 3,
4 MRAB levels, PP + TVB, the bench dt): element-by-element parity with the oracle
after two macro steps, bit-exact levels, positivity, and a lake at rest."""
import numpy as np
import pytest

import oracle
import paper_1403_1661_b200 as P
import swe_inputs as si
from tests.common import parity_rel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def c5():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = si.c5_tsunami(P=1)
    m = w.mesh
    x, y = P.nodes(m.vx, m.vy, m.etov, w.N)
    B, h, hu, hv = w.fields(x, y)
    dt = si.dt_for(m, w.N, w.g, 4001.0, w.params["a_floor"], w.dt_factor)
    return w, x, y, B, h, hu, hv, dt


def test_c5_fullsize_parity_and_levels(c5):
    w, x, y, B, h, hu, hv, dt = c5
    m = w.mesh
    oracle.set_threads(0)
    o = oracle.Oracle(m.vx, m.vy, m.etov, B, w.N, w.g, **w.params)
    s = P.Solver(m.vx, m.vy, m.etov, B, w.N, w.g, params=w.params)
    o.set_state(h, hu, hv)
    s.set_state(h, hu, hv)
    for _ in range(2):
        assert o.step(dt, w.nlevels) == 0
        s.step(dt, w.nlevels)
    lev = s.levels()
    assert np.array_equal(lev, o.levels())
    assert np.array_equal(lev, P.host_levels(m.vx, m.vy, m.etov, w.N, w.g, h, hu, hv, w.nlevels, params=w.params))
    assert np.bincount(lev, minlength=5)[1:].tolist() == [844800, 1359360, 2233600, 2618880]
    gs, go = s.get_state(), o.get_state()
    rel = parity_rel(gs, go, w.g)
    assert max(rel) <= 1e-12, rel
    assert gs[0].min() >= 0.0
    io, ig = o.info(), s.info()
    assert io["n_pp"] == ig["n_pp"] and io["n_dry"] == ig["n_dry"] and io["n_tvb"] == ig["n_tvb"]


def test_c5_fullsize_lake_at_rest(c5):
    w, x, y, B, h, hu, hv, dt = c5
    m = w.mesh
    Bw = B - 100.0  # fully wet basin, eta = 0
    s = P.Solver(m.vx, m.vy, m.etov, Bw, w.N, w.g, params=w.params)
    s.set_state(-Bw, np.zeros_like(Bw), np.zeros_like(Bw))
    for _ in range(2):
        s.step(dt, w.nlevels)
    hh, mu, mv = s.get_state()
    assert np.abs(hh + Bw).max() <= 1e-12 * 4100.0
    assert max(np.abs(mu).max(), np.abs(mv).max()) <= 1e-10 * 4100.0 * np.sqrt(9.81 * 4100.0)
    assert s.info()["n_tvb"] == 0


def _replayed_parity(w, nsteps, dt, nlevels, **over):
    """GPU run with the decision log, the oracle replaying it, element-wise parity."""
    m = w.mesh
    oracle.set_threads(0)
    Np = (w.N + 1) * (w.N + 2) // 2
    probe = oracle.Oracle(m.vx, m.vy, m.etov, np.zeros((m.K, Np)), w.N, w.g, vper=m.vper)
    x, y = probe.nodes()
    del probe
    B, h, hu, hv = w.fields(x, y)
    prm = dict(w.params)
    prm.update(over)
    s = P.Solver(m.vx, m.vy, m.etov, B, w.N, w.g, vper=m.vper, params=dict(prm, record_decisions=1))
    s.set_state(h, hu, hv)
    for _ in range(nsteps):
        s.step(dt, nlevels)
    o = oracle.Oracle(m.vx, m.vy, m.etov, B, w.N, w.g, vper=m.vper, **prm)
    o.set_replay(s.decisions())
    o.set_state(h, hu, hv)
    for _ in range(nsteps):
        assert o.step(dt, nlevels) == 0
    io, ig = o.info(), s.info()
    assert io["n_mismatch"] == 0, io
    assert np.array_equal(o.levels(), s.levels())
    rel = parity_rel(s.get_state(), o.get_state(), w.g)
    assert max(rel) <= 1e-12, rel
    for k in ("n_pp", "n_dry", "n_tvb", "n_posfix"):
        assert io[k] == ig[k], (k, io[k], ig[k])
    print(w.name, "levels", np.bincount(s.levels())[1:].tolist(), "rel", rel, "adopted", io["n_adopted"],
          {k: io[k] for k in ("n_pp", "n_dry", "n_tvb", "n_posfix")})
    io["levels_used"] = len(np.unique(s.levels()))
    return io


def test_c4_fullsize_100_macro_steps():
    """North_star: parity after 100 steps.  C4 at full size (187,560 triangles, N = 3, 3 MRAB levels,
    wet/dry dam break, PP + TVB), 100 macro steps (400 finest substeps)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = si.c4_dambreak(N=3, base=1)
    assert w.mesh.K == 187560
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    io = _replayed_parity(w, 100, dt, 3)
    assert io["n_pp"] > 0 and io["n_dry"] > 0 and io["levels_used"] == 3


def test_c5_base320_100_macro_steps():
    """C5 recipe at base_n = 320 (446,080 triangles, N = 3, 4 MRAB levels, PP + TVB), 100 macro steps."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = si.c5_tsunami(P=1, base_n=320)
    dt = si.dt_for(w.mesh, w.N, w.g, 4001.0, w.params["a_floor"], w.dt_factor)
    io = _replayed_parity(w, 100, dt, 4)
    assert io["n_pp"] > 0 and io["levels_used"] == 4


def test_periodic_vortex_mrab_100_macro_steps():
    """MRAB on a periodic mesh: the C2 vortex (N = 3, no limiters) on a graded periodic 2 x 16 x 16 mesh whose
    element sizes span 4x, so 3 levels are binned; 100 macro steps; the dense output crosses periodic faces."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = si.c2_vortex_graded(3, 16)
    dt = si.dt_for(w.mesh, 3, w.g, 1.0, 0.0, 0.1, u_max=2.0)
    io = _replayed_parity(w, 100, dt, 3)
    assert io["levels_used"] == 3


def test_c5_fullsize_1000_macro_steps_graph_replay(c5):
    """The bench's launch configuration (CUDA-graph replay, K2 list pass, one macro step = 15 K1 + 15 K2) run for 1000
    macro steps (8,000 finest substeps, ~1 minute of simulated time): every step finite (swe_step reports non-finite
    states), h >= 0 at every node, and mass conserved up to the dry branch's counted injection (Alg. 3, reading A13)."""
    w, x, y, B, h, hu, hv, dt = c5
    m = w.mesh
    s = P.Solver(m.vx, m.vy, m.etov, B, w.N, w.g, params=w.params)
    s.set_state(h, hu, hv)
    s.step(dt, w.nlevels)
    i0 = s.info()
    for _ in range(999):
        s.step(dt, w.nlevels)
    i1 = s.info()
    assert i1["min_h"] >= 0.0
    drift = i1["mass"] - i0["mass"] - (i1["injected_mass"] - i0["injected_mass"])
    assert abs(drift) <= 1e-11 * i0["mass"], (drift, i0["mass"])
    hh, _, _ = s.get_state()
    assert np.isfinite(hh).all() and hh.min() >= 0.0
    s.close()


@pytest.mark.parametrize("N,base", [(4, 1), (5, 2)])
def test_c4_tensor_path_100_macro_steps(N, base):
    """North_star's "after 100 steps" bar for the tensor-path K1 (k_rhs_update_mma2): the C4 dam break (3 MRAB
    levels, wet/dry, PP + TVB) at N = 4 on the full 187,560-triangle mesh and at N = 5 on the base-2 mesh,
    100 macro steps, element-wise parity with the oracle (decision replay) and equal counters."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = si.c4_dambreak(N=N, base=base)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    io = _replayed_parity(w, 100, dt, 3)
    assert io["n_pp"] > 0 and io["n_dry"] > 0 and io["levels_used"] == 3
