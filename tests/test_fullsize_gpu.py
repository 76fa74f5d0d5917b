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
