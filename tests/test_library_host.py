"""-m 'not gpu' tests of the product library: it loads, exports every symbol
include/swe.h declares, and its host builders agree with the independent
oracle (operators <= 1e-13, connectivity / Hk / levels / TVB pairs bit-exact)."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_1403_1661_b200 as P
import swe_inputs as si
from tests.common import make_oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    P.build()
    return P.lib()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "swe.h")).read()
    declared = set(re.findall(r"\b(swe_[a-z_]+)\s*\(", hdr))
    assert len(declared) >= 17
    L = P.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(P.EXPORTED)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_operators_match_oracle(N):
    ro = oracle.refel(N)
    for k in ["r", "s", "Dr", "Ds", "Mref", "Ic", "Ig", "P", "Pr", "Ps", "Lg", "wmean", "rc", "sc", "wc", "tg", "wg"]:
        a, b = P.host_refel(N, k), ro[k]
        assert a.shape == b.shape, k
        assert np.abs(a - b).max() <= 1e-13 * max(1.0, np.abs(b).max()), k


def test_p1_vertex_operator():
    """Pv q = vertex values of the L2 projection onto P1: exact on linear data, kills P1-orthogonal modes."""
    N = 3
    r, s = P.host_refel(N, "r"), P.host_refel(N, "s")
    Pv = P.host_refel(N, "Pv")
    lin = 0.7 - 0.2 * r + 0.45 * s
    assert np.allclose(Pv @ lin, [0.7 + 0.2 - 0.45, 0.7 - 0.2 - 0.45, 0.7 + 0.2 + 0.45], atol=1e-14)
    # mean preserved: average of vertex values == cell mean for any polynomial
    rng = np.random.default_rng(0)
    q = rng.standard_normal(len(r))
    w = P.host_refel(N, "wmean")
    assert abs((Pv @ q).mean() - 0.5 * w @ q) < 1e-14


def _meshes():
    yield "C1", si.c1_lake(N=2).mesh
    yield "C2", si.c2_vortex(2, 8).mesh
    yield "C4c", si.c4_dambreak(N=3, base=5).mesh
    m = si.shuffle(si.structured(7, 5, 0.0, 3.0, -1.0, 1.0), seed=11, flip_fraction=0.4)
    yield "flip", m


@pytest.mark.parametrize("name,mesh", list(_meshes()))
def test_connectivity_hk_tvb_bit_exact(name, mesh):
    e, f, nflip = P.host_connectivity(mesh.vx, mesh.vy, mesh.etov, mesh.vper)
    o = oracle.Oracle(mesh.vx, mesh.vy, mesh.etov, np.zeros((mesh.K, 3)), 1, 9.81, vper=mesh.vper)
    eo, fo = o.connectivity()
    assert np.array_equal(e, eo) and np.array_equal(f, fo)
    J, Hk, nf = o.geometry()
    assert nflip == nf
    assert np.array_equal(P.host_hk(mesh.vx, mesh.vy, mesh.etov, mesh.vper), Hk)  # bit-exact (A19)
    pairs, al = P.host_tvb_geometry(mesh.vx, mesh.vy, mesh.etov, mesh.vper)
    po, alo = o.tvb_geometry()
    assert np.array_equal(pairs, po)
    assert np.abs(al - alo).max() < 1e-13


def test_nodes_match_oracle():
    w = si.c1_lake(N=3)
    m = w.mesh
    x, y = P.nodes(m.vx, m.vy, m.etov, 3)
    o, d = make_oracle(w)
    assert np.abs(x - d["x"]).max() < 1e-14 and np.abs(y - d["y"]).max() < 1e-14


@pytest.mark.parametrize("case", ["C4c", "C1b", "C3", "random"])
def test_levels_bit_exact(case):
    if case == "C4c":
        w = si.c4_dambreak(N=3, base=3)
        L = 3
    elif case == "C1b":
        w = si.c1_lake(N=2, hump=True)
        L = 4
    elif case == "C3":
        w = si.c3_thacker(N=2, n=30)
        L = 5
    else:
        w = si.c1_lake(N=2, n=12)
        L = 6
    o, d = make_oracle(w)
    h, hu, hv = d["h"], d["hu"], d["hv"]
    if case == "random":
        rng = np.random.default_rng(4)
        h = np.abs(h) * rng.uniform(0.01, 3.0, (h.shape[0], 1))
        hu = rng.standard_normal(h.shape)
        hv = rng.standard_normal(h.shape)
    o.set_state(h, hu, hv)
    lev_o = o.bin_levels(L)
    m = w.mesh
    lev_p = P.host_levels(m.vx, m.vy, m.etov, w.N, w.g, h, hu, hv, L, params=w.params, vper=m.vper)
    assert np.array_equal(lev_o, lev_p)
    if case == "C4c":
        assert len(np.unique(lev_p)) == 3  # three geometric levels


def test_create_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    w = si.c1_lake(N=2, n=2)
    m = w.mesh
    with pytest.raises(P.SweError) as ei:
        P.Solver(m.vx, m.vy, m.etov, np.zeros((m.K, 6)), 2, 9.81, use_torch=False)
    assert ei.value.code == -7  # SWE_ERR_CUDA


def test_argument_errors():
    w = si.c1_lake(N=2, n=2)
    m = w.mesh
    with pytest.raises(P.SweError) as ei:
        P.nodes(m.vx, m.vy, np.array([[0, 1, 99]]), 2)
    assert ei.value.code == -2
    with pytest.raises(P.SweError) as ei:
        P.nodes(m.vx, m.vy, m.etov, 0)
    assert ei.value.code == -3
