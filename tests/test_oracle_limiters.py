"""Pins for the oracle's limiters: Alg. 3, TVB + Eq. modified_TVB
(P:224-253).  Hand values from SPEC.md (S:n lines, derived from the paper's
formulas by hand), closed forms and invariants."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import swe_inputs as si
from tests.common import make_oracle, tri_monomial_integral

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "limiter_examples.json")))

REF_TRI = (np.array([-1.0, 1.0, -1.0]), np.array([-1.0, -1.0, 1.0]), np.array([[0, 1, 2]], dtype=np.int32))


def one_element(N, h0=1e-14, **kw):
    Np = (N + 1) * (N + 2) // 2
    vx, vy, etov = REF_TRI
    return oracle.Oracle(vx, vy, etov, np.zeros((1, Np)), N, 9.81, h0=h0, **kw)


def test_pp_theta_example():
    ex = GOLDEN["pp_theta"]
    o = one_element(1, h0=1e-14, use_tvb=0)
    hv = np.array(ex["vertex_h"])[None, :]
    h, hu, hv2, dry = o.limit(hv, np.zeros((1, 3)), np.zeros((1, 3)))
    assert dry[0] == 0
    assert np.allclose(h[0], ex["expected_vertex_h"], atol=1e-13)
    assert abs(h[0].mean() - ex["mean"]) < 1e-15


def test_pp_dry_branch_and_injection():
    h0 = 1e-3
    o = one_element(2, h0=h0, use_tvb=0)
    h = np.full((1, 6), 0.5 * h0)  # mean h0/2
    h2, hu2, hv2, dry = o.limit(h, np.full((1, 6), 0.3), np.full((1, 6), -0.1))
    assert dry[0] == 1
    assert np.all(h2 == h0) and np.all(hu2 == 0) and np.all(hv2 == 0)
    assert abs(o.info()["injected_mass"] - 0.5 * h0 * 2.0) < 1e-18  # (h0 - hbar) * area, area = 2 J = 2


def test_pp_untouched_when_positive():
    o = one_element(3, h0=1e-6, use_tvb=0)
    rng = np.random.default_rng(5)
    h = rng.uniform(0.1, 1.0, (1, 10))
    hu, hv = rng.normal(size=(1, 10)), rng.normal(size=(1, 10))
    h2, hu2, hv2, dry = o.limit(h, hu, hv)
    assert np.array_equal(h2, h) and np.array_equal(hu2, hu) and np.array_equal(hv2, hv)


def test_projection_p1_drops_orthogonal_mode():
    """Pi_1 is the L2 projection onto P1 (keeps means): linear + (mode orthogonal to P1) -> linear."""
    N = 2
    re = oracle.refel(N)
    r, s = re["r"], re["s"]
    # phi = r^2 - (L2 projection of r^2 onto span{1, r, s}), exact rational Gram system
    basis = [(0, 0), (1, 0), (0, 1)]
    G = np.array([[float(tri_monomial_integral(a[0] + b[0], a[1] + b[1])) for b in basis] for a in basis])
    rhs = np.array([float(tri_monomial_integral(2 + a[0], a[1])) for a in basis])
    c = np.linalg.solve(G, rhs)
    phi = r ** 2 - (c[0] + c[1] * r + c[2] * s)
    lin = 1.0 + 0.2 * r - 0.3 * s
    h = (lin - 3.0 * phi)[None, :]
    assert h.min() < 0  # triggers Alg. 3
    o = one_element(N, h0=1e-12, use_tvb=0)
    h2, _, _, dry = o.limit(h, np.zeros_like(h), np.zeros_like(h))
    # linear part has vertex min 1 - 0.5 = 0.5 > h0 -> theta = 1: output is exactly the linear part
    assert np.abs(h2[0] - lin).max() < 1e-13


def test_pp_random_invariants():
    """Means preserved, vertex heights >= h0, idempotence."""
    w = si.c1_lake(N=3, n=4, shuffle_seed=None)
    o, d = make_oracle(w, h0=1e-3, use_tvb=0)
    rng = np.random.default_rng(7)
    K, Np = d["h"].shape
    h = rng.uniform(-0.2, 1.0, (K, Np)) + 0.3
    hu, hv = rng.normal(size=(K, Np)), rng.normal(size=(K, Np))
    h2, hu2, hv2, dry = o.limit(h, hu, hv)
    wm = oracle.refel(3)["wmean"]
    for a, b in ((h, h2), (hu, hu2), (hv, hv2)):
        ma, mb = 0.5 * a @ wm, 0.5 * b @ wm
        wet = dry == 0
        assert np.abs(ma - mb)[wet].max() < 1e-14 * max(1.0, np.abs(ma).max())
    assert h2.min() >= 1e-3 * (1 - 1e-12)
    h3, hu3, hv3, dry3 = o.limit(h2, hu2, hv2)
    assert np.abs(h3 - h2).max() < 1e-14 and np.array_equal(dry3, dry)


def test_posfix_example():
    ex = GOLDEN["modified_tvb"]  # S:311, Eq. modified_TVB
    out = oracle.posfix(ex["Dhat"], ex["hbar"], ex["h0"])
    assert np.allclose(out, ex["expected"], atol=1e-15)
    # min vertex value hbar + (-D_i + D_j + D_k) equals h0 after the fix
    verts = [ex["hbar"] - out[i] + out[(i + 1) % 3] + out[(i + 2) % 3] for i in range(3)]
    assert abs(min(verts) - ex["h0"]) < 1e-15
    assert np.allclose(oracle.posfix([0.01, -0.02, 0.01], 1.0, 0.0), [0.01, -0.02, 0.01])  # theta = 1 branch
    assert np.allclose(oracle.posfix([0, 0, 0], 0.5, 0.1), [0, 0, 0])


def test_rebalance_and_minmod():
    D = oracle.rebalance([0.3, -0.1, -0.1])  # pos 0.3, neg 0.2 -> theta+ = 2/3
    assert np.allclose(D, [0.2, -0.1, -0.1]) and abs(D.sum()) < 1e-16
    assert np.allclose(oracle.rebalance([0.1, 0.2, 0.0]), [0, 0, 0])  # one-signed -> 0
    assert oracle.mbar(0.5, 2.0, 0.0) == (0.5, True)
    assert oracle.mbar(2.0, 0.5, 0.0) == (0.5, False)
    assert oracle.mbar(-2.0, -0.5, 0.0) == (-0.5, False)
    assert oracle.mbar(1.0, -1.0, 0.0) == (0.0, False)
    assert oracle.mbar(1.0, -1.0, 1.5) == (1.0, True)  # |a| <= M Hk^2: TVB keeps a


def test_characteristic_matrices():
    rng = np.random.default_rng(9)
    g = 9.81
    for _ in range(10):
        h, u, v = rng.uniform(0.5, 3), rng.normal(), rng.normal()
        th = rng.uniform(0, 2 * math.pi)
        nx, ny = math.cos(th), math.sin(th)
        L, R = oracle.char_matrices(g, h, u, v, nx, ny)
        assert np.abs(L @ R - np.eye(3)).max() < 1e-14
        c2 = g * h
        dF = np.array([[0, 1, 0], [c2 - u * u, 2 * u, 0], [-u * v, v, u]])
        dG = np.array([[0, 0, 1], [-u * v, v, u], [c2 - v * v, 0, 2 * v]])
        An = nx * dF + ny * dG
        un, c = u * nx + v * ny, math.sqrt(c2)
        assert np.abs(L @ An @ R - np.diag([un - c, un, un + c])).max() < 1e-12


def _wall_mesh_state(fun, N=2, n=6):
    w = si.c1_lake(N=N, n=n, shuffle_seed=None)
    o, d = make_oracle(w, h0=1e-6, tvb_M=0.0, use_pp=1, use_tvb=1)
    h, hu, hv = fun(d["x"], d["y"])
    return o, d, h, hu, hv


def test_tvb_constant_and_linear_states_untouched():
    # constant state: bit-identical
    o, d, h, hu, hv = _wall_mesh_state(lambda x, y: (np.full_like(x, 2.0), np.full_like(x, 0.3), np.full_like(x, 0.1)))
    h2, hu2, hv2, _ = o.limit(h, hu, hv)
    assert np.array_equal(h2, h) and np.array_equal(hu2, hu) and np.array_equal(hv2, hv)
    # linear state, M = 0: elements with three real neighbours keep their polynomial
    # (Delta u_i = grad u . (m_i - b0) = u_tilde_i, so mbar(a, nu a) = a)
    lin = lambda x, y: (2.0 + 0.3 * x - 0.2 * y, 0.5 + 0.1 * x + 0.2 * y, -0.3 + 0.05 * x)  # noqa: E731
    o, d, h, hu, hv = _wall_mesh_state(lin)
    h2, hu2, hv2, _ = o.limit(h, hu, hv)
    e2e, e2f = o.connectivity()
    interior = np.all(e2e != np.arange(o.K)[:, None], axis=1)
    for a, b in ((h, h2), (hu, hu2), (hv, hv2)):
        assert np.abs(a - b)[interior].max() < 1e-13


def test_tvb_limits_oscillation_and_skips_near_dry():
    def osc(x, y):
        h = 1.0 + 0.2 * np.sign(np.sin(7 * x + 3 * y)) + 0.05 * np.cos(25 * x)
        return h, np.zeros_like(x), np.zeros_like(x)

    o, d, h, hu, hv = _wall_mesh_state(osc)
    h2, hu2, hv2, dry = o.limit(h, hu, hv)
    assert o.info()["n_tvb"] > 0  # oscillatory data does get limited
    wm = oracle.refel(2)["wmean"]
    assert np.abs(0.5 * h2 @ wm - 0.5 * h @ wm).max() < 1e-14  # means preserved
    # make element 0 dry: neither it nor its neighbours may be touched by TVB
    e2e, _ = o.connectivity()
    h_d = h.copy()
    h_d[0] = 1e-9
    nb = [n for n in e2e[0] if n != 0]
    o2, d2, _, _, _ = _wall_mesh_state(osc)
    h3, _, _, dry3 = o2.limit(h_d, hu, hv)
    assert dry3[0] == 1
    for n in nb:
        if h_d[n].min() > 1e-6:  # PP leaves it alone, so any change would be TVB's
            assert np.array_equal(h3[n], h_d[n])
