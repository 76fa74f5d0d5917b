"""Pins for the oracle's reference element.

Every check is against mathematics, not against the oracle's own formulas:
closed-form 1D rules, exact monomial integrals on the triangle (rational
arithmetic), exact derivatives of random polynomials, numpy's independent
Gauss-Legendre for line integrals."""
import math

import numpy as np
import pytest

import oracle
from tests.common import poly_dr, poly_ds, poly_eval, poly_integral, poly_mul, random_poly, tri_monomial_integral


@pytest.mark.parametrize("q", range(1, 10))
def test_gauss_legendre_exactness(q):
    x, w = oracle.quad("gl", q)
    for k in range(2 * q):
        exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
        assert abs(np.dot(w, x ** k) - exact) < 1e-14
    k = 2 * q  # first failing degree
    assert abs(np.dot(w, x ** k) - 2.0 / (k + 1)) > 1e-8
    xr, wr = np.polynomial.legendre.leggauss(q)
    assert np.allclose(x, xr, atol=1e-15) and np.allclose(w, wr, atol=1e-15)


@pytest.mark.parametrize("q", range(1, 10))
def test_gauss_jacobi10_exactness(q):
    # int_{-1}^{1} (1-x) x^k dx = 2/(k+1) [k even] - 2/(k+2) [k odd]
    x, w = oracle.quad("gj10", q)
    for k in range(2 * q):
        exact = (2.0 / (k + 1) if k % 2 == 0 else 0.0) - (2.0 / (k + 2) if k % 2 == 1 else 0.0)
        assert abs(np.dot(w, x ** k) - exact) < 1e-14
    assert np.all(w > 0) and np.all(np.abs(x) < 1)


def test_lobatto_closed_forms():
    assert np.allclose(oracle.quad("lgl", 1)[0], [-1, 1])
    assert np.allclose(oracle.quad("lgl", 2)[0], [-1, 0, 1], atol=1e-16)
    assert np.allclose(oracle.quad("lgl", 3)[0], [-1, -1 / math.sqrt(5), 1 / math.sqrt(5), 1], atol=1e-15)
    assert np.allclose(oracle.quad("lgl", 4)[0], [-1, -math.sqrt(3 / 7), 0, math.sqrt(3 / 7), 1], atol=1e-15)


@pytest.mark.parametrize("N", range(1, 9))
def test_nodes(N):
    re = oracle.refel(N)
    r, s = re["r"], re["s"]
    Np = (N + 1) * (N + 2) // 2
    assert len(r) == Np  # P:631 Np = (N+1)(N+2)/2
    lgl = oracle.quad("lgl", N)[0]
    # exactly N+1 nodes per edge, at the LGL points (warp of Warp & Blend)
    on_f0 = np.abs(s + 1) < 1e-12
    on_f1 = np.abs(r + s) < 1e-12
    on_f2 = np.abs(r + 1) < 1e-12
    assert on_f0.sum() == N + 1 and on_f1.sum() == N + 1 and on_f2.sum() == N + 1
    assert np.allclose(np.sort(r[on_f0]), lgl, atol=1e-14)
    assert np.allclose(np.sort(s[on_f2]), lgl, atol=1e-14)
    # symmetric under the triangle's symmetry group (as multisets): barycentric permutations
    L = np.stack([-(r + s) / 2, (1 + r) / 2, (1 + s) / 2], 1)
    key = lambda a: np.array(sorted(map(tuple, np.round(a, 12))))  # noqa: E731
    for perm in [(1, 0, 2), (0, 2, 1), (2, 1, 0), (1, 2, 0)]:
        assert np.allclose(key(L[:, perm]), key(L), atol=1e-12)
    # HW Nodes2D order: rows of constant s upward, r increasing in a row
    assert np.allclose(r[: N + 1], lgl, atol=1e-14) and np.allclose(s[: N + 1], -1)
    if N == 1:
        assert np.allclose(np.c_[r, s], [[-1, -1], [1, -1], [-1, 1]])
    if N == 2:  # vertices + edge midpoints
        assert np.allclose(np.c_[r, s], [[-1, -1], [0, -1], [1, -1], [-1, 0], [0, 0], [-1, 1]], atol=1e-15)
    if N == 3:  # one interior node: the centroid
        inner = ~(on_f0 | on_f1 | on_f2)
        assert inner.sum() == 1 and np.allclose([r[inner][0], s[inner][0]], [-1 / 3, -1 / 3], atol=1e-15)


@pytest.mark.parametrize("N", range(1, 9))
def test_cubature_exactness(N):
    """P:81 + P:108-110 (reading A2'): symmetric rule of degree exactly 2N for N <= 5
    (Dunavant sizes 3, 6, 12, 16, 25), collapsed Gauss-Jacobi of degree 2N+1 above."""
    re = oracle.refel(N)
    rc, sc, wc = re["rc"], re["sc"], re["wc"]
    sym = N <= 5
    npts = {1: 3, 2: 6, 3: 12, 4: 16, 5: 25}[N] if sym else (N + 1) ** 2
    strength = 2 * N if sym else 2 * N + 1
    assert len(wc) == npts and np.all(wc > 0)
    assert abs(wc.sum() - 2.0) < 1e-14
    inside = (rc > -1) & (sc > -1) & (rc + sc < 0)
    assert inside.all()
    for a in range(strength + 1):
        for b in range(strength + 1 - a):
            ex = float(tri_monomial_integral(a, b))
            assert abs(np.dot(wc, rc ** a * sc ** b) - ex) < 1e-13, (a, b)
    # degree strength+1 is not integrated exactly by every monomial (rule strength pinned)
    d = strength + 1
    errs = [abs(np.dot(wc, rc ** a * sc ** (d - a)) - float(tri_monomial_integral(a, d - a))) for a in range(d + 1)]
    assert max(errs) > 1e-10


@pytest.mark.parametrize("N", range(1, 6))
def test_symmetric_cubature_orbits(N):
    """The rule is fully symmetric: invariant (as a weighted point set) under the six
    affine maps of the reference triangle onto itself (vertex permutations)."""
    re = oracle.refel(N)
    rc, sc, wc = re["rc"], re["sc"], re["wc"]
    # barycentric of (r,s): l1 = -(r+s)/2, l2 = (1+r)/2, l3 = (1+s)/2
    L = np.stack([-(rc + sc) / 2, (1 + rc) / 2, (1 + sc) / 2], 1)
    key = lambda lam, w: sorted(zip(np.round(lam[:, 0], 12), np.round(lam[:, 1], 12), np.round(w, 12)))
    base = key(L, wc)
    import itertools
    for perm in itertools.permutations(range(3)):
        assert key(L[:, perm], wc) == base, perm
    # Dunavant's published values (Table, degrees 2..10) agree to their printed digits
    pub = {3: (0.116786275726379, 0.501426509658179), 4: (0.103217370534718, 0.658861384496480)}
    if N in pub:
        w, a = pub[N]
        hit = np.isclose(L[:, 0], a, atol=1e-14) & np.isclose(L[:, 1], (1 - a) / 2, atol=1e-14)
        assert hit.sum() == 1 and abs(wc[hit][0] / 2 - w) < 1e-14


@pytest.mark.parametrize("N", range(1, 7))
def test_operators_exact_on_polynomials(N):
    re = oracle.refel(N)
    r, s = re["r"], re["s"]
    rng = np.random.default_rng(1403 + N)
    p = random_poly(N, rng)
    pv = poly_eval(p, r, s)
    scale = max(1.0, np.abs(pv).max())
    # Dr, Ds: exact derivatives
    assert np.abs(re["Dr"] @ pv - poly_eval(poly_dr(p), r, s)).max() < 1e-11 * scale * N ** 2
    assert np.abs(re["Ds"] @ pv - poly_eval(poly_ds(p), r, s)).max() < 1e-11 * scale * N ** 2
    # interpolation to cubature / Gauss points reproduces the polynomial
    assert np.abs(re["Ic"] @ pv - poly_eval(p, re["rc"], re["sc"])).max() < 1e-12 * scale
    assert np.abs(re["Ig"] @ pv - poly_eval(p, re["rg"], re["sg"])).max() < 1e-12 * scale
    # Mref: v^T M u = int u v  (exact rational integration)
    q = random_poly(N, rng)
    qv = poly_eval(q, r, s)
    assert abs(qv @ re["Mref"] @ pv - poly_integral(poly_mul(p, q))) < 1e-12 * scale
    assert abs(re["wmean"].sum() - 2.0) < 1e-13
    # P, Pr, Ps: v^T M (P F_c) = int v F for F of degree N, v^T M (Pr F_c) = int dv/dr F
    # for F of degree N+1 (integrands of degree 2N: the cubature strength, A2')
    M = re["Mref"]
    F0 = random_poly(N, rng)
    assert abs(qv @ M @ (re["P"] @ poly_eval(F0, re["rc"], re["sc"])) - poly_integral(poly_mul(q, F0))) < 1e-11 * scale
    F = random_poly(N + 1, rng)
    Fc = poly_eval(F, re["rc"], re["sc"])
    assert abs(qv @ M @ (re["Pr"] @ Fc) - poly_integral(poly_mul(poly_dr(q), F))) < 1e-11 * scale * N
    assert abs(qv @ M @ (re["Ps"] @ Fc) - poly_integral(poly_mul(poly_ds(q), F))) < 1e-11 * scale * N
    # Lg: v^T M (Lg F_g) = sum over faces of int_{-1}^{1} v F dt (face parameter t)
    tg, wg = np.polynomial.legendre.leggauss(2 * N + 4)
    verts = np.array([[-1, -1], [1, -1], [-1, 1]], dtype=float)
    exact = 0.0
    for f in range(3):
        a, b = verts[f], verts[(f + 1) % 3]
        pr = 0.5 * (1 - tg) * a[0] + 0.5 * (1 + tg) * b[0]
        ps = 0.5 * (1 - tg) * a[1] + 0.5 * (1 + tg) * b[1]
        exact += np.dot(wg, poly_eval(q, pr, ps) * poly_eval(F, pr, ps))
    Fg = poly_eval(F, re["rg"], re["sg"])
    assert abs(qv @ M @ (re["Lg"] @ Fg) - exact) < 1e-11 * scale


def test_gauss_points_along_faces():
    re = oracle.refel(3)
    Ng = re["Ng"]
    rg, sg = re["rg"].reshape(3, Ng), re["sg"].reshape(3, Ng)
    assert np.allclose(sg[0], -1) and np.all(np.diff(rg[0]) > 0)      # face 0: v0 -> v1
    assert np.allclose(rg[1] + sg[1], 0) and np.all(np.diff(sg[1]) > 0)  # face 1: v1 -> v2
    assert np.allclose(rg[2], -1) and np.all(np.diff(sg[2]) < 0)     # face 2: v2 -> v0
