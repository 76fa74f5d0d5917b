"""Pins for the oracle's RHS: flux, volume/surface assembly
(P:641-706), well-balancing (P:158 exact C-property), conservation."""
import math

import numpy as np
import pytest

import oracle
import swe_inputs as si
from tests.common import make_oracle


def test_velocity_desingularisation():
    # A4: vel -> m/h for h >> eps_u, 0 at h <= 0, bounded near 0
    assert abs(oracle.vel(2.0, 2.0, 1e-8) - 1.0) < 1e-15
    assert abs(oracle.vel(1.0, 3.0, 1e-8) - 3.0) < 1e-15
    assert oracle.vel(0.0, 1.0, 1e-3) == 0.0
    assert oracle.vel(-1.0, 1.0, 1e-3) == 0.0
    assert abs(oracle.vel(1e-3, 1e-6, 1e-3) - 1e-3 / math.sqrt(2.0) * math.sqrt(2.0)) < 1e-12


def fn(q, n, g):
    h, hu, hv = q
    u, v = hu / h, hv / h
    un = u * n[0] + v * n[1]
    return np.array([h * un, hu * un + 0.5 * g * h * h * n[0], hv * un + 0.5 * g * h * h * n[1]])


def test_flux_consistency_flat_bottom():
    rng = np.random.default_rng(0)
    for _ in range(20):
        q = np.array([rng.uniform(0.5, 2), rng.normal(), rng.normal()])
        th = rng.uniform(0, 2 * math.pi)
        n = (math.cos(th), math.sin(th))
        F = oracle.flux(q, 0.0, q, 0.0, n, g=9.81)
        assert np.abs(F - fn(q, n, 9.81)).max() < 1e-13  # LF consistency, penalty vanishes


def test_flux_rotational_invariance_and_conservation():
    rng = np.random.default_rng(1)
    g = 9.81
    for _ in range(20):
        qm = np.array([rng.uniform(0.5, 2), rng.normal(), rng.normal()])
        qp = np.array([rng.uniform(0.5, 2), rng.normal(), rng.normal()])
        th = rng.uniform(0, 2 * math.pi)
        n = np.array([math.cos(th), math.sin(th)])
        F = oracle.flux(qm, 0.0, qp, 0.0, n, g=g)
        # rotate to the normal frame: (h, m.n, m.t) with n -> (1,0)
        Rot = np.array([[1, 0, 0], [0, n[0], n[1]], [0, -n[1], n[0]]])
        Fr = oracle.flux(Rot @ qm, 0.0, Rot @ qp, 0.0, (1.0, 0.0), g=g)
        assert np.abs(Rot.T @ Fr - F).max() < 1e-12
        # the neighbour sees the opposite normal: all components antisymmetric with flat B
        Fo = oracle.flux(qp, 0.0, qm, 0.0, -n, g=g)
        assert np.abs(F + Fo).max() < 1e-12


def test_hydrostatic_reconstruction_examples():
    g = 1.0
    # (h+,B+,h-,B-) = (2,0,1,1): Bmax = 1, h*+ = 1, h*- = 1: equal stars -> no mass flux, lake pressure
    F = oracle.flux([1.0, 0.0, 0.0], 1.0, [2.0, 0.0, 0.0], 0.0, (1.0, 0.0), g=g)
    # own total = g/2 h*^2 n + g/2((h-)^2 - (h*-)^2 - (B-)^2) n = g/2 (1 - 1) n
    assert np.allclose(F, [0.0, 0.5 * g * (1.0 - 1.0), 0.0], atol=1e-15)
    # (h+,B+,h-,B-) = (0,2,1,0): h*+ = 0, h*- = max(0, 1-2) = 0, dry wall blocks flow
    F = oracle.flux([1.0, 0.5, 0.0], 0.0, [0.0, 0.0, 0.0], 2.0, (1.0, 0.0), g=g)
    assert F[0] == 0.0 and abs(F[1] - 0.5 * g * 1.0) < 1e-15


def test_lake_at_rest_flux_is_split_pressure():
    rng = np.random.default_rng(2)
    g = 9.81
    for _ in range(10):
        eta = 1.0
        bm, bp = rng.uniform(-1, 0.5, 2)
        th = rng.uniform(0, 2 * math.pi)
        n = (math.cos(th), math.sin(th))
        F = oracle.flux([eta - bm, 0, 0], bm, [eta - bp, 0, 0], bp, n, g=g)
        p = 0.5 * g * ((eta - bm) ** 2 - bm ** 2)
        assert np.abs(F - np.array([0.0, p * n[0], p * n[1]])).max() < 1e-13


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_lake_at_rest_rhs_vanishes(N):
    """Exact C-property with the split source (reading A3), at the paper's quadrature."""
    w = si.c1_lake(N=N, n=6)
    o, d = make_oracle(w)
    R = o.rhs(d["h"], d["hu"], d["hv"])
    scale = 9.81 * 1.0 * 2.0  # g * h * |grad B|
    for r in R:
        assert np.abs(r).max() < 1e-12 * scale * N ** 2


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_free_stream_preserved_periodic(N):
    w = si.c2_vortex(N, 6)
    o, d = make_oracle(w)
    h = np.full_like(d["x"], 1.3)
    R = o.rhs(h, 0.4 * h, -0.7 * h)
    for r in R:
        assert np.abs(r).max() < 1e-12


@pytest.mark.parametrize("N", [1, 2, 3])
def test_semidiscrete_conservation_periodic(N):
    """sum_e J int R_h = 0 (mass), and momentum too with flat bottom, on a periodic mesh."""
    w = si.c2_vortex(N, 8)
    o, d = make_oracle(w)
    ex = si.vortex_exact()
    rng = np.random.default_rng(3)
    h, hu, hv = ex(d["x"], d["y"], 0.3)
    h = h + 0.05 * rng.standard_normal(h.shape)  # discontinuous across elements
    R = o.rhs(h, hu, hv)
    J, Hk, _ = o.geometry()
    wm = oracle.refel(N)["wmean"]
    for k, r in enumerate(R):
        tot = np.sum(J[:, None] * r * wm[None, :])
        assert abs(tot) < 1e-12 * np.abs(J[:, None] * r).sum(), k


def test_vortex_rhs_consistency_order():
    """R(Q_exact) -> dQ/dt of the exact vortex (g = 2) at rate H^N in L2."""
    ex = si.vortex_exact()
    N = 3
    errs = []
    for n in (64, 128):
        w = si.c2_vortex(N, n)
        o, d = make_oracle(w)
        x, y = d["x"], d["y"]
        R = o.rhs(*ex(x, y, 0.0))
        dt = 1e-5
        dq = [(a - b) / (2 * dt) for a, b in zip(ex(x, y, dt), ex(x, y, -dt))]
        J, _, _ = o.geometry()
        wm = oracle.refel(N)["wmean"]
        errs.append(np.sqrt(sum(np.sum(J[:, None] * wm[None, :] * (r - q) ** 2) for r, q in zip(R, dq))))
    assert np.log2(errs[0] / errs[1]) > N - 0.3


@pytest.mark.parametrize("N", [2, 3])
def test_vortex_convergence_eoc(N):
    """Translating vortex to t = 0.25: L2 error in h decays like H^{N+1} (paper: >= N+1/2)."""
    ex = si.vortex_exact()
    T = 0.25
    errs = []
    for n in (32, 64):
        w = si.c2_vortex(N, n)
        o, d = make_oracle(w)
        o.set_state(d["h"], d["hu"], d["hv"])
        dt0 = si.dt_for(w.mesh, N, 2.0, 1.0, 0.0, 0.1, u_max=2.0)
        nst = int(np.ceil(T / dt0))
        for _ in range(nst):
            assert o.step(T / nst, 1) == 0
        h, _, _ = o.get_state()
        he, _, _ = ex(d["x"], d["y"], T)
        J, _, _ = o.geometry()
        wm = oracle.refel(N)["wmean"]
        errs.append(np.sqrt(np.sum(J[:, None] * wm[None, :] * (h - he) ** 2)))
    assert np.log2(errs[0] / errs[1]) > N + 0.5
