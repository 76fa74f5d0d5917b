"""Pins for the oracle's time stepping: AB3, level grouping,
MRAB recursive schedule with dense output (Alg. 1, reading A17), mesh and
whole-scheme invariants (P:158 C-property, P:220 positivity, P:221 mass)."""
import json
import math
import os

import numpy as np
import pytest
from scipy.linalg import expm

import oracle
import swe_inputs as si
from tests.common import make_oracle

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "limiter_examples.json")))


def _toy_errors(A, level, L, T, dts, seeded, coupling=0):
    K = A.shape[0]
    y0 = np.linspace(1.0, 0.5, K)
    errs = []
    for dt in dts:
        nsteps = int(round(T / (dt * 2 ** (L - 1))))
        s0 = s1 = None
        if seeded:  # exact AB history at each element's own level step
            lev = np.asarray(level)
            h = dt * 2.0 ** (lev - 1)
            s0 = np.array([(A @ expm(-2 * h[e] * A) @ y0)[e] for e in range(K)])
            s1 = np.array([(A @ expm(-1 * h[e] * A) @ y0)[e] for e in range(K)])
        y = oracle.toy_mrab(A, level, y0, dt, L, nsteps, s0, s1, coupling=coupling)
        errs.append(np.abs(y - expm(T * A) @ y0).max())
    return np.array(errs)


def test_ab3_single_rate_order():
    A = np.array([[-1.0]])
    dts = [0.1, 0.05, 0.025]
    e = _toy_errors(A, [1], 1, 1.0, dts, seeded=True)
    assert np.all(np.abs(np.log2(e[:-1] / e[1:]) - 3.0) < 0.1)
    e = _toy_errors(A, [1], 1, 1.0, dts, seeded=False)  # Euler -> AB2 -> AB3 ramp (A18)
    assert np.all(np.abs(np.log2(e[:-1] / e[1:]) - 2.0) < 0.15)


def test_mrab_three_level_order():
    """Recursive slowest-first MRAB with AB3 dense output is third order (A17)."""
    A = np.array([[-1.0, 0.5, 0.0], [0.3, -0.8, 0.4], [0.0, 0.6, -0.5]])
    level = [1, 2, 3]
    dts = [0.02, 0.01, 0.005]
    e = _toy_errors(A, level, 3, 2.0, dts, seeded=True)
    assert np.all(np.abs(np.log2(e[:-1] / e[1:]) - 3.0) < 0.15)
    e = _toy_errors(A, level, 3, 2.0, dts, seeded=False)
    assert np.all(np.log2(e[:-1] / e[1:]) > 1.85)


def test_mrab_printed_order_latest_committed_is_first_order():
    """The variant (SPEC's reading of Alg. 1): the printed loop nest (levels
    descending, substeps inner) with every neighbour at its latest committed value.
    Coupled levels see each other up to one coarse step out of sync, so the scheme is first order
    (SPEC S:419 reports 0.99), while uncoupled levels keep AB3's third order."""
    A = np.array([[-1.0, 0.5, 0.0], [0.3, -0.8, 0.4], [0.0, 0.6, -0.5]])
    dts = [0.02, 0.01, 0.005]
    e = _toy_errors(A, [1, 2, 3], 3, 2.0, dts, seeded=True, coupling=1)
    assert np.all(np.abs(np.log2(e[:-1] / e[1:]) - 1.0) < 0.1)
    Ad = np.diag([-1.0, -0.8, -0.5])  # no coupling: each level is plain AB3
    e = _toy_errors(Ad, [1, 2, 3], 3, 2.0, dts, seeded=True, coupling=1)
    assert np.all(np.abs(np.log2(e[:-1] / e[1:]) - 3.0) < 0.15)
    # one level: identical to the default schedule
    y1 = oracle.toy_mrab(A, [1, 1, 1], [1.0, 2.0, 0.5], 0.01, 1, 40, coupling=1)
    y0 = oracle.toy_mrab(A, [1, 1, 1], [1.0, 2.0, 0.5], 0.01, 1, 40, coupling=0)
    assert np.array_equal(y1, y0)


def test_single_level_is_textbook_ab3():
    """nlevels = 1 reduces to plain AB3 with the Euler/AB2 ramp."""
    A = np.array([[-0.7, 0.2], [0.1, -0.3]])
    y = np.array([1.0, 2.0])
    dt, n = 0.01, 50
    hist = []
    for k in range(n):
        hist.insert(0, A @ y)
        if k == 0:
            y = y + dt * hist[0]
        elif k == 1:
            y = y + dt * (1.5 * hist[0] - 0.5 * hist[1])
        else:
            y = y + dt * (23 * hist[0] - 16 * hist[1] + 5 * hist[2]) / 12
    yo = oracle.toy_mrab(A, [1, 1], [1.0, 2.0], dt, 1, n)
    assert np.abs(yo - y).max() < 1e-14
    # all elements on level 1 of a 3-level schedule == 4 single-rate steps per macro step
    yo3 = oracle.toy_mrab(A, [1, 1], [1.0, 2.0], dt, 3, n // 4 + (1 if n % 4 else 0))
    yref = oracle.toy_mrab(A, [1, 1], [1.0, 2.0], dt, 1, 4 * (n // 4 + (1 if n % 4 else 0)))
    assert np.abs(yo3 - yref).max() < 1e-15


def _triangles(scales, gap=100.0):
    """Disjoint 3-4-5 right triangles scaled by `scales` (Hk = 2 * scale)."""
    vx, vy, etov = [], [], []
    for k, s in enumerate(scales):
        x0 = k * gap
        base = len(vx)
        vx += [x0, x0 + 4 * s, x0]
        vy += [0.0, 0.0, 3 * s]
        etov.append([base, base + 1, base + 2])
    return np.array(vx), np.array(vy), np.array(etov, dtype=np.int32)


def test_hk_and_level_binning_examples():
    ex = GOLDEN["level_binning"]  # S:387-389 of the grouping rule P:127
    a_floor = 10.0
    # r_e = Hk / a_floor = dt_e  ->  Hk = 10 dt_e, scale = Hk / 2
    scales = [a_floor * d / 2.0 for d in ex["dt"]]
    vx, vy, etov = _triangles(scales)
    o = oracle.Oracle(vx, vy, etov, np.zeros((3, 3)), 1, 9.81, a_floor=a_floor, use_pp=0, use_tvb=0)
    J, Hk, nflip = o.geometry()
    assert abs(Hk[0] / scales[0] - GOLDEN["hk_345"]["Hk"]) < 1e-15
    z = np.zeros((3, 3))
    o.set_state(z, z, z)  # dry: a_e = a_floor
    assert list(o.bin_levels(4)) == ex["levels"]
    assert list(o.bin_levels(2)) == [1, 2, 2]  # capped at nlevels
    assert list(o.bin_levels(1)) == [1, 1, 1]
    # uniform dt -> single level; 0.199 < 2 * 0.1 -> level 1
    vx, vy, etov = _triangles([0.5, 0.995])
    o = oracle.Oracle(vx, vy, etov, np.zeros((2, 3)), 1, 9.81, a_floor=a_floor, use_pp=0, use_tvb=0)
    z = np.zeros((2, 3))
    o.set_state(z, z, z)
    assert list(o.bin_levels(3)) == [1, 1]


def test_mesh_connectivity_bruteforce():
    m = si.shuffle(si.structured(5, 4, 0.0, 5.0, 0.0, 4.0), seed=3, flip_fraction=0.3)
    o = oracle.Oracle(m.vx, m.vy, m.etov, np.zeros((m.K, 3)), 1, 9.81)
    e2e, e2f = o.connectivity()
    J, Hk, nflip = o.geometry()
    assert nflip > 0 and np.all(J > 0)
    assert abs(np.sum(2 * J) - 20.0) < 1e-12  # total area = domain area
    # brute force: faces as vertex sets
    faces = {}
    for e in range(m.K):
        v = m.etov[e]
        for a in range(3):
            for b in range(a + 1, 3):
                faces.setdefault(frozenset((v[a], v[b])), []).append(e)
    for e in range(m.K):
        for f in range(3):
            n, nf = e2e[e, f], e2f[e, f]
            if n == e:
                assert nf == f
                continue
            assert e2e[n, nf] == e and e2f[n, nf] == f  # involution
    nint = sum(1 for v in faces.values() if len(v) == 2)
    assert (e2e != np.arange(m.K)[:, None]).sum() == 2 * nint


def test_mesh_errors_and_periodic():
    vx = np.array([0.0, 1.0, 0.0, 1.0])
    vy = np.array([0.0, 0.0, 1.0, 1.0])
    with pytest.raises(ValueError):  # out of range
        oracle.Oracle(vx, vy, np.array([[0, 1, 7]]), np.zeros((1, 3)), 1, 9.81)
    with pytest.raises(ValueError):  # zero area
        oracle.Oracle(vx, vy, np.array([[0, 1, 1]]), np.zeros((1, 3)), 1, 9.81)
    with pytest.raises(ValueError):  # duplicated element -> face with 3 owners? (non-conforming)
        oracle.Oracle(vx, vy, np.array([[0, 1, 3], [0, 1, 3], [0, 1, 2]]), np.zeros((3, 3)), 1, 9.81)
    o = oracle.Oracle(vx, vy, np.array([[0, 1, 2]]), np.zeros((1, 3)), 1, 9.81)
    e2e, e2f = o.connectivity()
    assert list(e2e[0]) == [0, 0, 0] and list(e2f[0]) == [0, 1, 2]
    m = si.structured(4, 3, 0.0, 1.0, 0.0, 1.0, periodic=True)
    o = oracle.Oracle(m.vx, m.vy, m.etov, np.zeros((m.K, 3)), 1, 9.81, vper=m.vper)
    e2e, _ = o.connectivity()
    assert np.all(e2e != np.arange(m.K)[:, None])  # every face matched


def test_lake_at_rest_100_steps_with_limiters():
    """C1a: max|h + B - 0| <= 1e-12 after 100 steps, no TVB trigger."""
    w = si.c1_lake(N=2)
    o, d = make_oracle(w)
    o.set_state(d["h"], d["hu"], d["hv"])
    dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2)
    for _ in range(100):
        assert o.step(dt, 1) == 0
    h, hu, hv = o.get_state()
    assert np.abs(h + d["B"]).max() < 1e-12
    assert max(np.abs(hu).max(), np.abs(hv).max()) < 1e-12
    assert o.info()["n_tvb"] == 0


def test_thacker_mass_positivity_accuracy():
    """C3 (coarse): mass conserved to round-off modulo dry injection (A13), h >= 0
    at every node after every step, and the solution tracks Eq. pb_exact."""
    w = si.c3_thacker(N=2, n=40)
    o, d = make_oracle(w)
    o.set_state(d["h"], d["hu"], d["hv"])
    ex, om = si.thacker_exact()
    i0 = o.info()
    dt = si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)
    nsteps = 150
    for _ in range(nsteps):
        assert o.step(dt, 1) == 0
        assert o.info()["min_h"] >= 0.0
    i1 = o.info()
    drift = i1["mass"] - i0["mass"] - (i1["injected_mass"] - i0["injected_mass"])
    assert abs(drift) < 1e-13 * i0["mass"]
    assert i1["n_pp"] > 0
    h, hu, hv = o.get_state()
    he, _, _ = ex(d["x"], d["y"], nsteps * dt)
    assert np.abs(h - he).max() < 0.05 * he.max()


def test_thacker_initial_state_at_the_origin():
    """Alg. 2 line 1 leaves the smooth wet interior of the bowl untouched: the oracle's
    limited initial depth at the node sitting on the origin is Eq. pb_exact's 1/(X+Y) (golden)."""
    w = si.c3_thacker(N=2, n=40)
    o, d = make_oracle(w)
    o.set_state(d["h"], d["hu"], d["hv"])
    at0 = (np.abs(d["x"]) < 1e-9) & (np.abs(d["y"]) < 1e-9)
    assert at0.sum() >= 1
    assert np.abs(o.get_state()[0][at0] - GOLDEN["thacker_h_origin"]["h"]).max() < 1e-12


@pytest.mark.parametrize("N", [1, 2, 3])
def test_thacker_global_error_rate(N):
    """on the parabolic bowl the global L2 error of the height converges like O(H^1.5) for
    N = 1, 2, 3 (the front is continuous but not C^1), while away from the front it is faster.
    Meshes 2 x n x n, n = 16, 32, 64 (H = 500, 250, 125 m), to t = T/4 (T = 2 pi / omega).
    Measured: global rates 1.37/1.68 (N=1), 1.29/1.51 (N=2), 1.23/1.47 (N=3)."""
    import math
    from tests.test_oracle_verification import _l2
    ex, om = si.thacker_exact()
    t_end = 0.25 * 2 * math.pi / om
    glob, loc = [], []
    for n in (16, 32, 64):
        w = si.c3_thacker(N=N, n=n)
        o, d = make_oracle(w)
        o.set_state(d["h"], d["hu"], d["hv"])
        dt = si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)
        ns = int(math.ceil(t_end / dt))
        for _ in range(ns):
            assert o.step(t_end / ns, 1) == 0
        assert o.info()["min_h"] >= 0.0
        glob.append(_l2(o, w, t_end))
        loc.append(_l2(o, w, t_end, region=lambda x, y: x * x + y * y < 1500.0 ** 2))
    rates = [math.log2(glob[0] / glob[1]), math.log2(glob[1] / glob[2])]
    assert rates[0] > 1.1 and rates[1] > 1.4, rates
    assert math.log2(loc[1] / loc[2]) > rates[1] + 0.2


def test_oracle_regroup_is_set_state_of_the_current_state():
    """Level regrouping: identical to swe_set_state of the current state, except that the
    simulated time continues."""
    w = si.c4_dambreak(N=2, base=10)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    a, d = make_oracle(w)
    b, _ = make_oracle(w)
    for o in (a, b):
        o.set_state(d["h"], d["hu"], d["hv"])
        for _ in range(3):
            assert o.step(dt, 3) == 0
    t1 = a.info()["t"]
    a.regroup()
    b.set_state(*b.get_state())
    for o in (a, b):
        for _ in range(2):
            assert o.step(0.5 * dt, 2) == 0
    for x, y in zip(a.get_state(), b.get_state()):
        assert np.array_equal(x, y)
    assert np.array_equal(a.levels(), b.levels())
    assert abs(a.info()["t"] - (t1 + b.info()["t"])) < 1e-12 * t1
