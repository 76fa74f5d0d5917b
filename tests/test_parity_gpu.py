"""GPU parity: the CUDA path (through the C ABI) against the independent CPU
oracle on identical seeded inputs.  Tolerance (north_star): relative L_inf
<= 1e-12 per field (A23 scales) after the stated number of steps; levels and
connectivity bit-exact."""
import numpy as np
import pytest

import oracle
import paper_1403_1661_b200 as P
import swe_inputs as si
from tests.common import make_oracle, parity_rel

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    P.build()
    P.lib()


def make_pair(w, **over):
    o, d = make_oracle(w, **{k: v for k, v in over.items() if k != "record_decisions"})
    prm = dict(w.params)
    prm.update(over)
    m = w.mesh
    s = P.Solver(m.vx, m.vy, m.etov, d["B"], w.N, w.g, vper=m.vper, params=prm, vbc=m.vbc)
    return o, s, d


def run_both(w, nsteps, dt, nlevels=1, **over):
    o, s, d = make_pair(w, **over)
    o.set_state(d["h"], d["hu"], d["hv"])
    s.set_state(d["h"], d["hu"], d["hv"])
    for _ in range(nsteps):
        assert o.step(dt, nlevels) == 0
        s.step(dt, nlevels)
    return o, s, d


def assert_parity(o, s, g, tol=TOL):
    rel = parity_rel(s.get_state(), o.get_state(), g)
    assert max(rel) <= tol, rel
    return rel


def test_initial_limiting_matches():
    """Alg. 2 line 1 on a wet/dry state: get_state right after set_state."""
    w = si.c3_thacker(N=2, n=30)
    o, s, d = make_pair(w)
    o.set_state(d["h"], d["hu"], d["hv"])
    s.set_state(d["h"], d["hu"], d["hv"])
    assert_parity(o, s, w.g)
    assert s.info()["n_dry"] == o.info()["n_dry"] > 0


def test_lake_at_rest_c1a_gpu():
    w = si.c1_lake(N=2)
    o, s, d = make_pair(w)
    s.set_state(d["h"], d["hu"], d["hv"])
    dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2)
    for _ in range(100):
        s.step(dt, 1)
    h, hu, hv = s.get_state()
    assert np.abs(h + d["B"]).max() < 1e-12
    assert max(np.abs(hu).max(), np.abs(hv).max()) < 1e-12
    assert s.info()["n_tvb"] == 0


def test_parity_c1b_hump_100_steps():
    w = si.c1_lake(N=2, hump=True)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2)
    o, s, _ = run_both(w, 100, dt)
    assert_parity(o, s, w.g)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_parity_vortex_periodic(N):
    w = si.c2_vortex(N, 12)
    dt = si.dt_for(w.mesh, N, 2.0, 1.0, 0.0, 0.1, u_max=2.0)
    o, s, _ = run_both(w, 60, dt)
    assert_parity(o, s, w.g)


def test_parity_thacker_pp_tvb():
    """C3 recipe (wet/dry, PP + TVB) on a 2x40x40 mesh, 100 steps."""
    w = si.c3_thacker(N=2, n=40)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)
    o, s, _ = run_both(w, 100, dt)
    assert_parity(o, s, w.g)
    io, ig = o.info(), s.info()
    assert io["n_pp"] == ig["n_pp"] and io["n_dry"] == ig["n_dry"] and io["n_tvb"] == ig["n_tvb"]
    assert abs(io["injected_mass"] - ig["injected_mass"]) <= 1e-12 * max(1.0, io["injected_mass"])


def _counters_equal(o, s, keys=("n_pp", "n_dry", "n_tvb", "n_posfix", "n_tvb_cw")):
    io, ig = o.info(), s.info()
    for k in keys:
        assert io[k] == ig[k], (k, io[k], ig[k])
    assert abs(io["injected_mass"] - ig["injected_mass"]) <= 1e-12 * max(1.0, abs(io["injected_mass"]))
    return io


def run_replayed(w, nsteps, dt, nlevels=1, **over):
    """GPU run with the limiter decision log on, then the oracle replaying it: where the
    oracle's own decision lies within 1e-9 (relative) of a threshold it adopts the GPU's; any larger
    disagreement is a mismatch.  The discontinuous limiters (Alg. 3, TVB, Eq. modified_TVB) act on
    states that sit exactly on their thresholds (a vertex lifted to h0 stays at h0 while the element
    is at rest), where the last bit of two independent codes decides the branch."""
    o, s, d = make_pair(w, record_decisions=1, **over)
    s.set_state(d["h"], d["hu"], d["hv"])
    for _ in range(nsteps):
        s.step(dt, nlevels)
    log = s.decisions()
    o.set_replay(log)
    o.set_state(d["h"], d["hu"], d["hv"])
    for _ in range(nsteps):
        assert o.step(dt, nlevels) == 0
    assert o.info()["n_mismatch"] == 0, o.info()
    return o, s, d


def test_parity_thacker_tvb_and_modified_tvb_fire():
    """C3 Thacker bowl with a small TVB constant (M = 1e-7) so that the TVB limiter replaces elements
    along the moving wet/dry front and Eq. modified_TVB lifts vertices to h0 -- the paper's
    wet/dry limiter interplay -- 100 steps, decision replay, counters equal, 1e-12 parity."""
    w = si.c3_thacker(N=2, n=40)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)
    o, s, _ = run_replayed(w, 100, dt, tvb_M=1e-7)
    rel = assert_parity(o, s, w.g)
    io = _counters_equal(o, s)
    assert io["n_tvb"] > 1000 and io["n_posfix"] > 100, io
    print("thacker M=1e-7:", rel, io)


def test_parity_oscillating_lake_tvb_and_modified_tvb_fire():
    """Oscillating lake (the paper's test of "the positivity preserving limiter and the
    modified TVB limiter") with M = 0.01: TVB and Eq. modified_TVB act along the moving front every step.
    This configuration amplifies round-off (reading A29): the oracle itself, started from its
    input perturbed by 1e-15 (relative), drifts from its unperturbed run to ~1e-12 by step 20 and ~1e-9 by
    step 100 -- the GPU and the oracle part on the same curve.  So: 1e-12 parity and equal counters after
    10 steps; after 100 steps the GPU-oracle distance must stay within 10x the oracle's own sensitivity."""
    w = si.c8_oscillating_lake(2, 16)
    dt = si.dt_for(w.mesh, w.N, w.g, 0.2, 0.0, 0.2, u_max=0.5)
    o, s, _ = run_replayed(w, 10, dt, tvb_M=0.01)
    rel10 = assert_parity(o, s, w.g)
    io = _counters_equal(o, s)
    assert io["n_tvb"] > 100 and io["n_posfix"] > 20, io
    o, s, d = run_replayed(w, 100, dt, tvb_M=0.01)
    op, _ = make_oracle(w, tvb_M=0.01)
    rng = np.random.default_rng(1)
    op.set_state(*(a * (1 + 1e-15 * rng.standard_normal(a.shape)) for a in (d["h"], d["hu"], d["hv"])))
    for _ in range(100):
        assert op.step(dt, 1) == 0
    sens = max(parity_rel(op.get_state(), o.get_state(), w.g))
    rel = max(parity_rel(s.get_state(), o.get_state(), w.g))
    assert sens > 1e-12  # ill-conditioned: otherwise the plain 1e-12 bound applies
    assert rel <= 10 * sens, (rel, sens)
    io, ig = o.info(), s.info()
    assert io["n_tvb"] > 1000 and io["n_posfix"] > 100 and abs(io["n_posfix"] - ig["n_posfix"]) <= 10
    print("lake M=0.01: rel@10", rel10, "rel@100", rel, "oracle sensitivity@100", sens, io)


def test_parity_mrab_dambreak_tvb_fires():
    """C4 dam break, 3 MRAB levels, M = 0.05: TVB replacements through the level-aware schedule."""
    w = si.c4_dambreak(N=3, base=5)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    o, s, _ = run_replayed(w, 12, dt, nlevels=3, tvb_M=0.05)
    assert np.array_equal(o.levels(), s.levels())
    rel = assert_parity(o, s, w.g)
    io = _counters_equal(o, s)
    assert io["n_tvb"] > 100, io
    print("C4 M=0.05:", rel, io)


def test_decision_log_without_replay_differs_only_at_ties():
    """Without replay, the oracle's own decisions on the Thacker M = 1e-7 run: every one of them that
    differs from the GPU's log must be a near-threshold case (the replay adopts them all, n_mismatch
    = 0 above), and the state still agrees to 1e-12."""
    w = si.c3_thacker(N=2, n=40)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)
    o, s, _ = run_both(w, 100, dt, tvb_M=1e-7)
    assert_parity(o, s, w.g)


def test_parity_tvb_active():
    """Hump with a small TVB constant so the limiter really fires near the hump (M > 0: with
    M = 0 minmod acts on round-off noise in the flat region and its decisions are random, A14)."""
    w = si.c1_lake(N=2, hump=True, n=16)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2)
    o, s, _ = run_both(w, 60, dt, tvb_M=0.1)
    assert o.info()["n_tvb"] > 0
    assert_parity(o, s, w.g)
    assert o.info()["n_tvb"] == s.info()["n_tvb"]


@pytest.mark.parametrize("nlevels", [2, 3])
def test_parity_mrab_dambreak(nlevels):
    """C4 recipe (NVB-graded, 3 geometric levels, wet/dry, PP + TVB) on a coarsened base mesh."""
    w = si.c4_dambreak(N=3, base=5)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    o, s, _ = run_both(w, 12, dt, nlevels=nlevels)
    assert np.array_equal(o.levels(), s.levels())  # bit-exact level assignment
    assert len(np.unique(s.levels())) == nlevels
    assert_parity(o, s, w.g)


def test_parity_mrab_dambreak_n4_tensor_path():
    """N = 4 runs the volume term and the lift on the FP64 tensor path (DMMA, k_rhs_update_mma2): C4 wet/dry with
    PP + TVB and 3 MRAB levels against the oracle."""
    w = si.c4_dambreak(N=4, base=5)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    o, s, _ = run_both(w, 8, dt, nlevels=3)
    assert np.array_equal(o.levels(), s.levels())
    assert_parity(o, s, w.g)
    assert s.info()["n_pp"] == o.info()["n_pp"] > 0


def test_parity_mrab_smooth_wet():
    """Dense-output coupling without limiter decisions: fully wet graded C4 mesh, smooth hump, 3 levels."""
    w = si.c4_dambreak(N=3, base=5)
    w.bathymetry = (lambda B0: (lambda x, y: B0(x, y) - 4.0))(w.bathymetry)
    w.initial = lambda x, y: (0.1 * np.exp(-((x - 20.0) ** 2 + (y - 15.0) ** 2) / 8.0) - w.bathymetry(x, y),
                              np.zeros_like(x), np.zeros_like(x))
    dt = si.dt_for(w.mesh, w.N, w.g, 4.2, 13.0, 0.2)
    o, s, _ = run_both(w, 10, dt, nlevels=3, tvb_M=1e6)
    assert np.array_equal(o.levels(), s.levels())
    assert len(np.unique(s.levels())) == 3
    assert o.info()["n_pp"] == 0 and o.info()["n_tvb"] == 0
    assert_parity(o, s, w.g)


def test_parity_mrab_dambreak_n5():
    """N = 5 (polynomial order 5, integration order 10 -- the 25-point degree-10 rule) on
    the FP64 tensor path: C4 wet/dry with PP + TVB and 3 MRAB levels against the oracle."""
    w = si.c4_dambreak(N=5, base=5)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    o, s, _ = run_both(w, 6, dt, nlevels=3)
    assert np.array_equal(o.levels(), s.levels())
    assert len(np.unique(s.levels())) == 3
    _counters_equal(o, s)
    assert s.info()["n_pp"] > 0
    assert_parity(o, s, w.g)


@pytest.mark.parametrize("N", [4, 5])
def test_tensor_path_is_run_to_run_bit_identical(N):
    """k_rhs_update_mma2 hands the face fluxes and the RHS between lanes through a shared tile ordered by
    __syncwarp (compute-sanitizer is not available on this pool): a missing order would show up as a result that
    changes from run to run.  Two identical runs on a graded wet/dry mesh, 3 levels, must agree bit for bit."""
    w = si.c4_dambreak(N=N, base=5)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    m = w.mesh
    x, y = P.nodes(m.vx, m.vy, m.etov, N)
    B, h, hu, hv = w.fields(x, y)
    out = []
    for _ in range(2):
        s = P.Solver(m.vx, m.vy, m.etov, B, N, w.g, params=w.params)
        s.set_state(h, hu, hv)
        for _ in range(6):
            s.step(dt, 3)
        out.append(s.get_state())
        s.close()
    for a, b in zip(*out):
        assert np.array_equal(a, b)


def test_get_state_async_matches_synchronous_reads():
    """swe_get_state_async (snapshot gathered on the device, D2H on a copy stream while the next steps run; two
    snapshot buffers) delivers, after swe_wait_state, exactly the state swe_get_state reads at the same point --
    also with three snapshots in flight, where the third waits for the first buffer's copy."""
    import torch
    w = si.c4_dambreak(N=3, base=5)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    m = w.mesh
    x, y = P.nodes(m.vx, m.vy, m.etov, 3)
    B, h, hu, hv = w.fields(x, y)
    ref = []
    s = P.Solver(m.vx, m.vy, m.etov, B, 3, w.g, params=w.params)
    s.set_state(h, hu, hv)
    for _ in range(4):
        s.step(dt, 3)
        ref.append(s.get_state())
    s.close()
    pin = lambda: torch.zeros(h.shape, dtype=torch.float64).pin_memory().numpy()  # noqa: E731
    outs = [tuple(pin() for _ in range(3)) for _ in range(4)]
    s = P.Solver(m.vx, m.vy, m.etov, B, 3, w.g, params=w.params)
    s.set_state(h, hu, hv)
    for k in range(4):
        s.step(dt, 3)
        s.get_state_async(*outs[k])
    s.wait_state()
    s.close()
    for k in range(4):
        for a, b in zip(outs[k], ref[k]):
            assert np.array_equal(a, b), k


def test_convergence_sweep_n1_to_n5_through_the_abi():
    """C2 (BASELINE configs[1]): the translating vortex on periodic meshes 2 x n x n,
    n = 16, 32, 64, N = 1..5, through the C ABI; the L2 error of h converges at least like
    O(H^{N+1/2}) between the two finest meshes (less 0.25 of margin), and the GPU state equals
    the oracle's to 1e-12 on the coarsest one."""
    import math
    rates = []
    for N in range(1, 6):
        errs = []
        for n in (16, 32, 64):
            w = si.c2_vortex(N, n)
            m = w.mesh
            x, y = P.nodes(m.vx, m.vy, m.etov, N)
            B, h, hu, hv = w.fields(x, y)
            s = P.Solver(m.vx, m.vy, m.etov, B, N, w.g, vper=m.vper, params=w.params)
            s.set_state(h, hu, hv)
            # dt ~ H^((N+1)/2): the AB ramp's O(dt^2) temporal error (A18) stays below the O(H^(N+1))
            # spatial error, so the measured rate is the spatial one
            t_end = 0.25
            dt0 = si.dt_for(si.c2_vortex(N, 16).mesh, N, w.g, 1.0, 0.0, 0.1, u_max=2.0) * (16 / n) ** ((N + 1) / 2)
            ns = int(math.ceil(t_end / min(dt0, si.dt_for(m, N, w.g, 1.0, 0.0, 0.1, u_max=2.0))))
            for _ in range(ns):
                s.step(t_end / ns, 1)
            he = w.exact(x, y, t_end)[0]
            v = m.etov
            X, Y = m.vx[v], m.vy[v]
            A = 0.5 * np.abs((X[:, 1] - X[:, 0]) * (Y[:, 2] - Y[:, 0]) - (X[:, 2] - X[:, 0]) * (Y[:, 1] - Y[:, 0]))
            wm = P.host_refel(N, "wmean")
            errs.append(math.sqrt(float(((A / 2.0)[:, None] * wm[None, :] * (s.get_state()[0] - he) ** 2).sum())))
            if n == 16:
                o, d = make_oracle(w)
                o.set_state(d["h"], d["hu"], d["hv"])
                for _ in range(ns):
                    assert o.step(t_end / ns, 1) == 0
                assert max(parity_rel(s.get_state(), o.get_state(), w.g)) <= TOL
            s.close()
        rates.append((N, errs, math.log2(errs[0] / errs[1]), math.log2(errs[1] / errs[2])))
    print("vortex convergence (N, errors n=16/32/64, rates):", rates)
    for N, errs, r0, r1 in rates:
        assert errs[2] < errs[1] < errs[0]
        assert r1 >= N + 0.25, (N, errs, r1)


def test_parity_vortex_dirichlet_boundaries():
    """Dirichlet boundaries (reading A7''; the vortex in [-5,10] x [-6,6] with boundary data from
    the exact solution), N = 2 and 3, 60 steps with the boundary state refreshed before every step."""
    for N in (2, 3):
        w = si.c2_vortex_dirichlet(N, 12)
        o, s, d = make_pair(w)
        x, y = d["x"], d["y"]
        dt = si.dt_for(w.mesh, N, w.g, 1.0, 0.0, 0.1, u_max=2.0)
        for solver in (o, s):
            solver.set_boundary_state(*w.exact(x, y, 0.0))
            solver.set_state(d["h"], d["hu"], d["hv"])
        for k in range(60):
            bs = w.exact(x, y, (k + 0.5) * dt)
            o.set_boundary_state(*bs)
            s.set_boundary_state(*bs)
            assert o.step(dt, 1) == 0
            s.step(dt, 1)
        assert_parity(o, s, w.g)


def test_dirichlet_requires_boundary_state():
    w = si.c2_vortex_dirichlet(2, 8)
    m = w.mesh
    x, y = P.nodes(m.vx, m.vy, m.etov, 2)
    B, h, hu, hv = w.fields(x, y)
    s = P.Solver(m.vx, m.vy, m.etov, B, 2, w.g, params=w.params, vbc=m.vbc)
    s.set_state(h, hu, hv)
    with pytest.raises(P.SweError) as ei:
        s.step(1e-3, 1)
    assert ei.value.code == -4


def test_all_dry_domain():
    """Degenerate case: no water anywhere (h = 0 at every node over a varying bed).  Alg. 2 line 1 makes
    every element dry (h = h0), nothing is non-finite, TVB never runs, and the state, the
    injected mass and the counters agree with the oracle through MRAB steps."""
    w = si.c4_dambreak(N=3, base=10)
    w.initial = lambda x, y: (np.zeros_like(x), np.zeros_like(x), np.zeros_like(x))
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    o, s, _ = run_both(w, 5, dt, nlevels=3)
    io = _counters_equal(o, s)
    assert io["n_dry"] > 0 and io["n_tvb"] == 0
    assert_parity(o, s, w.g)
    h = s.get_state()[0]
    assert np.all(h == w.params["h0"])


def test_mass_conservation_gpu_single_rate():
    w = si.c3_thacker(N=2, n=40)
    o, s, d = make_pair(w)
    s.set_state(d["h"], d["hu"], d["hv"])
    i0 = s.info()
    dt = si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)
    for _ in range(100):
        s.step(dt, 1)
        assert s.info()["min_h"] >= 0.0  # positivity at every node
    i1 = s.info()
    drift = i1["mass"] - i0["mass"] - (i1["injected_mass"] - i0["injected_mass"])
    assert abs(drift) < 1e-13 * i0["mass"]


def test_lake_at_rest_mrab_graded():
    """Well-balancing through the MRAB schedule (dense output of a zero RHS)."""
    w = si.c4_dambreak(N=3, base=5)
    m = w.mesh
    x, y = P.nodes(m.vx, m.vy, m.etov, 3)
    B = w.bathymetry(x, y) - 4.0  # fully wet: eta = 0 everywhere
    s = P.Solver(m.vx, m.vy, m.etov, B, 3, 9.81, params=w.params)
    s.set_state(-B, np.zeros_like(B), np.zeros_like(B))
    dt = si.dt_for(m, 3, 9.81, 4.0, 13.0, 0.2)
    for _ in range(5):
        s.step(dt, 3)
    h, hu, hv = s.get_state()
    assert np.abs(h + B).max() < 1e-12 * 4.0
    assert max(np.abs(hu).max(), np.abs(hv).max()) < 1e-11


def test_schedule_and_state_errors():
    w = si.c1_lake(N=2, n=4)
    m = w.mesh
    x, y = P.nodes(m.vx, m.vy, m.etov, 2)
    B, h, hu, hv = w.fields(x, y)
    s = P.Solver(m.vx, m.vy, m.etov, B, 2, 9.81, params=w.params)
    with pytest.raises(P.SweError) as ei:
        s.step(1e-3, 1)
    assert ei.value.code == -4
    s.set_state(h, hu, hv)
    s.step(1e-3, 2)
    with pytest.raises(P.SweError) as ei:
        s.step(2e-3, 2)
    assert ei.value.code == -5
    with pytest.raises(P.SweError) as ei:
        s.step(-1.0, 2)
    assert ei.value.code == -1
    s.set_state(h, hu, hv)  # resets the schedule
    s.step(2e-3, 1)
    with pytest.raises(P.SweError) as ei:
        P.Solver(m.vx, m.vy, m.etov, np.zeros((m.K, 28)), 6, 9.81)
    assert ei.value.code == -3


def test_single_element_and_nonfinite():
    vx, vy = np.array([0.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0])
    etov = np.array([[0, 2, 1]], dtype=np.int32)  # clockwise: flipped
    x, y = P.nodes(vx, vy, etov, 2)
    s = P.Solver(vx, vy, etov, np.zeros_like(x), 2, 9.81, params={"use_pp": 1, "use_tvb": 1})
    h = 1.0 + 0.1 * x
    s.set_state(h, np.zeros_like(h), np.zeros_like(h))
    for _ in range(10):
        s.step(1e-3, 1)
    assert s.info()["nflipped"] == 1
    h[0, 0] = np.nan
    s.set_state(h, np.zeros_like(h), np.zeros_like(h))
    with pytest.raises(P.SweError) as ei:
        s.step(1e-3, 1)
    assert ei.value.code == -6


def test_ragged_level_ranges_many_levels():
    """nlevels up to 8 with empty levels and ragged (non multiple of 128) ranges."""
    w = si.c4_dambreak(N=2, base=10)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    o, s, _ = run_both(w, 2, dt, nlevels=8)
    assert np.array_equal(o.levels(), s.levels())
    assert_parity(o, s, w.g)


def test_set_state_again_reuses_or_rebuilds_layout():
    """swe_set_state on a live context: a state that bins to the resident levels reuses the internal
    layout (only the state is scattered) and must reproduce a fresh run bit for bit; a state that bins
    to other levels rebuilds the layout and must match the oracle."""
    w = si.c4_dambreak(N=2, base=5)
    m = w.mesh
    o, s, d = make_pair(w)
    dt = si.dt_for(m, w.N, w.g, 1.875, 13.0, 0.2)
    s.set_state(d["h"], d["hu"], d["hv"])
    for _ in range(3):
        s.step(dt, 3)
    first = s.get_state()
    lev1 = s.levels()
    s.set_state(d["h"], d["hu"], d["hv"])  # same state -> same levels -> layout reused
    for _ in range(3):
        s.step(dt, 3)
    again = s.get_state()
    assert np.array_equal(s.levels(), lev1)
    for a, b in zip(first, again):
        assert np.array_equal(a, b)
    # a local jet in the reservoir (speeds above a_floor = 13 m/s) moves elements to finer levels ->
    # layout rebuilt; set_state resets the schedule, so a smaller dt is allowed
    x, y = P.nodes(m.vx, m.vy, m.etov, w.N)
    h2, hu2, hv2 = d["h"], d["hu"] + 20.0 * np.exp(-((x - 8.0) ** 2 + (y - 15.0) ** 2) / 20.0) * d["h"], d["hv"]
    s.set_state(h2, hu2, hv2)
    o.set_state(h2, hu2, hv2)
    for _ in range(3):
        s.step(0.5 * dt, 3)
        assert o.step(0.5 * dt, 3) == 0
    assert np.array_equal(s.levels(), o.levels())
    assert not np.array_equal(s.levels(), lev1)
    assert_parity(o, s, w.g)


def test_parity_couette_annulus():
    """Couette flow on the annulus (readings A27/A28): curved-boundary walls at r = 2, 4."""
    w = si.c6_couette(3, 4, 24)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2, u_max=0.1)
    o, s, _ = run_both(w, 100, dt)
    assert_parity(o, s, w.g)


def test_parity_rarefaction_dry_bed():
    """Rarefaction into a dry bed from the exact state at t = 2 s: PP on, TVB off."""
    w = si.c7_rarefaction(2, 2)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2, u_max=2.0)
    o, s, _ = run_both(w, 100, dt)
    assert_parity(o, s, w.g)
    io, ig = o.info(), s.info()
    assert io["n_pp"] == ig["n_pp"] > 0 and io["n_dry"] == ig["n_dry"]


def test_parity_oscillating_lake():
    """Oscillating lake: moving wet/dry front, PP + TVB, reflecting walls."""
    w = si.c8_oscillating_lake(2, 16)
    dt = si.dt_for(w.mesh, w.N, w.g, 0.2, 0.0, 0.2, u_max=0.5)
    o, s, _ = run_both(w, 100, dt)
    assert_parity(o, s, w.g)
    io, ig = o.info(), s.info()
    assert io["n_pp"] == ig["n_pp"] > 0 and io["n_dry"] == ig["n_dry"] and io["n_tvb"] == ig["n_tvb"]


def test_parity_mrab_printed_order_variant():
    """mrab_coupling = 1: Alg. 1's printed loop order with latest committed
    neighbours, on the C4 wet/dry MRAB case; it differs from the default coupling."""
    w = si.c4_dambreak(N=3, base=5)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    o, s, _ = run_both(w, 8, dt, nlevels=3, mrab_coupling=1)
    assert np.array_equal(o.levels(), s.levels())
    assert_parity(o, s, w.g)
    _, s0, _ = run_both(w, 8, dt, nlevels=3)
    assert max(parity_rel(s.get_state(), s0.get_state(), w.g)) > 1e-10  # far above the 1e-12 parity level


def test_parity_regroup():
    """swe_regroup (NEXT-4): re-binned levels, restarted ramp, continued time; against the
    oracle's regroup, with a new (dt, nlevels) after the regroup."""
    w = si.c4_dambreak(N=3, base=5)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.875, 13.0, 0.2)
    o, s, d = run_both(w, 4, dt, nlevels=3)
    o.regroup()
    s.regroup()
    for _ in range(4):
        assert o.step(0.5 * dt, 2) == 0
        s.step(0.5 * dt, 2)
    assert np.array_equal(o.levels(), s.levels())
    assert_parity(o, s, w.g)
    assert abs(o.info()["t"] - s.info()["t"]) <= 1e-12 * o.info()["t"]


def test_parity_outflow_boundary():
    """Transmissive outflow boundary (reading A7'): the rarefaction started at t = 4.8 s crosses
    x = 30 within the run; PP on."""
    w = si.c7_rarefaction_outflow(2, 4, True, t0=4.8)
    assert w.mesh.vbc is not None and w.mesh.vbc.sum() > 0
    dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2, u_max=2.0)
    o, s, _ = run_both(w, 150, dt)
    assert_parity(o, s, w.g)


def test_parity_outflow_boundary_tensor_path():
    """The N = 4 tensor-path K1 (k_rhs_update_mma2) with a transmissive outflow boundary (A7')."""
    w = si.c7_rarefaction_outflow(4, 2, True, t0=4.8)
    dt = si.dt_for(w.mesh, w.N, w.g, 1.0, 0.0, 0.2, u_max=2.0)
    o, s, _ = run_both(w, 80, dt)
    assert_parity(o, s, w.g)
