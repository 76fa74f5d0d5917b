"""Seeded synthetic inputs shared by the oracle and the product path.

This module holds NONE of the method's arithmetic: it builds triangulations
(structured, periodic, newest-vertex-bisection graded) and evaluates the
closed-form bathymetries / initial states of the paper's workloads at node
coordinates supplied by the caller (the oracle's ``nodes()`` in the parity
tests, the library's ``swe_nodes`` in bench.py).  Recipes: SURVEY.md §8(d)
"Configs as concrete synthetic inputs" and DESIGN.md "Input recipe".
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

SEED = 14031661
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libmeshgen.so")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "meshgen.cpp")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-fPIC", "-shared", "-std=c++17", src, "-o", _LIB + ".tmp"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_mg = None


def _lib():
    global _mg
    if _mg is None:
        build()
        L = C.CDLL(_LIB)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.mg_nvb.restype = C.c_void_p
        L.mg_nvb.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, dp, dp, ip]
        L.mg_sizes.argtypes = [C.c_void_p, ip, ip]
        L.mg_copy.argtypes = [C.c_void_p, dp, dp, ip, ip]
        L.mg_free.argtypes = [C.c_void_p]
        _mg = L
    return _mg


# ------------------------------------------------------------------ meshes
@dataclass
class Mesh:
    vx: np.ndarray
    vy: np.ndarray
    etov: np.ndarray            # (K, 3) int32
    vper: np.ndarray | None = None   # canonical vertex ids for periodic face matching
    gen: np.ndarray | None = None    # NVB generation per element (graded meshes)
    vbc: np.ndarray | None = None    # vertex boundary tags: 1 = transmissive outflow (reading A7')

    @property
    def K(self) -> int:
        return int(self.etov.shape[0])


def structured(nx, ny, x0, x1, y0, y1, periodic=False) -> Mesh:
    """nx*ny squares, each split SW->NE into two counter-clockwise triangles."""
    xs = x0 + (x1 - x0) / nx * np.arange(nx + 1)
    ys = y0 + (y1 - y0) / ny * np.arange(ny + 1)
    X, Y = np.meshgrid(xs, ys)
    vx, vy = X.ravel().copy(), Y.ravel().copy()
    vid = lambda i, j: j * (nx + 1) + i  # noqa: E731
    i, j = np.meshgrid(np.arange(nx), np.arange(ny))
    i, j = i.ravel(), j.ravel()
    v00, v10, v01, v11 = vid(i, j), vid(i + 1, j), vid(i, j + 1), vid(i + 1, j + 1)
    lower = np.stack([v10, v11, v00], 1)
    upper = np.stack([v01, v00, v11], 1)
    etov = np.empty((2 * nx * ny, 3), dtype=np.int32)
    etov[0::2] = lower
    etov[1::2] = upper
    vper = None
    if periodic:
        I, J = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1))
        vper = (np.mod(J, ny) * (nx + 1) + np.mod(I, nx)).ravel().astype(np.int32)
    return Mesh(vx, vy, etov, vper)


def nvb_graded(nx, ny, x0, x1, y0, y1, bands) -> Mesh:
    """Structured base refined by newest-vertex bisection; bands = [(x_lo, x_hi, depth), ...]."""
    L = _lib()
    lo = np.array([b[0] for b in bands], dtype=np.float64)
    hi = np.array([b[1] for b in bands], dtype=np.float64)
    dp = np.array([b[2] for b in bands], dtype=np.int32)
    h = L.mg_nvb(nx, ny, x0, x1, y0, y1, len(bands), lo.ctypes.data_as(C.POINTER(C.c_double)),
                 hi.ctypes.data_as(C.POINTER(C.c_double)), dp.ctypes.data_as(C.POINTER(C.c_int)))
    nv, ne = C.c_int(), C.c_int()
    L.mg_sizes(h, C.byref(nv), C.byref(ne))
    vx = np.zeros(nv.value)
    vy = np.zeros(nv.value)
    etov = np.zeros((ne.value, 3), dtype=np.int32)
    gen = np.zeros(ne.value, dtype=np.int32)
    L.mg_copy(h, vx.ctypes.data_as(C.POINTER(C.c_double)), vy.ctypes.data_as(C.POINTER(C.c_double)),
              etov.ctypes.data_as(C.POINTER(C.c_int)), gen.ctypes.data_as(C.POINTER(C.c_int)))
    L.mg_free(h)
    return Mesh(vx, vy, etov, None, gen)


def shuffle(mesh: Mesh, seed: int = SEED, rotate: bool = True, flip_fraction: float = 0.0) -> Mesh:
    """Permute element order (PCG64), cyclically rotate vertex lists, optionally
    reverse a fraction of elements to clockwise (exercises the orientation fix)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    perm = rng.permutation(mesh.K)
    etov = mesh.etov[perm].copy()
    if rotate:
        rot = rng.integers(0, 3, size=mesh.K)
        idx = (np.arange(3)[None, :] + rot[:, None]) % 3
        etov = np.take_along_axis(etov, idx, axis=1)
    if flip_fraction > 0:
        flip = rng.random(mesh.K) < flip_fraction
        etov[flip] = etov[flip][:, [0, 2, 1]]
    gen = None if mesh.gen is None else mesh.gen[perm]
    return Mesh(mesh.vx, mesh.vy, np.ascontiguousarray(etov, dtype=np.int32), mesh.vper, gen, mesh.vbc)


# ------------------------------------------------------------------ workloads
@dataclass
class Workload:
    """One synthetic workload: mesh, closed-form B and initial state, parameters."""
    name: str
    mesh: Mesh
    N: int
    g: float
    bathymetry: object              # B(x, y)
    initial: object                 # (x, y) -> (h, hu, hv)
    params: dict = field(default_factory=dict)
    nlevels: int = 1
    dt_factor: float = 0.2          # dt = dt_factor * r_min / (N+1)^2 (reading A22)
    steps: int = 100
    exact: object = None            # (x, y, t) -> (h, hu, hv), when the paper gives one

    def fields(self, x, y):
        B = self.bathymetry(x, y)
        h, hu, hv = self.initial(x, y)
        return np.ascontiguousarray(B), np.ascontiguousarray(h), np.ascontiguousarray(hu), np.ascontiguousarray(hv)


def dt_for(mesh: Mesh, N: int, g: float, h_max: float, a_floor: float, factor: float, u_max: float = 0.0) -> float:
    """dt = factor * min_k Hk / a / (N+1)^2 with a = max(a_floor, u_max + sqrt(g h_max)) (reading A22).
    Uses an upper bound of the wave speed over the domain, so it never depends on the solver."""
    v = mesh.etov
    x = mesh.vx[v]
    y = mesh.vy[v]
    A = 0.5 * np.abs((x[:, 1] - x[:, 0]) * (y[:, 2] - y[:, 0]) - (x[:, 2] - x[:, 0]) * (y[:, 1] - y[:, 0]))
    per = sum(np.hypot(x[:, (f + 1) % 3] - x[:, f], y[:, (f + 1) % 3] - y[:, f]) for f in range(3))
    Hk = 4 * A / per
    a = max(a_floor, u_max + math.sqrt(g * h_max))
    return factor * float(Hk.min()) / a / (N + 1) ** 2


def c1_lake(N: int = 2, n: int = 16, hump: bool = False, shuffle_seed: int | None = SEED) -> Workload:
    """C1: lake at rest over a Gaussian bump on [0,1]^2, walls."""
    m = structured(n, n, 0.0, 1.0, 0.0, 1.0)
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed, flip_fraction=0.1)

    def B(x, y):
        return -1.0 + 0.2 * np.exp(-((x - 0.5) ** 2 + (y - 0.5) ** 2) / (2 * 0.1 ** 2))

    def init(x, y):
        eta = np.zeros_like(x)
        if hump:
            eta = 0.01 * np.exp(-((x - 0.3) ** 2 + (y - 0.6) ** 2) / (2 * 0.05 ** 2))
        return eta - B(x, y), np.zeros_like(x), np.zeros_like(x)

    prm = dict(h0=1e-8, tvb_M=50.0, tvb_nu=1.5, use_pp=1, use_tvb=1)
    return Workload("C1b" if hump else "C1a", m, N, 9.81, B, init, prm, 1, 0.2, 100)


def vortex_exact(beta=5.0, x0=0.0, y0=0.0):
    """Translating isentropic vortex, g = 2."""
    def ex(x, y, t):
        r2 = (x - t - x0) ** 2 + (y - y0) ** 2
        e = np.exp(1.0 - r2)
        h = 1.0 - beta ** 2 / (32 * math.pi ** 2) * e ** 2
        u = 1.0 - beta * e * (y - y0) / (2 * math.pi)
        v = beta * e * (x - t - x0) / (2 * math.pi)
        return h, h * u, h * v
    return ex


def c2_vortex(N: int, n: int, shuffle_seed: int | None = SEED) -> Workload:
    """C2: translating vortex on the periodic square [-10,10]^2, 2 n^2 triangles, no limiters."""
    m = structured(n, n, -10.0, 10.0, -10.0, 10.0, periodic=True)
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)
    ex = vortex_exact()
    prm = dict(h0=1e-8, use_pp=0, use_tvb=0)
    return Workload(f"C2-n{n}", m, N, 2.0, lambda x, y: np.zeros_like(x), lambda x, y: ex(x, y, 0.0), prm, 1,
                    0.1, 0, ex)


def c2_vortex_dirichlet(N: int, n: int, shuffle_seed: int | None = SEED) -> Workload:
    """The translating vortex in the rectangle [-5, 10] x [-6, 6] with Dirichlet boundaries set to the
    exact solution (reading A7''): every boundary vertex tagged 2.  2 x (5 n / 4) x n triangles
    (n divisible by 4), no limiters."""
    m = structured(5 * n // 4, n, -5.0, 10.0, -6.0, 6.0)
    on_bnd = (np.abs(m.vx + 5.0) < 1e-12) | (np.abs(m.vx - 10.0) < 1e-12) | (np.abs(np.abs(m.vy) - 6.0) < 1e-12)
    m.vbc = np.where(on_bnd, 2, 0).astype(np.int8)
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)
    ex = vortex_exact()
    prm = dict(h0=1e-8, use_pp=0, use_tvb=0)
    return Workload(f"C2D-n{n}", m, N, 2.0, lambda x, y: np.zeros_like(x), lambda x, y: ex(x, y, 0.0), prm, 1,
                    0.1, 0, ex)


def c2_vortex_graded(N: int, n: int, a: float = 0.6, shuffle_seed: int | None = SEED) -> Workload:
    """The C2 vortex on a periodic mesh with graded spacing: the vertices of the 2 n^2 periodic square are
    moved by x -> x + a (L / 2 pi) sin(2 pi (x + 10) / L) (and likewise y), L = 20, which keeps x = +-10
    fixed (periodic partners still coincide) and makes the spacing vary by (1 + a) / (1 - a) (4x at
    a = 0.6): three MRAB levels binned from the element sizes (reading A19) on a periodic domain."""
    m = structured(n, n, -10.0, 10.0, -10.0, 10.0, periodic=True)
    L = 20.0
    m.vx = m.vx + a * L / (2 * math.pi) * np.sin(2 * math.pi * (m.vx + 10.0) / L)
    m.vy = m.vy + a * L / (2 * math.pi) * np.sin(2 * math.pi * (m.vy + 10.0) / L)
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)
    ex = vortex_exact()
    prm = dict(h0=1e-8, use_pp=0, use_tvb=0)
    return Workload(f"C2G-n{n}", m, N, 2.0, lambda x, y: np.zeros_like(x), lambda x, y: ex(x, y, 0.0), prm, 1,
                    0.1, 0, ex)


THACKER = dict(alpha=1.6e-7, X=1.0, Y=-0.41884, g=9.81)


def thacker_exact(alpha=THACKER["alpha"], X=THACKER["X"], Y=THACKER["Y"], g=THACKER["g"]):
    """Parabolic bowl: B = alpha r^2, omega^2 = 8 g alpha."""
    om = math.sqrt(8 * g * alpha)

    def ex(x, y, t):
        r2 = x * x + y * y
        d = X + Y * math.cos(om * t)
        h = np.maximum(0.0, 1.0 / d + alpha * (Y * Y - X * X) * r2 / (d * d))
        f = -Y * om * math.sin(om * t) / d * 0.5
        return h, h * f * x, h * f * y
    return ex, om


def c3_thacker(N: int = 2, n: int = 100, shuffle_seed: int | None = SEED) -> Workload:
    """C3: Thacker parabolic bowl on [-4000,4000]^2, walls, PP + TVB."""
    m = structured(n, n, -4000.0, 4000.0, -4000.0, 4000.0)
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)
    ex, om = thacker_exact()
    al = THACKER["alpha"]
    prm = dict(h0=1e-6, tvb_M=1e-5, tvb_nu=1.5, use_pp=1, use_tvb=1)
    return Workload("C3", m, N, THACKER["g"], lambda x, y: al * (x * x + y * y), lambda x, y: ex(x, y, 0.0), prm,
                    1, 0.2, 100, ex)


def c4_dambreak(N: int = 3, base: int = 1, shuffle_seed: int | None = SEED) -> Workload:
    """C4: dam break over three humps, NVB-graded mesh, 3 MRAB levels.
    base=1 is the full 0.5 m base mesh (2*150*60 before refinement); base=k coarsens it k times."""
    nx, ny = 150 // base, 60 // base
    m = nvb_graded(nx, ny, 0.0, 75.0, 0.0, 30.0, [(6.0, 12.0, 2), (56.0, 64.0, 2), (12.0, 56.0, 4)])
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)

    def B(x, y):
        b1 = 1.0 - 0.125 * np.sqrt((x - 30.0) ** 2 + (y - 6.0) ** 2)
        b2 = 1.0 - 0.125 * np.sqrt((x - 30.0) ** 2 + (y - 24.0) ** 2)
        b3 = 3.0 - 0.3 * np.sqrt((x - 47.5) ** 2 + (y - 15.0) ** 2)
        return np.maximum(0.0, np.maximum(np.maximum(b1, b2), b3))

    def init(x, y):
        h = np.where(x < 16.0, np.maximum(0.0, 1.875 - B(x, y)), 0.0)
        return h, np.zeros_like(x), np.zeros_like(x)

    prm = dict(h0=1e-4, tvb_M=5.0, tvb_nu=1.5, a_floor=13.0, use_pp=1, use_tvb=1)
    return Workload("C4", m, N, 9.81, B, init, prm, 3, 0.2, 100)


def annulus(nr: int, nth: int, r0: float, r1: float) -> Mesh:
    """Polar grid of the annulus r0 <= r <= r1 (nr rings, nth sectors), each cell split into two
    counter-clockwise triangles; the seam at theta = 0 closes through shared vertices."""
    rs = r0 + (r1 - r0) / nr * np.arange(nr + 1)
    th = 2.0 * math.pi / nth * np.arange(nth)
    R, TH = np.meshgrid(rs, th, indexing="ij")  # vertex (i, j) -> i * nth + j
    vx, vy = (R * np.cos(TH)).ravel().copy(), (R * np.sin(TH)).ravel().copy()
    vid = lambda i, j: i * nth + (j % nth)  # noqa: E731
    i, j = np.meshgrid(np.arange(nr), np.arange(nth), indexing="ij")
    i, j = i.ravel(), j.ravel()
    a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
    etov = np.empty((2 * nr * nth, 3), dtype=np.int32)
    etov[0::2] = np.stack([a, b, c], 1)  # (r, th) -> (r+, th) -> (r+, th+): counter-clockwise
    etov[1::2] = np.stack([a, c, d], 1)
    return Mesh(vx, vy, etov, None)


COUETTE = dict(r0=2.0, r1=4.0, g=1.0)


def couette_exact():
    """Couette flow between concentric cylinders: h = 1, u_theta = (-r + 16/r)/75,
    B = (r^2/2 - 32 log r - 128/r^2)/75^2; steady.  g = 1 (reading A27: forced by the balance
    u_theta^2 / r = g dB/dr); annulus 2 <= r <= 4 (reading A28)."""
    def B(x, y):
        r2 = x * x + y * y
        return (0.5 * r2 - 16.0 * np.log(r2) - 128.0 / r2) / 75.0 ** 2

    def ex(x, y, t):
        r = np.sqrt(x * x + y * y)
        ut = (-r + 16.0 / r) / 75.0
        h = np.ones_like(x)
        return h, -h * ut * y / r, h * ut * x / r
    return B, ex


def c6_couette(N: int = 2, nr: int = 4, nth: int = 24, shuffle_seed: int | None = SEED) -> Workload:
    """Couette flow on the annulus 2 <= r <= 4 (walls = the two cylinders, straight-sided),
    smooth steady state, no limiters."""
    m = annulus(nr, nth, COUETTE["r0"], COUETTE["r1"])
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)
    B, ex = couette_exact()
    prm = dict(h0=1e-8, use_pp=0, use_tvb=0)
    return Workload(f"Couette-{nr}x{nth}", m, N, COUETTE["g"], B, lambda x, y: ex(x, y, 0.0), prm, 1, 0.2, 0, ex)


def rarefaction_exact(h0: float = 1.0, g: float = 1.0, x0: float = 20.0):
    """Dam break into a dry bed: xi = (x - 20)/t; h = h0 left of -sqrt(g h0),
    0 right of 2 sqrt(g h0), (xi - 2 sqrt(g h0))^2 / (9 g) between; u = 2/3 (xi + sqrt(g h0))."""
    c0 = math.sqrt(g * h0)

    def ex(x, y, t):
        xi = (x - x0) / t
        h = np.where(xi < -c0, h0, np.where(xi > 2 * c0, 0.0, (xi - 2 * c0) ** 2 / (9 * g)))
        u = np.where(xi < -c0, 0.0, np.where(xi > 2 * c0, 0.0, 2.0 / 3.0 * (xi + c0)))
        return h, h * u, np.zeros_like(x)
    return ex


def c7_rarefaction(N: int = 2, n: int = 1, t0: float = 2.0, shuffle_seed: int | None = SEED) -> Workload:
    """Rarefaction wave on the flat 50 m x 40 m box, g = 1, h0 = 1: initial state =
    the exact solution at t0 = 2 s (C0); PP limiter on, TVB off.  Walls: the wave stays
    inside x in [20 - t, 20 + 2t] for t <= 15.  Mesh: 2 x (10 n) x (8 n) triangles (H = 5/n)."""
    m = structured(10 * n, 8 * n, 0.0, 50.0, 0.0, 40.0)
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)
    ex = rarefaction_exact()
    prm = dict(h0=1e-6, use_pp=1, use_tvb=0)
    w = Workload(f"Rarefaction-n{n}", m, N, 1.0, lambda x, y: np.zeros_like(x), lambda x, y: ex(x, y, t0), prm,
                 1, 0.2, 0, ex)
    w.t0 = t0
    return w


def c7_rarefaction_outflow(N: int = 2, n: int = 2, outflow: bool = True, t0: float = 2.0,
                           shuffle_seed: int | None = SEED) -> Workload:
    """The rarefaction on the short box [0, 30] x [0, 8] whose right side x = 30 is a
    transmissive outflow boundary (reading A7'; outflow=False: a wall): the dry front leaves the
    domain at t = 5 s and the fan keeps matching the exact solution.  2 x (6 n) x (2 n) triangles."""
    m = structured(6 * n, 2 * n, 0.0, 30.0, 0.0, 8.0)
    if outflow:
        m.vbc = (np.abs(m.vx - 30.0) < 1e-12).astype(np.int8)
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)
    ex = rarefaction_exact()
    prm = dict(h0=1e-6, use_pp=1, use_tvb=0)
    w = Workload(f"RarefactionOut-n{n}-{'out' if outflow else 'wall'}", m, N, 1.0, lambda x, y: np.zeros_like(x),
                 lambda x, y: ex(x, y, t0), prm, 1, 0.2, 0, ex)
    w.t0 = t0
    return w


LAKE = dict(a=1.0, sigma=0.5, h0=0.1, g=9.81)


def lake_exact(a=LAKE["a"], sigma=LAKE["sigma"], h0=LAKE["h0"], g=LAKE["g"]):
    """Oscillating lake in a parabolic bowl (Eq. lake2d): B = h0 (x^2+y^2)/a^2,
    h = max(0, sigma h0/a^2 (2x cos wt + 2y sin wt - sigma) + h0 - B), u = -sigma w sin wt,
    v = sigma w cos wt, w = sqrt(2 g h0)/a."""
    om = math.sqrt(2 * g * h0) / a

    def B(x, y):
        return h0 * (x * x + y * y) / a ** 2

    def ex(x, y, t):
        h = np.maximum(0.0, sigma * h0 / a ** 2 * (2 * x * math.cos(om * t) + 2 * y * math.sin(om * t) - sigma)
                       + h0 - B(x, y))
        return h, h * (-sigma * om * math.sin(om * t)), h * (sigma * om * math.cos(om * t))
    return B, ex, om


def c8_oscillating_lake(N: int = 2, n: int = 16, shuffle_seed: int | None = SEED) -> Workload:
    """Oscillating lake on [-2,2]^2 with reflecting walls, PP + TVB.  H = 4/n."""
    m = structured(n, n, -2.0, 2.0, -2.0, 2.0)
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)
    B, ex, om = lake_exact()
    prm = dict(h0=1e-6, tvb_M=1.0, tvb_nu=1.5, use_pp=1, use_tvb=1)
    w = Workload(f"OscLake-n{n}", m, N, LAKE["g"], B, lambda x, y: ex(x, y, 0.0), prm, 1, 0.2, 0, ex)
    w.period = 2 * math.pi / om
    return w


C5_LX = 2.0e6


def c5_tsunami(P: int = 1, base_n: int = 1280, strip: int = 1, shuffle_seed: int | None = SEED,
               rows: tuple | None = None) -> Workload:
    """C5: synthetic ocean-basin tsunami, N=3, 4 MRAB levels.

    Domain [0, 2000 km] x [0, W], W = 2000 km * P / strip.  Base spacing 2000 km / base_n
    (1562.5 m at base_n = 1280, dyadic), NVB-refined by distance d = 2000 km - x to the coast:
    2 bisections for d < 400 km, 4 for d < 60 km, 6 for d < 8 km.  strip > 1 keeps a 1/strip
    y-strip of the same mesh (bounded CPU-oracle sample)."""
    ny = base_n * P // strip
    hb = C5_LX / base_n
    j0, j1 = (0, ny) if rows is None else (max(0, rows[0]), min(ny, rows[1]))
    m = nvb_graded(base_n, j1 - j0, 0.0, C5_LX, j0 * hb, j1 * hb,
                   [(C5_LX - 400e3, C5_LX + 1, 2), (C5_LX - 60e3, C5_LX + 1, 4), (C5_LX - 8e3, C5_LX + 1, 6)])
    if shuffle_seed is not None:
        m = shuffle(m, shuffle_seed)

    def B(x, y):
        b = np.where(x <= 1800e3, -4000.0,
                     np.where(x <= 1950e3, -4000.0 + (x - 1800e3) / 150e3 * 3800.0,
                              np.where(x <= 1995e3, -200.0 + (x - 1950e3) / 45e3 * 190.0,
                                       -10.0 + (x - 1995e3) / 5e3 * 50.0)))
        b = b + 500.0 * np.exp(-((x - 1200e3) ** 2 + (y - 1000e3) ** 2) / (2 * (50e3) ** 2))
        return b

    def init(x, y):
        eta = 1.0 * np.exp(-((x - 1000e3) ** 2 + (y - 1000e3) ** 2) / (2 * (80e3) ** 2))
        return np.maximum(0.0, eta - B(x, y)), np.zeros_like(x), np.zeros_like(x)

    # a_floor = 200 m/s >= sqrt(g * 4001 m): levels are purely geometric (reading A19/C5)
    prm = dict(h0=1e-3, tvb_M=1e-3, tvb_nu=1.5, a_floor=200.0, use_pp=1, use_tvb=1)
    return Workload(f"C5-P{P}" + (f"-strip{strip}" if strip > 1 else ""), m, 3, 9.81, B, init, prm, 4, 0.2, 20)


def centroid_keys(mesh: Mesh, h: float) -> np.ndarray:
    """Global element ids from exact centroid keys (dyadic vertex coordinates: 3*centroid is a
    multiple of h/64 for up to 6 NVB bisections of an h-spaced base grid)."""
    v = mesh.etov
    ix = np.round(mesh.vx[v].sum(1) * 64.0 / h).astype(np.int64)
    iy = np.round(mesh.vy[v].sum(1) * 64.0 / h).astype(np.int64)
    return (ix << 32) | iy


def c5_rank_strip(rank: int, nranks: int, base_n: int = 1280):
    """Rank `rank`'s share of the weak-scaling C5 basin ([0, 2000 km] x [0, 2000 km * nranks]):
    its own 2000 km y-strip plus two buffer rows on each side (ghost layer + refinement buffer);
    owner by centroid y, gid by exact centroid key."""
    hb = C5_LX / base_n
    w = c5_tsunami(P=nranks, base_n=base_n, rows=(rank * base_n - 2, (rank + 1) * base_n + 2), shuffle_seed=None)
    v = w.mesh.etov
    cy = w.mesh.vy[v].mean(1)
    owner = np.clip(np.floor(cy / C5_LX).astype(np.int32), 0, nranks - 1)
    return w, owner, centroid_keys(w.mesh, hb)
