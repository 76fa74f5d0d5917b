"""CPU oracle for arXiv:1403.1661 -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct C++ implementation of the paper's method
(oracle/*.cpp, every function citing the PAPER.md passage it follows), loaded
through ctypes.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this
package.  It shares no code with the CUDA product path
(``paper_1403_1661_b200``) and never imports it.

Parity status: every oracle function is pinned by a ``-m "not gpu"`` test
against values fixed by the paper or by mathematics (tests/test_oracle_*.py);
the MRAB dense-output coupling is pinned only through the toy-ODE order test
and the nlevels=1 reduction ("parity pins").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_SOURCES = ["refel.cpp", "mesh.cpp", "mrab.cpp", "swe.cpp"]

ORC_FLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c++17"]


def build(force: bool = False) -> str:
    """Compile oracle/liborc.so with g++ (plain -O2, no fast-math, no FMA contraction)."""
    srcs = [os.path.join(_HERE, s) for s in _SOURCES] + [os.path.join(_HERE, "oracle.hpp")]
    if not force and os.path.exists(_LIB_PATH):
        lib_m = os.path.getmtime(_LIB_PATH)
        if all(os.path.getmtime(s) <= lib_m for s in srcs):
            return _LIB_PATH
    cmd = ["g++"] + ORC_FLAGS + [os.path.join(_HERE, s) for s in _SOURCES] + ["-o", _LIB_PATH + ".tmp"]
    subprocess.check_call(cmd)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


class OrcParams(C.Structure):
    _fields_ = [
        ("h0", C.c_double), ("eps", C.c_double), ("tvb_M", C.c_double), ("tvb_nu", C.c_double),
        ("a_floor", C.c_double), ("eps_u", C.c_double), ("h_char", C.c_double),
        ("use_pp", C.c_int), ("use_tvb", C.c_int), ("mrab_coupling", C.c_int),
    ]


class OrcInfo(C.Structure):
    _fields_ = [
        ("t", C.c_double), ("mass", C.c_double), ("injected_mass", C.c_double), ("min_h", C.c_double),
        ("n_pp", C.c_long), ("n_dry", C.c_long), ("n_tvb", C.c_long),
        ("K", C.c_int), ("Np", C.c_int), ("nlevels", C.c_int), ("level_count", C.c_int * 16),
        ("n_posfix", C.c_long), ("n_tvb_cw", C.c_long), ("n_adopted", C.c_long), ("n_mismatch", C.c_long),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_int, dp, dp, C.c_int, ip, ip, dp, C.c_int, C.c_double,
                                 C.POINTER(OrcParams), ip, C.c_char_p, C.c_int]
        for name in ["orc_set_state", "orc_step", "orc_get_state", "orc_get_levels", "orc_bin_levels",
                     "orc_get_connectivity", "orc_get_geometry", "orc_get_tvb_geometry", "orc_nodes",
                     "orc_rhs", "orc_limit", "orc_get_info"]:
            getattr(L, name).restype = C.c_int
        L.orc_set_state.argtypes = [C.c_void_p, dp, dp, dp]
        L.orc_step.argtypes = [C.c_void_p, C.c_double, C.c_int]
        L.orc_get_state.argtypes = [C.c_void_p, dp, dp, dp]
        L.orc_get_levels.argtypes = [C.c_void_p, ip]
        L.orc_bin_levels.argtypes = [C.c_void_p, C.c_int, ip]
        L.orc_get_connectivity.argtypes = [C.c_void_p, ip, C.POINTER(C.c_int8)]
        L.orc_get_geometry.argtypes = [C.c_void_p, dp, dp, ip]
        L.orc_get_tvb_geometry.argtypes = [C.c_void_p, ip, dp]
        L.orc_nodes.argtypes = [C.c_void_p, dp, dp]
        L.orc_rhs.argtypes = [C.c_void_p, dp, dp, dp, dp, dp, dp]
        L.orc_limit.argtypes = [C.c_void_p, dp, dp, dp, ip]
        L.orc_get_info.argtypes = [C.c_void_p, C.POINTER(OrcInfo)]
        L.orc_destroy.restype = None
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_refel_sizes.argtypes = [C.c_int, ip]
        L.orc_refel_get.argtypes = [C.c_int, C.c_char_p, dp]
        L.orc_quad.argtypes = [C.c_int, C.c_int, dp, dp]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_regroup.argtypes = [C.c_void_p]
        L.orc_set_boundary.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_set_replay.argtypes = [C.c_void_p, C.c_void_p, C.c_long]
        L.orc_set_boundary_state.argtypes = [C.c_void_p, dp, dp, dp]
        L.orc_set_boundary_state.restype = C.c_int
        L.orc_set_replay.restype = C.c_int
        L.orc_toy_mrab.argtypes = [C.c_int, dp, ip, dp, C.c_double, C.c_int, C.c_int, dp, dp, dp, C.c_int]
        _lib = L
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def set_threads(n: int = 0) -> int:
    """Set (n > 0) / query the OpenMP thread count of the oracle."""
    return lib().orc_set_threads(int(n))


def refel(N: int) -> dict:
    """Reference-element data of order N (nodes, rules, operators) as numpy arrays."""
    L = lib()
    sz = (C.c_int * 4)()
    if L.orc_refel_sizes(N, sz) != 0:
        raise ValueError("order out of range")
    Np, Nfp, Ncub, Ng = list(sz)
    shapes = {"r": (Np,), "s": (Np,), "rc": (Ncub,), "sc": (Ncub,), "wc": (Ncub,), "tg": (Ng,), "wg": (Ng,),
              "rg": (3 * Ng,), "sg": (3 * Ng,), "wmean": (Np,), "Dr": (Np, Np), "Ds": (Np, Np),
              "Mref": (Np, Np), "Ic": (Ncub, Np), "Ig": (3 * Ng, Np), "P": (Np, Ncub), "Pr": (Np, Ncub),
              "Ps": (Np, Ncub), "Lg": (Np, 3 * Ng)}
    out = {"N": N, "Np": Np, "Nfp": Nfp, "Ncub": Ncub, "Ng": Ng}
    for k, shp in shapes.items():
        a = np.zeros(shp)
        if L.orc_refel_get(N, k.encode(), _p(a)) != 0:
            raise RuntimeError(k)
        out[k] = a
    return out


def quad(which: str, q: int):
    """1D rules: 'gl' Gauss-Legendre, 'gj10' Gauss-Jacobi(1,0), 'lgl' Lobatto points."""
    idx = {"gl": 0, "gj10": 1, "lgl": 2}[which]
    n = q + 1 if which == "lgl" else q
    x = np.zeros(n)
    w = np.zeros(n)
    lib().orc_quad(idx, q, _p(x), _p(w))
    return x, w


def toy_mrab(A, level, y0, dt, L, nsteps, seed0=None, seed1=None, coupling=0):
    A = _d(A)
    K = A.shape[0]
    lev = np.ascontiguousarray(level, dtype=np.int32)
    y0 = _d(y0)
    out = np.zeros(K)
    s0 = _p(_d(seed0)) if seed0 is not None else None
    s1 = _p(_d(seed1)) if seed1 is not None else None
    keep = (seed0, seed1)
    if seed0 is not None:
        s0a, s1a = _d(seed0), _d(seed1)
        s0, s1 = _p(s0a), _p(s1a)
        keep = (s0a, s1a)
    lib().orc_toy_mrab(K, _p(A), _p(lev, C.c_int), _p(y0), float(dt), int(L), int(nsteps), s0, s1, _p(out),
                       int(coupling))
    del keep
    return out


class Oracle:
    """One oracle solver instance (same calls as the C ABI of the product)."""

    def __init__(self, vx, vy, etov, B, N, g, vper=None, h0=1e-6, eps=0.0, tvb_M=0.0, tvb_nu=1.5,
                 a_floor=0.0, eps_u=0.0, h_char=0.0, use_pp=1, use_tvb=1, mrab_coupling=0, vbc=None):
        L = lib()
        self._vx, self._vy = _d(vx), _d(vy)
        self._etov = np.ascontiguousarray(etov, dtype=np.int32).reshape(-1, 3)
        self.K = self._etov.shape[0]
        self.N = N
        self.Np = (N + 1) * (N + 2) // 2
        self._B = _d(B).reshape(self.K, self.Np)
        self._vper = None if vper is None else np.ascontiguousarray(vper, dtype=np.int32)
        prm = OrcParams(h0, eps, tvb_M, tvb_nu, a_floor, eps_u, h_char, use_pp, use_tvb, mrab_coupling)
        err = C.c_int(0)
        msg = C.create_string_buffer(256)
        self._h = L.orc_create(len(self._vx), _p(self._vx), _p(self._vy), self.K, _p(self._etov, C.c_int),
                               None if self._vper is None else _p(self._vper, C.c_int), _p(self._B), N, float(g),
                               C.byref(prm), C.byref(err), msg, 256)
        if not self._h:
            raise ValueError(f"orc_create failed ({err.value}): {msg.value.decode()}")
        if vbc is not None:  # vertex boundary tags: 1 = transmissive outflow (reading A7')
            self._vbc = np.ascontiguousarray(vbc, dtype=np.int8)
            L.orc_set_boundary(self._h, self._vbc.ctypes.data_as(C.c_void_p))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    def _shape(self, a):
        return _d(a).reshape(self.K, self.Np)

    def set_state(self, h, hu, hv):
        h, hu, hv = self._shape(h), self._shape(hu), self._shape(hv)
        rc = lib().orc_set_state(self._h, _p(h), _p(hu), _p(hv))
        if rc:
            raise RuntimeError(f"orc_set_state failed ({rc})")

    def set_boundary_state(self, h, hu, hv):
        """Dirichlet boundary data (reading A7''): nodal state whose trace is the ghost on faces whose
        vertices are both tagged 2 (vbc); its cell mean is their TVB ghost mean."""
        h, hu, hv = self._shape(h), self._shape(hu), self._shape(hv)
        lib().orc_set_boundary_state(self._h, _p(h), _p(hu), _p(hv))

    def set_replay(self, log):
        """Decision replay: `log` = uint8 [nrec, K] limiter decisions of the product path
        (one record per limiter application, caller element order).  Takes effect from the next
        set_state; where this oracle's own decision lies within 1e-9 (relative) of its threshold it
        adopts the logged one (info()['n_adopted']), larger disagreements count in info()['n_mismatch']."""
        self._replay = np.ascontiguousarray(log, dtype=np.uint8).reshape(-1, self.K)
        lib().orc_set_replay(self._h, self._replay.ctypes.data_as(C.c_void_p), self._replay.shape[0])

    def step(self, dt, nlevels=1):
        return lib().orc_step(self._h, float(dt), int(nlevels))

    def regroup(self):
        """Re-bin the levels from the current state at the next step; time continues."""
        rc = lib().orc_regroup(self._h)
        if rc != 0:
            raise RuntimeError(f"orc_regroup failed ({rc})")

    def get_state(self):
        h, hu, hv = (np.zeros((self.K, self.Np)) for _ in range(3))
        rc = lib().orc_get_state(self._h, _p(h), _p(hu), _p(hv))
        if rc:
            raise RuntimeError(rc)
        return h, hu, hv

    def levels(self):
        a = np.zeros(self.K, dtype=np.int32)
        if lib().orc_get_levels(self._h, _p(a, C.c_int)):
            raise RuntimeError("not scheduled")
        return a

    def bin_levels(self, nlevels):
        a = np.zeros(self.K, dtype=np.int32)
        lib().orc_bin_levels(self._h, int(nlevels), _p(a, C.c_int))
        return a

    def connectivity(self):
        e = np.zeros((self.K, 3), dtype=np.int32)
        f = np.zeros((self.K, 3), dtype=np.int8)
        lib().orc_get_connectivity(self._h, _p(e, C.c_int), _p(f, C.c_int8))
        return e, f

    def geometry(self):
        J = np.zeros(self.K)
        Hk = np.zeros(self.K)
        nf = C.c_int(0)
        lib().orc_get_geometry(self._h, _p(J), _p(Hk), C.byref(nf))
        return J, Hk, nf.value

    def tvb_geometry(self):
        pairs = np.zeros((self.K, 3, 2), dtype=np.int32)
        al = np.zeros((self.K, 3, 2))
        lib().orc_get_tvb_geometry(self._h, _p(pairs, C.c_int), _p(al))
        return pairs, al

    def nodes(self):
        x = np.zeros((self.K, self.Np))
        y = np.zeros((self.K, self.Np))
        lib().orc_nodes(self._h, _p(x), _p(y))
        return x, y

    def rhs(self, h, hu, hv):
        h, hu, hv = self._shape(h), self._shape(hu), self._shape(hv)
        R = [np.zeros((self.K, self.Np)) for _ in range(3)]
        lib().orc_rhs(self._h, _p(h), _p(hu), _p(hv), _p(R[0]), _p(R[1]), _p(R[2]))
        return R

    def limit(self, h, hu, hv):
        h, hu, hv = (self._shape(a).copy() for a in (h, hu, hv))
        dry = np.zeros(self.K, dtype=np.int32)
        rc = lib().orc_limit(self._h, _p(h), _p(hu), _p(hv), _p(dry, C.c_int))
        if rc:
            raise RuntimeError(rc)
        return h, hu, hv, dry

    def info(self):
        inf = OrcInfo()
        lib().orc_get_info(self._h, C.byref(inf))
        return {"t": inf.t, "mass": inf.mass, "injected_mass": inf.injected_mass, "min_h": inf.min_h,
                "n_pp": inf.n_pp, "n_dry": inf.n_dry, "n_tvb": inf.n_tvb, "K": inf.K, "Np": inf.Np,
                "nlevels": inf.nlevels, "level_count": list(inf.level_count),
                "n_posfix": inf.n_posfix, "n_tvb_cw": inf.n_tvb_cw,
                "n_adopted": inf.n_adopted, "n_mismatch": inf.n_mismatch}


# ---------------------------------------------------------------- small pure functions (pins)
def _setup_pure(L):
    if getattr(L, "_pure_ready", False):
        return
    dp = C.POINTER(C.c_double)
    L.orc_vel.restype = C.c_double
    L.orc_vel.argtypes = [C.c_double, C.c_double, C.c_double]
    L.orc_flux.restype = None
    L.orc_flux.argtypes = [C.c_double, C.c_double, dp, C.c_double, dp, C.c_double, C.c_double, C.c_double, dp]
    L.orc_mbar.restype = C.c_int
    L.orc_mbar.argtypes = [C.c_double, C.c_double, C.c_double, dp]
    L.orc_rebalance.argtypes = [dp, dp]
    L.orc_posfix.argtypes = [dp, C.c_double, C.c_double, dp]
    L.orc_posfix.restype = C.c_int
    L.orc_char.argtypes = [C.c_double] * 6 + [dp, dp]
    L._pure_ready = True


def vel(h, m, eps_u=1e-8):
    L = lib()
    _setup_pure(L)
    return L.orc_vel(float(h), float(m), float(eps_u))


def flux(qm, bm, qp, bp, n, g=9.81, eps_u=1e-8):
    """Own-side well-balanced LLF flux (incl. the split-source boundary term) at one point."""
    L = lib()
    _setup_pure(L)
    a, b, out = _d(qm), _d(qp), np.zeros(3)
    L.orc_flux(float(g), float(eps_u), _p(a), float(bm), _p(b), float(bp), float(n[0]), float(n[1]), _p(out))
    return out


def mbar(a, b, thr):
    L = lib()
    _setup_pure(L)
    o = C.c_double()
    first = L.orc_mbar(float(a), float(b), float(thr), C.byref(o))
    return o.value, bool(first)


def rebalance(D):
    L = lib()
    _setup_pure(L)
    a, o = _d(D), np.zeros(3)
    L.orc_rebalance(_p(a), _p(o))
    return o


def posfix(D, hbar, h0):
    L = lib()
    _setup_pure(L)
    a, o = _d(D), np.zeros(3)
    L.orc_posfix(_p(a), float(hbar), float(h0), _p(o))
    return o


def char_matrices(g, h, u, v, nx, ny):
    L = lib()
    _setup_pure(L)
    Lm, Rm = np.zeros((3, 3)), np.zeros((3, 3))
    L.orc_char(float(g), float(h), float(u), float(v), float(nx), float(ny), _p(Lm), _p(Rm))
    return Lm, Rm
