"""paper_1403_1661_b200 -- B200-native nodal-DG shallow-water solver (arXiv:1403.1661).

Thin ctypes binding of the C ABI in include/swe.h (argument marshalling only:
every step of the hot path runs in the sm_100a kernels of libswe_b200.so).
PyTorch supplies the device memory (caching allocator) and the stream.
There is no CPU fallback: if the extension is missing the import of
``lib()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWE_LIB", os.path.join(_HERE, "libswe_b200.so"))  # SWE_LIB: A/B variants

SWE_ERRORS = {0: "SWE_OK", -1: "SWE_ERR_ARG", -2: "SWE_ERR_MESH", -3: "SWE_ERR_ORDER", -4: "SWE_ERR_STATE",
              -5: "SWE_ERR_SCHEDULE", -6: "SWE_ERR_NONFINITE", -7: "SWE_ERR_CUDA", -8: "SWE_ERR_NCCL",
              -9: "SWE_ERR_NOMEM"}

EXPORTED = ["swe_nodes", "swe_create", "swe_set_state", "swe_step", "swe_get_state", "swe_regroup", "swe_destroy",
            "swe_get_levels",
            "swe_get_connectivity", "swe_get_info", "swe_last_error", "swe_profile", "swe_profile_read",
            "swe_nccl_unique_id", "swe_link_group", "swe_step_group",
            "swe_host_refel", "swe_host_connectivity", "swe_host_hk", "swe_host_levels", "swe_host_tvb_geometry",
            "swe_host_halo_plan", "swe_get_decisions", "swe_ipc_handle", "swe_ipc_open", "swe_set_boundary_state",
            "swe_get_state_async", "swe_wait_state"]


class SweError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{SWE_ERRORS.get(code, code)}: {msg}")
        self.code = code


class SweMesh(C.Structure):
    _fields_ = [("nverts", C.c_int32), ("vx", C.POINTER(C.c_double)), ("vy", C.POINTER(C.c_double)),
                ("nelems", C.c_int32), ("etov", C.POINTER(C.c_int32)), ("vperiodic", C.POINTER(C.c_int32)),
                ("vbc", C.POINTER(C.c_int8))]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class SweParams(C.Structure):
    _fields_ = [("h0", C.c_double), ("eps", C.c_double), ("tvb_M", C.c_double), ("tvb_nu", C.c_double),
                ("a_floor", C.c_double), ("eps_u", C.c_double), ("h_char", C.c_double),
                ("use_pp", C.c_int32), ("use_tvb", C.c_int32), ("device", C.c_int32), ("stream", C.c_void_p),
                ("dev_alloc", ALLOC_FN), ("dev_free", FREE_FN), ("alloc_user", C.c_void_p),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("owner", C.POINTER(C.c_int32)),
                ("gid", C.POINTER(C.c_int64)), ("nccl_id", C.c_void_p), ("precision", C.c_int32),
                ("mrab_coupling", C.c_int32), ("record_decisions", C.c_int32)]


class SweInfo(C.Structure):
    _fields_ = [("t", C.c_double), ("mass", C.c_double), ("injected_mass", C.c_double), ("min_h", C.c_double),
                ("n_pp", C.c_int64), ("n_dry", C.c_int64), ("n_tvb", C.c_int64), ("n_updates", C.c_int64),
                ("K", C.c_int32), ("Np", C.c_int32), ("N", C.c_int32), ("nlevels", C.c_int32),
                ("nflipped", C.c_int32), ("level_count", C.c_int32 * 8), ("n_posfix", C.c_int64),
                ("n_tvb_cw", C.c_int64)]


_lib = None


def build(force: bool = False) -> str:
    from . import buildlib as _b
    return _b.build(force=force)


def lib():
    """Load libswe_b200.so (fails loudly when it is missing: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run python -m paper_1403_1661_b200.build")
        L = C.CDLL(LIB_PATH)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        vp = C.c_void_p
        L.swe_nodes.argtypes = [C.POINTER(SweMesh), C.c_int, dp, dp]
        L.swe_create.argtypes = [C.POINTER(SweMesh), dp, C.c_int, C.c_double, C.POINTER(SweParams), C.POINTER(vp)]
        L.swe_set_state.argtypes = [vp, dp, dp, dp]
        L.swe_step.argtypes = [vp, C.c_double, C.c_int]
        L.swe_set_boundary_state.argtypes = [vp, dp, dp, dp]
        L.swe_regroup.argtypes = [vp]
        L.swe_get_state.argtypes = [vp, dp, dp, dp]
        L.swe_get_state_async.argtypes = [vp, dp, dp, dp]
        L.swe_wait_state.argtypes = [vp]
        L.swe_destroy.argtypes = [vp]
        L.swe_destroy.restype = None
        L.swe_get_levels.argtypes = [vp, ip]
        L.swe_get_connectivity.argtypes = [vp, ip, C.POINTER(C.c_int8)]
        L.swe_get_info.argtypes = [vp, C.POINTER(SweInfo)]
        L.swe_get_decisions.argtypes = [vp, C.c_void_p, C.POINTER(C.c_int64)]
        L.swe_ipc_handle.argtypes = [vp, C.c_void_p, C.POINTER(C.c_size_t)]
        L.swe_ipc_open.argtypes = [vp, C.c_void_p]
        L.swe_last_error.argtypes = [vp]
        L.swe_last_error.restype = C.c_char_p
        L.swe_profile.argtypes = [vp, C.c_int]
        L.swe_profile_read.argtypes = [vp, dp, C.POINTER(C.c_int64), dp]
        L.swe_host_refel.argtypes = [C.c_int, C.c_char_p, dp, ip, ip]
        L.swe_host_connectivity.argtypes = [C.POINTER(SweMesh), ip, C.POINTER(C.c_int8), ip]
        L.swe_host_hk.argtypes = [C.POINTER(SweMesh), dp]
        L.swe_host_levels.argtypes = [C.POINTER(SweMesh), C.c_int, C.c_double, dp, dp, dp, C.POINTER(SweParams),
                                      C.c_int, ip]
        L.swe_host_tvb_geometry.argtypes = [C.POINTER(SweMesh), ip, dp]
        L.swe_nccl_unique_id.argtypes = [C.c_void_p]
        L.swe_link_group.argtypes = [C.POINTER(vp), C.c_int]
        L.swe_step_group.argtypes = [C.POINTER(vp), C.c_int, C.c_double, C.c_int]
        L.swe_host_halo_plan.argtypes = [C.POINTER(SweMesh), C.POINTER(C.c_int64), ip, C.c_int, ip, ip,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        for n in EXPORTED:
            if n not in ("swe_destroy", "swe_last_error"):
                getattr(L, n).restype = C.c_int
        _lib = L
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


class _MeshArgs:
    """Keeps the numpy buffers of a swe_mesh alive."""

    def __init__(self, vx, vy, etov, vper=None, vbc=None):
        self.vx, self.vy = _d(vx), _d(vy)
        self.etov = np.ascontiguousarray(etov, dtype=np.int32).reshape(-1, 3)
        self.vper = None if vper is None else np.ascontiguousarray(vper, dtype=np.int32)
        self.vbc = None if vbc is None else np.ascontiguousarray(vbc, dtype=np.int8)
        self.K = self.etov.shape[0]
        self.s = SweMesh(len(self.vx), _p(self.vx), _p(self.vy), self.K, _p(self.etov, C.c_int32),
                         _p(self.vper, C.c_int32) if self.vper is not None else C.POINTER(C.c_int32)(),
                         _p(self.vbc, C.c_int8) if self.vbc is not None else C.POINTER(C.c_int8)())


def _check(rc, ctx=None):
    if rc != 0:
        msg = lib().swe_last_error(ctx).decode() if ctx else ""
        raise SweError(rc, msg)


def _params(p: dict | None, device=0, stream=None, alloc=None, part=None) -> SweParams:
    p = dict(p or {})
    sp = SweParams()
    sp.nranks = 1
    if part is not None:
        sp.rank, sp.nranks = int(part["rank"]), int(part["nranks"])
        sp.owner = _p(part["owner"], C.c_int32)
        if part.get("gid") is not None:
            sp.gid = _p(part["gid"], C.c_int64)
        if part.get("nccl_id") is not None:
            sp.nccl_id = C.cast(part["nccl_id"], C.c_void_p)
    for k in ("h0", "eps", "tvb_M", "tvb_nu", "a_floor", "eps_u", "h_char"):
        setattr(sp, k, float(p.get(k, 0.0)))
    sp.use_pp = int(p.get("use_pp", 1))
    sp.use_tvb = int(p.get("use_tvb", 1))
    sp.precision = int(p.get("precision", 64))  # 32: FP32 variant
    sp.mrab_coupling = int(p.get("mrab_coupling", 0))  # 1: Alg. 1 printed order, latest committed (NEXT-4)
    sp.record_decisions = int(p.get("record_decisions", 0))  # decision log for oracle replay
    sp.device = int(device)
    sp.stream = stream
    if alloc is not None:
        sp.dev_alloc, sp.dev_free = alloc
    return sp


def nodes(vx, vy, etov, N, vper=None):
    """Physical node coordinates [K, Np] (x, y) in the library's node order (host only)."""
    m = _MeshArgs(vx, vy, etov, vper)
    Np = (N + 1) * (N + 2) // 2
    x = np.zeros((m.K, Np))
    y = np.zeros((m.K, Np))
    _check(lib().swe_nodes(C.byref(m.s), N, _p(x), _p(y)))
    return x, y


def host_refel(N, name):
    r, c = C.c_int32(), C.c_int32()
    _check(lib().swe_host_refel(N, name.encode(), None, C.byref(r), C.byref(c)))
    out = np.zeros((r.value, c.value))
    _check(lib().swe_host_refel(N, name.encode(), _p(out), C.byref(r), C.byref(c)))
    return out[:, 0] if c.value == 1 else out


def host_connectivity(vx, vy, etov, vper=None):
    m = _MeshArgs(vx, vy, etov, vper)
    e = np.zeros((m.K, 3), dtype=np.int32)
    f = np.zeros((m.K, 3), dtype=np.int8)
    nf = C.c_int32()
    _check(lib().swe_host_connectivity(C.byref(m.s), _p(e, C.c_int32), _p(f, C.c_int8), C.byref(nf)))
    return e, f, nf.value


def host_hk(vx, vy, etov, vper=None):
    m = _MeshArgs(vx, vy, etov, vper)
    hk = np.zeros(m.K)
    _check(lib().swe_host_hk(C.byref(m.s), _p(hk)))
    return hk


def host_levels(vx, vy, etov, N, g, h, hu, hv, nlevels, params=None, vper=None):
    m = _MeshArgs(vx, vy, etov, vper)
    lev = np.zeros(m.K, dtype=np.int32)
    h, hu, hv = _d(h), _d(hu), _d(hv)
    sp = _params(params)
    _check(lib().swe_host_levels(C.byref(m.s), N, float(g), _p(h), _p(hu), _p(hv), C.byref(sp), int(nlevels),
                                 _p(lev, C.c_int32)))
    return lev


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().swe_nccl_unique_id(buf))
    return buf.raw


def host_halo_plan(vx, vy, etov, owner, rank, gid=None, vper=None):
    """Halo plan of `rank` (host only): dict(owned, ghosts, peers=[(rank, nsend, nrecv)], send_gids, recv_gids)."""
    m = _MeshArgs(vx, vy, etov, vper)
    own = np.ascontiguousarray(owner, dtype=np.int32)
    g = None if gid is None else np.ascontiguousarray(gid, dtype=np.int64)
    gp = None if g is None else _p(g, C.c_int64)
    cnt = np.zeros(3, dtype=np.int32)
    _check(lib().swe_host_halo_plan(C.byref(m.s), gp, _p(own, C.c_int32), int(rank), _p(cnt, C.c_int32), None, None,
                                    None))
    peers = np.zeros((max(1, cnt[2]), 3), dtype=np.int32)
    _check(lib().swe_host_halo_plan(C.byref(m.s), gp, _p(own, C.c_int32), int(rank), _p(cnt, C.c_int32),
                                    _p(peers, C.c_int32), None, None))
    ns, nr = int(peers[:cnt[2], 1].sum()), int(peers[:cnt[2], 2].sum())
    sg, rg = np.zeros(max(1, ns), dtype=np.int64), np.zeros(max(1, nr), dtype=np.int64)
    _check(lib().swe_host_halo_plan(C.byref(m.s), gp, _p(own, C.c_int32), int(rank), _p(cnt, C.c_int32),
                                    _p(peers, C.c_int32), _p(sg, C.c_int64), _p(rg, C.c_int64)))
    return {"owned": int(cnt[0]), "ghosts": int(cnt[1]), "peers": [tuple(map(int, r)) for r in peers[:cnt[2]]],
            "send_gids": sg[:ns], "recv_gids": rg[:nr]}


def host_tvb_geometry(vx, vy, etov, vper=None):
    m = _MeshArgs(vx, vy, etov, vper)
    pairs = np.zeros((m.K, 3, 2), dtype=np.int32)
    al = np.zeros((m.K, 3, 2))
    _check(lib().swe_host_tvb_geometry(C.byref(m.s), _p(pairs, C.c_int32), _p(al)))
    return pairs, al


class _TorchAllocator:
    """Device memory from the torch caching allocator (PyTorch is plumbing only)."""

    def __init__(self, device):
        import torch
        self.torch = torch
        self.device = device

        def _alloc(nbytes, stream, user):
            return int(torch.cuda.caching_allocator_alloc(int(nbytes), self.device, stream))

        def _free(ptr, stream, user):
            try:
                torch.cuda.caching_allocator_delete(ptr)
            except Exception:  # interpreter shutdown: the allocator is gone with the process
                pass

        self.alloc = ALLOC_FN(_alloc)
        self.free = FREE_FN(_free)


class Solver:
    """One solver context (swe_create ... swe_destroy)."""

    def __init__(self, vx, vy, etov, B, N, g, vper=None, params: dict | None = None, device: int = 0, vbc=None,
                 use_torch: bool = True, rank: int = 0, nranks: int = 1, owner=None, gid=None, nccl_id=None):
        L = lib()
        self._mesh = _MeshArgs(vx, vy, etov, vper, vbc)
        self.K = self._mesh.K
        self.N = N
        self.Np = (N + 1) * (N + 2) // 2
        self._B = _d(B).reshape(self.K, self.Np)
        stream = None
        self._alloc = None
        if use_torch:
            import torch
            torch.cuda.set_device(device)
            stream = C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
            self._alloc = _TorchAllocator(device)
        self._part = None
        if nranks > 1:
            self._part = {"rank": rank, "nranks": nranks,
                          "owner": np.ascontiguousarray(owner, dtype=np.int32),
                          "gid": None if gid is None else np.ascontiguousarray(gid, dtype=np.int64),
                          "nccl_id": None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)}
        self._sp = _params(params, device, stream,
                           None if self._alloc is None else (self._alloc.alloc, self._alloc.free), self._part)
        h = C.c_void_p()
        rc = L.swe_create(C.byref(self._mesh.s), _p(self._B), N, float(g), C.byref(self._sp), C.byref(h))
        if rc != 0:
            raise SweError(rc, "swe_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().swe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _shape(self, a):
        return _d(a).reshape(self.K, self.Np)

    def set_state(self, h, hu, hv):
        h, hu, hv = self._shape(h), self._shape(hu), self._shape(hv)
        _check(lib().swe_set_state(self._h, _p(h), _p(hu), _p(hv)), self._h)

    def step(self, dt, nlevels=1):
        _check(lib().swe_step(self._h, float(dt), int(nlevels)), self._h)

    def set_boundary_state(self, h, hu, hv):
        """Dirichlet boundary data (include/swe.h, reading A7''): nodal state [K, Np] x 3."""
        h, hu, hv = self._shape(h), self._shape(hu), self._shape(hv)
        _check(lib().swe_set_boundary_state(self._h, _p(h), _p(hu), _p(hv)), self._h)

    def _out(self, a):
        """An output buffer the library may write K*Np doubles into: float64, C-contiguous, K*Np elements."""
        if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous or \
                a.size != self.K * self.Np or not a.flags.writeable:
            raise ValueError(f"output buffer must be a writeable C-contiguous float64 array of {self.K * self.Np} "
                             f"elements")
        return a

    def get_state(self, out=None):
        if out is None:
            out = tuple(np.zeros((self.K, self.Np)) for _ in range(3))
        h, hu, hv = (self._out(a) for a in out)
        _check(lib().swe_get_state(self._h, _p(h), _p(hu), _p(hv)), self._h)
        return h, hu, hv

    def regroup(self):
        """Re-bin the levels from the current state at the next step; time continues."""
        _check(lib().swe_regroup(self._h), self._h)

    def get_state_into(self, h, hu, hv):
        """Write into caller-provided (e.g. pinned) contiguous float64 buffers of K*Np elements."""
        h, hu, hv = self._out(h), self._out(hu), self._out(hv)
        _check(lib().swe_get_state(self._h, _p(h), _p(hu), _p(hv)), self._h)

    def get_state_async(self, h, hu, hv):
        """Enqueue a copy of the current state into h, hu, hv (pinned for overlap) and return at once; the buffers
        hold the state after wait_state().  The solver keeps references to them until then."""
        h, hu, hv = self._out(h), self._out(hu), self._out(hv)
        self._pending = getattr(self, "_pending", []) + [(h, hu, hv)]
        _check(lib().swe_get_state_async(self._h, _p(h), _p(hu), _p(hv)), self._h)

    def wait_state(self):
        _check(lib().swe_wait_state(self._h), self._h)
        self._pending = []

    def levels(self):
        a = np.zeros(self.K, dtype=np.int32)
        _check(lib().swe_get_levels(self._h, _p(a, C.c_int32)), self._h)
        return a

    def connectivity(self):
        e = np.zeros((self.K, 3), dtype=np.int32)
        f = np.zeros((self.K, 3), dtype=np.int8)
        _check(lib().swe_get_connectivity(self._h, _p(e, C.c_int32), _p(f, C.c_int8)), self._h)
        return e, f

    def info(self) -> dict:
        inf = SweInfo()
        _check(lib().swe_get_info(self._h, C.byref(inf)), self._h)
        return {k: (list(getattr(inf, k)) if k == "level_count" else getattr(inf, k)) for k, _ in SweInfo._fields_}

    def ipc_handle(self) -> bytes:
        """This rank's CUDA-IPC exchange-block handle (include/swe.h, swe_ipc_handle)."""
        n = C.c_size_t(0)
        _check(lib().swe_ipc_handle(self._h, None, C.byref(n)), self._h)
        buf = C.create_string_buffer(n.value)
        _check(lib().swe_ipc_handle(self._h, buf, C.byref(n)), self._h)
        return buf.raw[:n.value]

    def ipc_open(self, blobs):
        """Map every rank's exchange block (blobs in rank order) and use the CUDA-IPC transport."""
        raw = b"".join(bytes(b) for b in blobs)
        self._ipc_blobs = C.create_string_buffer(raw, len(raw))
        _check(lib().swe_ipc_open(self._h, self._ipc_blobs), self._h)

    def decisions(self):
        """Limiter decision log (params record_decisions=1): uint8 [nrec, K] (include/swe.h)."""
        n = C.c_int64(0)
        _check(lib().swe_get_decisions(self._h, None, C.byref(n)), self._h)
        out = np.zeros((n.value, self.K), dtype=np.uint8)
        if n.value:
            _check(lib().swe_get_decisions(self._h, out.ctypes.data_as(C.c_void_p), C.byref(n)), self._h)
        return out

    def profile(self, on: bool):
        _check(lib().swe_profile(self._h, int(on)), self._h)

    def profile_read(self):
        t = np.zeros(2)
        n = np.zeros(2, dtype=np.int64)
        b = np.zeros(2)
        _check(lib().swe_profile_read(self._h, _p(t), _p(n, C.c_int64), _p(b)), self._h)
        return {"k1_ms": t[0], "k2_ms": t[1], "k1_launches": int(n[0]), "k2_launches": int(n[1]),
                "k1_bytes": b[0], "k2_bytes": b[1]}


def ipc_connect(solver, group=None):
    """Exchange the CUDA-IPC handles of all ranks over torch.distributed (plumbing only) and open them."""
    import torch.distributed as dist
    blobs = [None] * dist.get_world_size(group)
    dist.all_gather_object(blobs, solver.ipc_handle(), group=group)
    solver.ipc_open(blobs)


def link_group(solvers):
    """Link in-process solvers (ranks 0..n-1 of one partition, same device/stream)."""
    arr = (C.c_void_p * len(solvers))(*[s._h for s in solvers])
    _check(lib().swe_link_group(arr, len(solvers)))
    return arr


def step_group(solvers, dt, nlevels=1):
    arr = (C.c_void_p * len(solvers))(*[s._h for s in solvers])
    rc = lib().swe_step_group(arr, len(solvers), float(dt), int(nlevels))
    _check(rc, solvers[0]._h)
