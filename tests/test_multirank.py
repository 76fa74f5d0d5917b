"""Multi-rank (element partition) tests.

-m 'not gpu': the host halo plan of each rank, exchanged between two real
processes over torch.distributed (gloo, world_size 2): rank r's send list to q
must equal q's receive list from r, also when each rank passes only its own
sub-mesh (owned elements + one ghost layer, different local numbering).
-m gpu: in-process ranks on one GPU (swe_link_group / swe_step_group) must be
bit-identical to the single-rank run (per-element arithmetic is unchanged by
the partition; only data movement differs) and within 1e-12 of the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1403_1661_b200 as P
import swe_inputs as si


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partition(mesh, nparts, axis=0):
    v = mesh.etov
    cx = (mesh.vx[v].mean(1) if axis == 0 else mesh.vy[v].mean(1))
    edges = np.quantile(cx, np.linspace(0, 1, nparts + 1)[1:-1])
    return np.searchsorted(edges, cx, side="right").astype(np.int32)


def _submesh(mesh, owner, rank):
    """Owned elements + all face neighbours (one layer), renumbered; gid = global index."""
    e2e, _, _ = P.host_connectivity(mesh.vx, mesh.vy, mesh.etov)
    own = np.where(owner == rank)[0]
    keep = np.unique(np.concatenate([own, e2e[own].ravel()]))
    rng = np.random.default_rng(rank)
    keep = rng.permutation(keep)  # local order unrelated to the global one
    return mesh.etov[keep], owner[keep], keep.astype(np.int64)


def _worker(rank, world, port, results, submesh):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = si.c4_dambreak(N=2, base=10).mesh
    owner = _partition(m, world)
    if submesh:
        etov, own, gid = _submesh(m, owner, rank)
        plan = P.host_halo_plan(m.vx, m.vy, etov, own, rank, gid=gid)
    else:
        plan = P.host_halo_plan(m.vx, m.vy, m.etov, owner, rank)
    mine = {"rank": rank, "peers": plan["peers"], "send": plan["send_gids"].tolist(),
            "recv": plan["recv_gids"].tolist(), "owned": plan["owned"]}
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    ok = True
    for q in range(world):
        if q == rank:
            continue
        # my receive list from q == q's send list to me (same gid order)
        def lst(d, which, peer):
            off = 0
            for (pr, ns, nr) in d["peers"]:
                n = ns if which == "send" else nr
                if pr == peer:
                    return d[which][off:off + n]
                off += n
            return []
        ok = ok and lst(mine, "recv", q) == lst(gathered[q], "send", rank)
        ok = ok and lst(mine, "send", q) == lst(gathered[q], "recv", rank)
    total_owned = sum(d["owned"] for d in gathered)
    results[rank] = (ok, total_owned, m.K, len(mine["recv"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("submesh", [False, True])
def test_halo_plan_consistent_across_two_processes(submesh):
    P.lib()
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results, submesh), nprocs=world, join=True)
    for r in range(world):
        ok, total_owned, K, nrecv = results[r]
        assert ok
        assert total_owned == K  # the partition covers every element exactly once
        assert nrecv > 0


def test_halo_plan_three_ranks_single_process():
    m = si.c4_dambreak(N=2, base=10).mesh
    owner = _partition(m, 3)
    plans = [P.host_halo_plan(m.vx, m.vy, m.etov, owner, r) for r in range(3)]
    for r in range(3):
        for (q, ns, nr) in plans[r]["peers"]:
            assert q != r
            back = [p for p in plans[q]["peers"] if p[0] == r][0]
            assert back[1] == nr and back[2] == ns
    assert sum(p["owned"] for p in plans) == m.K


@pytest.mark.gpu
@pytest.mark.parametrize("nparts,nlevels", [(2, 3), (3, 2)])
def test_partitioned_group_bit_identical(nparts, nlevels):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests.common import make_oracle, parity_rel
    w = si.c4_dambreak(N=3, base=5)
    m = w.mesh
    o, d = make_oracle(w)
    dt = si.dt_for(m, w.N, w.g, 1.875, 13.0, 0.2)
    ref = P.Solver(m.vx, m.vy, m.etov, d["B"], w.N, w.g, params=w.params)
    ref.set_state(d["h"], d["hu"], d["hv"])
    owner = _partition(m, nparts, axis=0)  # x bands cut across the refinement levels
    parts = [P.Solver(m.vx, m.vy, m.etov, d["B"], w.N, w.g, params=w.params, rank=r, nranks=nparts, owner=owner)
             for r in range(nparts)]
    P.link_group(parts)
    for s in parts:
        s.set_state(d["h"], d["hu"], d["hv"])
    o.set_state(d["h"], d["hu"], d["hv"])
    for _ in range(6):
        ref.step(dt, nlevels)
        P.step_group(parts, dt, nlevels)
        assert o.step(dt, nlevels) == 0
    full = ref.get_state()
    merged = [np.full_like(full[0], np.nan) for _ in range(3)]
    for r, s in enumerate(parts):
        out = tuple(np.full_like(full[0], np.nan) for _ in range(3))
        s.get_state(out)
        sel = owner == r
        for f in range(3):
            merged[f][sel] = out[f][sel]
            assert np.all(np.isnan(out[f][~sel]))  # only owned rows are written
    for f in range(3):
        assert np.array_equal(merged[f], full[f])  # bit-identical to the single-rank run
    assert max(parity_rel(merged, o.get_state(), w.g)) <= 1e-12
    assert np.array_equal(parts[0].levels(), ref.levels())


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3])
def test_c5_rank_strips_bit_identical(nranks):
    """bench.py's multi-rank setup without NCCL: every rank builds only its own C5 y-strip plus
    buffer rows (si.c5_rank_strip: own numbering, owner by centroid, gid = exact centroid key); the
    ranks run as an in-process group on one GPU.  By global id, their owned elements must equal a
    single-rank run of the whole basin bit for bit, levels included."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base_n, N, L = 80, 3, 4
    full = si.c5_tsunami(P=nranks, base_n=base_n, shuffle_seed=None)
    mf = full.mesh
    x, y = P.nodes(mf.vx, mf.vy, mf.etov, N)
    Bf, hf, huf, hvf = full.fields(x, y)
    dt = si.dt_for(mf, N, full.g, 4001.0, full.params["a_floor"], full.dt_factor)
    ref = P.Solver(mf.vx, mf.vy, mf.etov, Bf, N, full.g, params=full.params)
    ref.set_state(hf, huf, hvf)
    gid_full = si.centroid_keys(mf, si.C5_LX / base_n)
    where = {int(g): i for i, g in enumerate(gid_full)}
    parts, owners, gids = [], [], []
    for r in range(nranks):
        w, owner, gid = si.c5_rank_strip(r, nranks, base_n)
        m = w.mesh
        xr, yr = P.nodes(m.vx, m.vy, m.etov, N)
        B, h, hu, hv = w.fields(xr, yr)
        s = P.Solver(m.vx, m.vy, m.etov, B, N, w.g, params=w.params, rank=r, nranks=nranks, owner=owner, gid=gid)
        parts.append((s, (h, hu, hv)))
        owners.append(owner)
        gids.append(gid)
    P.link_group([s for s, _ in parts])
    for s, st in parts:
        s.set_state(*st)
    for _ in range(3):
        ref.step(dt, L)
        P.step_group([s for s, _ in parts], dt, L)
    fs = ref.get_state()
    flev = ref.levels()
    covered = 0
    for r, (s, st) in enumerate(parts):
        out = tuple(np.full_like(st[0], np.nan) for _ in range(3))
        s.get_state(out)
        lev = s.levels()
        own = np.where(owners[r] == r)[0]
        idx = np.array([where[int(g)] for g in gids[r][own]])
        for f in range(3):
            assert np.array_equal(out[f][own], fs[f][idx])
        assert np.array_equal(lev[own], flev[idx])
        covered += len(own)
    assert covered == mf.K


# ---------------------------------------------------------------- CUDA-IPC transport, one process per rank
def _ipc_worker(rank, world, port, outdir, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)  # every rank on the one GPU of the box: NCCL refuses this, IPC does not
    if case.startswith("c4"):  # "c4": N = 3 (scalar K1); "c4n5": N = 5 (the persistent DMMA K1 on sub-ranges)
        w = si.c4_dambreak(N=5 if case == "c4n5" else 3, base=5)
        m = w.mesh
        owner = _partition(m, world)
        gid = None
        L, nsteps = 3, 6
        dt = si.dt_for(m, w.N, w.g, 1.875, 13.0, 0.2)
    else:  # bench.py's weak-scaling setup: every rank builds only its own C5 strip (+ buffer rows)
        w, owner, gid = si.c5_rank_strip(rank, world, 80)
        m = w.mesh
        L, nsteps = 4, 8
        full = si.c5_tsunami(P=world, base_n=80, shuffle_seed=None)
        dt = si.dt_for(full.mesh, 3, full.g, 4001.0, full.params["a_floor"], full.dt_factor)
    x, y = P.nodes(m.vx, m.vy, m.etov, w.N)
    B, h, hu, hv = w.fields(x, y)
    s = P.Solver(m.vx, m.vy, m.etov, B, w.N, w.g, params=w.params, rank=rank, nranks=world, owner=owner, gid=gid)
    P.ipc_connect(s)
    s.set_state(h, hu, hv)
    for _ in range(nsteps):
        s.step(dt, L)
    out = tuple(np.full_like(h, np.nan) for _ in range(3))
    s.get_state(out)
    np.save(os.path.join(outdir, f"state{rank}.npy"), np.stack(out))
    np.save(os.path.join(outdir, f"levels{rank}.npy"), s.levels())
    np.save(os.path.join(outdir, f"owner{rank}.npy"), owner)
    if gid is not None:
        np.save(os.path.join(outdir, f"gid{rank}.npy"), gid)
    dist.barrier()  # every rank is done reading the others' exchange blocks
    s.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case,world", [("c4", 2), ("c4", 3), ("c5", 2), ("c4n5", 2)])
def test_ipc_ranks_bit_identical(case, world, tmp_path):
    """The CUDA-IPC transport with one process per rank (all on this box's single GPU): boundary-first
    level updates with the halo exchanges on a communication stream (stream-memory-op flags, peer copies
    of face traces), the macro steps after the AB ramp captured as CUDA graphs and replayed.  The owned
    elements must equal a single-rank run bit for bit, levels included."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.spawn(_ipc_worker, args=(world, _free_port(), str(tmp_path), case), nprocs=world, join=True)
    if case.startswith("c4"):
        w = si.c4_dambreak(N=5 if case == "c4n5" else 3, base=5)
        m = w.mesh
        L, nsteps = 3, 6
        dt = si.dt_for(m, w.N, w.g, 1.875, 13.0, 0.2)
    else:
        w = si.c5_tsunami(P=world, base_n=80, shuffle_seed=None)
        m = w.mesh
        L, nsteps = 4, 8
        dt = si.dt_for(m, 3, w.g, 4001.0, w.params["a_floor"], w.dt_factor)
    x, y = P.nodes(m.vx, m.vy, m.etov, w.N)
    B, h, hu, hv = w.fields(x, y)
    ref = P.Solver(m.vx, m.vy, m.etov, B, w.N, w.g, params=w.params)
    ref.set_state(h, hu, hv)
    for _ in range(nsteps):
        ref.step(dt, L)
    full = np.stack(ref.get_state())
    flev = ref.levels()
    where = None
    if case == "c5":
        where = {int(g): i for i, g in enumerate(si.centroid_keys(m, si.C5_LX / 80))}
    covered = 0
    for r in range(world):
        st = np.load(tmp_path / f"state{r}.npy")
        lev = np.load(tmp_path / f"levels{r}.npy")
        owner = np.load(tmp_path / f"owner{r}.npy")
        own = np.where(owner == r)[0]
        idx = own if where is None else np.array([where[int(g)] for g in np.load(tmp_path / f"gid{r}.npy")[own]])
        assert np.array_equal(st[:, own], full[:, idx])
        assert np.array_equal(lev[own], flev[idx])
        covered += len(own)
    assert covered == m.K
