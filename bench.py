#!/usr/bin/env python
"""Benchmark of the hot path: FP64 DOF-updates/s of the MRAB + PP + TVB nodal-DG
shallow-water step at N = 3 on the synthetic C5 tsunami basin.

One "step" = one MRAB macro step (2^(L-1) finest substeps, every level updated
its 2^(L-l) times, K1 + K2 per update).  DOF-update = (element, node, field)
advanced by one substep of its level: U = 3 Np sum_l K_l 2^(L-l) per macro step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle
(the deliberately slow checker) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import atexit
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "DOF-updates/s (FP64, N=3) at 1/2/4/8 B200; % HBM roofline"
UNIT = "DOF-updates/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []  # (host time, fields)
        self.proc = None
        self.window = None  # host-time window of the timed region

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", os.environ.get("BENCH_CLK_MS", "25")], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append((time.time(), parts))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        """Samples taken inside the timed region; if the region is shorter than nvidia-smi's sampling
        interval, the samples of the warm-up steps just before it (same kernels, GPU busy) are used and
        the window says so."""
        rows, window = [], "timed"
        if self.window:
            t0, t1, tw = self.window
            rows = [r for t, r in self.rows if t0 <= t <= t1]
            if not rows:
                rows, window = [r for t, r in self.rows if tw <= t <= t1], "warmup+timed"
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "window": window}


class GpmDram:
    """DRAM bandwidth utilisation of the GPU over an interval, from the hardware counters NVML's GPU
    Performance Monitoring reads (NVML_GPM_METRIC_DRAM_BW_UTIL, Hopper and later): an in-run measurement of
    the traffic the step really moves, next to the algorithmic byte count."""

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml as nv
            self.nv = nv
            nv.nvmlInit()
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            if not nv.nvmlGpmQueryDeviceSupport(self.h).isSupportedDevice:
                return
            self.s1, self.s2 = nv.nvmlGpmSampleAlloc(), nv.nvmlGpmSampleAlloc()
            mem_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_MEM)
            bus = nv.nvmlDeviceGetMemoryBusWidth(self.h)
            self.theoretical_gbs = 2.0 * mem_mhz * 1e6 * bus / 8 / 1e9  # double data rate
            self.ok = True
        except Exception as e:  # no NVML / GPM on this box: reported as unavailable
            self.err = repr(e)

    def start(self):
        if self.ok:
            try:
                self.nv.nvmlGpmSampleGet(self.h, self.s1)
            except Exception as e:  # GPM present but not permitted here (e.g. containerised driver)
                self.ok, self.err = False, repr(e)

    def stop(self):
        if not self.ok:
            return None
        try:
            nv = self.nv
            nv.nvmlGpmSampleGet(self.h, self.s2)
            mg = nv.c_nvmlGpmMetricsGet_t()
            mg.version = nv.NVML_GPM_METRICS_GET_VERSION
            mg.numMetrics = 1
            mg.sample1, mg.sample2 = self.s1, self.s2
            mg.metrics[0].metricId = nv.NVML_GPM_METRIC_DRAM_BW_UTIL
            nv.nvmlGpmMetricsGet(mg)
            if mg.metrics[0].nvmlReturn != 0:
                return None
            return float(mg.metrics[0].value)
        except Exception as e:
            self.err = repr(e)
            return None


def workload(P_strip: int, base_n: int, strip: int = 1):
    import swe_inputs as si
    return si.c5_tsunami(P=P_strip, base_n=base_n, strip=strip)


def dof_per_macro_step(levels: np.ndarray, L: int, Np: int) -> int:
    cnt = np.bincount(levels, minlength=L + 1)
    return int(3 * Np * sum(int(cnt[l]) * 2 ** (L - l) for l in range(1, L + 1)))


def cpu_baseline(args, seconds_budget=30.0):
    """The oracle as it stands, on a bounded sample: a y-strip of the C5 mesh, 1 macro step."""
    import oracle
    import swe_inputs as si
    cores = oracle.set_threads(0)
    w = workload(1, args.base_n, strip=args.cpu_strip)
    m = w.mesh
    Np = 10
    probe = oracle.Oracle(m.vx, m.vy, m.etov, np.zeros((m.K, Np)), 3, w.g, **w.params)
    x, y = probe.nodes()
    del probe
    B, h, hu, hv = w.fields(x, y)
    o = oracle.Oracle(m.vx, m.vy, m.etov, B, 3, w.g, **w.params)
    o.set_state(h, hu, hv)
    dt = si.dt_for(m, 3, w.g, 4001.0, w.params["a_floor"], w.dt_factor)
    o.step(dt, w.nlevels)  # schedule + first (Euler) step, untimed
    lev = o.levels()
    U = dof_per_macro_step(lev, w.nlevels, Np)
    t0 = time.perf_counter()
    n = 0
    while True:
        rc = o.step(dt, w.nlevels)
        assert rc == 0
        n += 1
        if time.perf_counter() - t0 > seconds_budget * 0.5 or n >= args.cpu_steps:
            break
    el = time.perf_counter() - t0
    out = {"value": U * n / el, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"C5 y-strip 1/{args.cpu_strip} ({m.K} elements, N=3, L={w.nlevels}), {n} macro step(s) after "
                     f"the first, {el:.1f} s"}
    del o
    # the same oracle on one core, on a 1/32 strip (one macro step after the first)
    oracle.set_threads(1)
    try:
        w1 = workload(1, args.base_n, strip=32)
        m1 = w1.mesh
        probe = oracle.Oracle(m1.vx, m1.vy, m1.etov, np.zeros((m1.K, Np)), 3, w1.g, **w1.params)
        x1, y1 = probe.nodes()
        del probe
        B1, h1, hu1, hv1 = w1.fields(x1, y1)
        o1 = oracle.Oracle(m1.vx, m1.vy, m1.etov, B1, 3, w1.g, **w1.params)
        o1.set_state(h1, hu1, hv1)
        dt1 = si.dt_for(m1, 3, w1.g, 4001.0, w1.params["a_floor"], w1.dt_factor)
        assert o1.step(dt1, w1.nlevels) == 0
        U1 = dof_per_macro_step(o1.levels(), w1.nlevels, Np)
        t0 = time.perf_counter()
        assert o1.step(dt1, w1.nlevels) == 0
        el1 = time.perf_counter() - t0
        out["one_core"] = {"value": U1 / el1, "cores": 1,
                           "sample": f"C5 y-strip 1/32 ({m1.K} elements), 1 macro step after the first, {el1:.1f} s"}
    finally:
        oracle.set_threads(cores)
    return out


def workloads_table(args, dev):
    """SURVEY 8(d) "oracle beside it": the CPU oracle and the GPU path on the smaller configs C1-C4 (same inputs, same
    steps after an untimed start), DOF-updates/s each; bounded so that it adds ~20 s to the run."""
    import torch

    import oracle
    import paper_1403_1661_b200 as P
    import swe_inputs as si
    cores = oracle.set_threads(0)
    cases = [
        ("C1b lake + hump, N=2, 512 el, 1 level", si.c1_lake(N=2, n=16, hump=True), 1, 100,
         lambda w: si.dt_for(w.mesh, 2, w.g, 1.0, 0.0, 0.2)),
        ("C2 vortex, N=3, periodic 2x64x64, 1 level", si.c2_vortex(3, 64), 1, 20,
         lambda w: si.dt_for(w.mesh, 3, 2.0, 1.0, 0.0, 0.1, u_max=2.0)),
        ("C3 Thacker, N=2, 20k el, PP+TVB, 1 level", si.c3_thacker(N=2, n=100), 1, 20,
         lambda w: si.dt_for(w.mesh, w.N, w.g, 1.75, 0.0, 0.2, u_max=0.5)),
        ("C4 dam break, N=3, 188k el, PP+TVB, 3 levels", si.c4_dambreak(N=3, base=1), 3, 3,
         lambda w: si.dt_for(w.mesh, 3, w.g, 1.875, 13.0, 0.2)),
    ]
    rows = []
    for name, w, L, nsteps, dtf in cases:
        m = w.mesh
        Np = (w.N + 1) * (w.N + 2) // 2
        x, y = P.nodes(m.vx, m.vy, m.etov, w.N)
        B, h, hu, hv = w.fields(x, y)
        dt = dtf(w)
        o = oracle.Oracle(m.vx, m.vy, m.etov, B, w.N, w.g, vper=m.vper, **w.params)
        o.set_state(h, hu, hv)
        for _ in range(3):  # past the AB ramp
            assert o.step(dt, L) == 0
        U = dof_per_macro_step(o.levels(), L, Np)
        t0 = time.perf_counter()
        for _ in range(nsteps):
            assert o.step(dt, L) == 0
        t_cpu = time.perf_counter() - t0
        del o
        s = P.Solver(m.vx, m.vy, m.etov, B, w.N, w.g, vper=m.vper, params=w.params, device=dev)
        s.set_state(h, hu, hv)
        for _ in range(3):
            s.step(dt, L)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(nsteps):
            s.step(dt, L)
        torch.cuda.synchronize()
        t_gpu = time.perf_counter() - t0
        s.close()
        rows.append({"config": name, "elements": int(m.K), "steps": nsteps,
                     "oracle_dof_per_s": U * nsteps / t_cpu, "gpu_dof_per_s": U * nsteps / t_gpu})
    cpu_model = ""
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name"):
                cpu_model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"oracle_cores": cores, "cpu_model": cpu_model, "runs": rows,
            "note": "wall clock after 3 untimed steps; the small GPU cases are launch-bound (CUDA-graph replay)"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle timed as it stands on the box's host cores."""
    if rank != 0:
        return
    import oracle
    import swe_inputs as si
    cores = oracle.set_threads(0)
    w = workload(1, args.base_n, strip=args.cpu_strip)
    m = w.mesh
    Np = 10
    probe = oracle.Oracle(m.vx, m.vy, m.etov, np.zeros((m.K, Np)), 3, w.g, **w.params)
    x, y = probe.nodes()
    del probe
    B, h, hu, hv = w.fields(x, y)
    o = oracle.Oracle(m.vx, m.vy, m.etov, B, 3, w.g, **w.params)
    o.set_state(h, hu, hv)
    dt = si.dt_for(m, 3, w.g, 4001.0, w.params["a_floor"], w.dt_factor)
    for _ in range(args.warmup):
        assert o.step(dt, w.nlevels) == 0
    lev = o.levels()
    U = dof_per_macro_step(lev, w.nlevels, Np)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        assert o.step(dt, w.nlevels) == 0
    el = time.perf_counter() - t0
    val = U * args.steps / el
    sample = f"C5 y-strip 1/{args.cpu_strip} ({m.K} elements, N=3, L={w.nlevels})"
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": sample, "N": 3, "nlevels": w.nlevels},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--order", type=int, default=3, help="polynomial order N of the GPU arm (headline: 3)")
    ap.add_argument("--precision", type=int, default=64, choices=(32, 64),
                    help="device arithmetic of the GPU arm (headline: 64; 32 = FP32 variant, SURVEY NEXT-2)")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--base-n", type=int, default=1280)
    ap.add_argument("--cpu-strip", type=int, default=4)
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-workloads", action="store_true", help="skip the C1-C4 oracle/GPU table")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="halo exchange for N > 1: CUDA-IPC peer copies (default; also ranks sharing a GPU) or NCCL")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "W >= 3"

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # no launcher: start one process per rank here (same environment contract as torchrun)
        import socket

        import torch.multiprocessing as mp
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        mp.spawn(_spawned_rank, args=(args, port), nprocs=args.gpus, join=True)
        return
    run_rank(args)


def _spawned_rank(local, args, port):
    os.environ.update(RANK=str(local), LOCAL_RANK=str(local), WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    run_rank(args)


def run_rank(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    import paper_1403_1661_b200 as P
    import swe_inputs as si

    ndev = torch.cuda.device_count()
    dev = local % ndev  # ranks beyond the device count share GPUs (CUDA-IPC transport only)
    torch.cuda.set_device(dev)
    shared = world > ndev
    backend = "gloo" if shared else "nccl"
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
        if shared and args.transport == "nccl":
            raise SystemExit("bench.py: NCCL cannot run two ranks on one GPU; use --transport ipc")
    tdev = "cuda" if backend == "nccl" else "cpu"

    def allreduce(x, op):
        t = torch.tensor([x], device=tdev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=op)
        return float(t.item())

    P.lib()

    # ---- workload: C5 tsunami basin.  N=1: the full 2000 km x 2000 km basin.  N>1 (weak scaling):
    # a 2000 km x (2000 km * N) basin, rank r owns the r-th 2000 km y-strip; every rank generates its
    # strip plus two buffer rows, ghosts are refreshed by NCCL halo exchanges after every level update.
    t_setup = time.time()
    if world > 1:
        w, owner, gid = si.c5_rank_strip(rank, world, args.base_n)
        part = dict(rank=rank, nranks=world, owner=owner, gid=gid)
        if args.transport == "nccl":
            idbuf = [P.nccl_unique_id() if rank == 0 else None]
            torch.distributed.broadcast_object_list(idbuf, src=0)
            part["nccl_id"] = idbuf[0]
    else:
        w = workload(1, args.base_n)
        owner = None
        part = {}
    m = w.mesh
    N, L = args.order, w.nlevels
    Np = (N + 1) * (N + 2) // 2
    x, y = P.nodes(m.vx, m.vy, m.etov, N)
    B, h, hu, hv = w.fields(x, y)
    del x, y
    s = P.Solver(m.vx, m.vy, m.etov, B, N, w.g, params=dict(w.params, precision=args.precision), device=dev,
                 **part)
    if world > 1 and args.transport == "ipc":
        P.ipc_connect(s)
    dt = si.dt_for(m, N, w.g, 4001.0, w.params["a_floor"], w.dt_factor)
    if world > 1:
        dt = allreduce(dt, torch.distributed.ReduceOp.MIN)
    s.set_state(h, hu, hv)
    stream = torch.cuda.current_stream()
    clk = ClockSampler(dev).__enter__()  # started early: nvidia-smi needs a moment before its first row
    atexit.register(clk.__exit__, None, None, None)  # no stray nvidia-smi if the run fails below
    time.sleep(0.5)
    t_warm = time.time()
    for _ in range(args.warmup):
        s.step(dt, L)
    lev_all = s.levels()
    lev = lev_all if owner is None else lev_all[owner == rank]
    U = dof_per_macro_step(lev, L, Np)
    t_setup = time.time() - t_setup

    # ---- timed region: K macro steps, device time with CUDA events on the solver's stream
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    gpm = GpmDram(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    gpm.start()
    ev0.record(stream)
    for _ in range(args.steps):
        s.step(dt, L)  # single rank: each macro step replays a captured CUDA graph
    ev1.record(stream)
    torch.cuda.synchronize()
    dram_util = gpm.stop()
    clk.window = (t0, time.time(), t_warm)
    time.sleep(0.05)  # let the reader thread take the last rows of the window
    clk.__exit__(None, None, None)
    ms = ev0.elapsed_time(ev1)
    # per-kernel device times (K1 / K2 events on the solver stream) from a second, profiled run of the
    # same length (profiling launches eagerly, so it is kept out of the timed region above)
    s.profile(True)
    for _ in range(args.steps):
        s.step(dt, L)
    torch.cuda.synchronize()
    s.profile(False)
    prof = s.profile_read()
    prof_ms = prof["k1_ms"] + prof["k2_ms"]
    ms_rank = ms
    if world > 1:
        ms = allreduce(ms, torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
    ms_per_step = ms / args.steps
    U_all = U
    if world > 1:
        U_all = int(allreduce(float(U), torch.distributed.ReduceOp.SUM))
    value = U_all * args.steps / (ms / 1e3)

    # ---- roofline.  Bytes: SURVEY 8(d)'s algorithmic count per element-update, B_alg = esz (6 Np [Q r+w] +
    # 9 Np [AB ring 2 r + 1 w] + Np [B] + 9 Nfp [neighbour face values] + 3 Nfp [neighbour B] + 6 [vertices]
    # + 12 [means]) + 16 [indices] -- 1824 B at N = 3 in FP64 -- times the element-updates of the run.
    # Time: the dominant kernel K1, every launch timed with CUDA events on the solver stream (profiled run of
    # the same steps), and the whole graph-replayed step.
    peak, peak_kind = load_peaks()
    Nfp = N + 1
    esz = 8 if args.precision == 64 else 4
    b_alg = esz * (6 * Np + 9 * Np + Np + 9 * Nfp + 3 * Nfp + 6 + 12) + 16
    upd = U * args.steps / (3 * Np)  # element-updates of this rank in the timed (and in the profiled) steps
    k1_gbs = b_alg * upd / (prof["k1_ms"] / 1e3) / 1e9
    step_gbs = b_alg * upd / (ms_rank / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": k1_gbs, "peak": peak, "unit": "GB/s", "frac": k1_gbs / peak,
            "traffic": None, "kernel": f"k_rhs_update<{N}>", "peak_kind": peak_kind,
            "bytes_model": "SURVEY 8(d) B_alg per element-update", "algorithmic_bytes_per_elem_update": b_alg,
            "k1_launch_ms_avg": prof["k1_ms"] / max(1, prof["k1_launches"]),
            "step_achieved": step_gbs, "step_frac": step_gbs / peak,
            "k1_share_of_kernel_time": prof["k1_ms"] / prof_ms if prof_ms > 0 else None,
            "k2_share_of_kernel_time": prof["k2_ms"] / prof_ms if prof_ms > 0 else None,
            "eager_kernel_ms_over_graph_step_ms": prof_ms / ms_rank if ms_rank > 0 else None,
            "library_k1_model_bytes_per_elem_update": prof["k1_bytes"] / upd if upd else None}
    if dram_util is None:
        roof["dram_measured"] = {"source": "NVML GPM DRAM_BW_UTIL", "unavailable": getattr(gpm, "err", "no GPM")}
    else:  # measured in this run: hardware DRAM counters over the timed region
        dram_gbs = dram_util / 100.0 * gpm.theoretical_gbs
        roof["dram_measured"] = {
            "source": "NVML GPM DRAM_BW_UTIL over the timed region (whole step, all kernels)",
            "util_pct_of_theoretical": dram_util, "theoretical_gbs": gpm.theoretical_gbs, "gbs": dram_gbs,
            "frac_of_measured_peak": dram_gbs / peak,
            "bytes_per_elem_update": dram_gbs * 1e9 * (ms_rank / 1e3) / upd if upd else None}
    traffic_path = os.path.join(ROOT, "profiles", "r02b_k1_traffic.json")
    if N == 3 and args.precision == 64 and os.path.exists(traffic_path):
        try:  # K1's own DRAM bytes per launch: ncu --set full capture committed under profiles/ (not this run)
            tr = json.load(open(traffic_path))
            roof["traffic"] = tr["bytes_per_launch"]
            roof["traffic_source"] = "ncu dram__bytes_read.sum + dram__bytes_write.sum, " + os.path.relpath(
                traffic_path, ROOT) + " (one level-4 K1 launch; not measured in this run)"
            roof["traffic_launch_elements"] = tr["elements"]
            roof["traffic_bytes_per_elem_update"] = tr["bytes_per_elem_update"]
        except Exception:
            pass

    info = s.info()

    # ---- end to end through the C ABI with host buffers.  Timed region: swe_set_state from pinned host
    # memory (H2D of the state, level binning, initial limiting), then every macro step swe_step + the
    # step's result read back to the host (swe_get_info: mass, min h and limiter counters, D2H of the
    # per-block partials and counters), and the final state D2H into pinned host memory.
    e2e = None
    if args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        hh, hhu, hhv = pin(h), pin(hu), pin(hv)
        oh, ohu, ohv = pin(np.zeros_like(h)), pin(np.zeros_like(h)), pin(np.zeros_like(h))
        s.get_state_into(oh, ohu, ohv)  # untimed warm-up of the read-back path (its one-time device buffer)
        state_bytes = 3 * h.size * 8
        info_bytes = 2 * 8 * ((len(lev) + 255) // 256) + 8 * 6 * 64 + 8 * 64  # partials + counters + injected
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.set_state(hh, hhu, hhv)
        for _ in range(args.e2e_steps):
            s.step(dt, L)
            s.info()
        s.get_state_into(oh, ohu, ohv)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:
            el = allreduce(el, torch.distributed.ReduceOp.MAX)
        k = args.e2e_steps
        e2e = {"value": U_all * k / el, "unit": UNIT,
               "h2d_bytes_per_step": int(state_bytes / k), "d2h_bytes_per_step": int(info_bytes + state_bytes / k),
               "steps": k,
               "note": "wall clock, max over ranks: swe_set_state (H2D from pinned memory + level binning + initial "
                       "limiting) once, then per macro step swe_step + swe_get_info (the step's diagnostics D2H), then "
                       "the final state D2H (swe_get_state into pinned memory)"}
        # secondary: the full state read back after every macro step (output-every-step usage), synchronously
        # (swe_get_state) and overlapped with the next steps (swe_get_state_async into two pinned buffer sets,
        # swe_wait_state before the clock stops)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.set_state(hh, hhu, hhv)
        for _ in range(args.e2e_steps):
            s.step(dt, L)
            s.get_state_into(oh, ohu, ohv)
        torch.cuda.synchronize()
        el2 = time.perf_counter() - t0
        e2e["state_every_step"] = {"value": U_all * k / el2, "d2h_bytes_per_step": int(state_bytes)}
        if world == 1:
            ring = [(oh, ohu, ohv), (pin(np.zeros_like(h)), pin(np.zeros_like(h)), pin(np.zeros_like(h)))]
            s.get_state_async(*ring[1])  # untimed: the snapshot buffers' one-time allocation
            s.wait_state()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.set_state(hh, hhu, hhv)
            for i in range(args.e2e_steps):
                s.step(dt, L)
                s.get_state_async(*ring[i % 2])
            s.wait_state()
            torch.cuda.synchronize()
            el3 = time.perf_counter() - t0
            e2e["state_every_step_async"] = {"value": U_all * k / el3, "d2h_bytes_per_step": int(state_bytes)}

    if world > 1:
        torch.distributed.barrier()  # every rank is done with the others' exchange blocks
    s.close()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)
        if world == 1 and not args.no_workloads and args.order == 3 and args.precision == 64:
            cpu["workloads"] = workloads_table(args, dev)
    if rank == 0:
        out = {
            "metric": METRIC.replace("N=3", f"N={N}").replace("FP64", "FP64" if args.precision == 64 else "FP32"),
            "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if args.precision == 64 else "f32", "data": "synthetic",
            "config": {"workload": f"C5 synthetic tsunami basin (SURVEY 8(d)), N={N}, 4 MRAB levels, PP+TVB"
                                   + (f", {world} y-strips (weak scaling, {args.transport} halo exchange)"
                                      if world > 1 else ""),
                       "ranks_share_gpus": bool(world > 1 and shared),
                       "K_per_rank": int(len(lev)), "level_counts": [int(c) for c in np.bincount(lev, minlength=L + 1)[1:]],
                       "dof_updates_per_step": U_all, "dt": dt, "l2": "inputs larger than L2 (state+history ~13 GB/rank)",
                       "parallelism": f"element partition x{world}", "setup_s": round(t_setup, 1)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(prof["k1_launches"] + prof["k2_launches"]),
            "clocks": clk.summary(),
            "counters": {k: info[k] for k in ("n_pp", "n_dry", "n_tvb", "n_posfix", "n_tvb_cw")},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
