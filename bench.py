#!/usr/bin/env python
"""Benchmark of the SRCD hot path (one outer iteration = F half-step + W half-step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4|C5] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, the script re-launches itself
through ``torch.distributed.run --nproc-per-node N`` (one process per GPU,
NCCL; it fails if fewer than N GPUs are visible).

Default workload: BASELINE.json config C4 (102,660 x 300,000, ~68M nnz,
r=100, alpha1=alpha2=0.01, fp32 storage / fp64 arithmetic) -- the config the
metric "outer iterations/sec and nnz*r coordinate updates/sec at 1/2/4/8
B200" is specified on.  Synthetic data of that shape (synth.py), U(0,1)
initial factors rounded to fp32.  Under torchrun (N>1) each rank owns a
share of each side's subproblems balanced by modelled device time, and the
solver kernels store their results into every peer's copy over NVLink
(fused exchange; NCCL all-gather with KLNMF_FUSED_EXCHANGE=0), a barrier per
half-step (strong scaling: fixed C4).

value      nnz*r coordinate updates/s = 2*nnz*r / step time, data resident in HBM,
           device time (CUDA events, max over ranks), L2 flushed between steps.
e2e        the same metric through the public API (factorize with HOST numpy
           inputs: upload, device CSR build, bucketing, K iterations, download);
           the median of E2E_JOBS (5) complete jobs, each job's seconds listed.
roofline   the dominant solver kernel: SURVEY.md §8(d) algorithmic bytes of the
           launch / its CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the reference algorithm (oracle port of _kernels.sweep_range, dense
           maintained product as in the reference) on the host cores, on a
           stratified sample of subproblems, extrapolated to a full iteration,
           AT THE STATE OF THE TIMED WINDOW: the factors and visit order the
           GPU holds after its warm-up (iteration W+1).  The reference arm
           (--impl reference) reaches the same iteration by running W full
           iterations of the reference algorithm (oracle, support-t variant:
           bitwise the reference's iterates) before its sampled steps.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "outer iterations/sec and nnz·r coordinate updates/sec at 1/2/4/8 B200"
UNIT = "nnz*r updates/s"
E2E_JOBS = 5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=6.0,
                    help="wall seconds of one CPU-baseline sample (both arms use the same budget per sample)")
    ap.add_argument("--cpu-samples", type=int, default=3, help="CPU-baseline samples of the GPU arm")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu legs)")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-kernel-events", action="store_true")
    ap.add_argument("--e2e-jobs", type=int, default=None, help="complete factorize jobs timed for e2e "
                    "(default 5; 1 for C5)")
    return ap.parse_args()


def relaunch_distributed(args) -> int:
    """--gpus N > 1 outside torchrun: start N ranks of this script, one per
    GPU, through torch.distributed.run (rendezvous on 127.0.0.1)."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if args.gpus > have:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {have} CUDA device(s) are visible"}),
              flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    # the communicator lines (ranks, transports, NVLS) go to stderr
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(launch_cmd(args.gpus, port, sys.argv[1:]), env=env)


def launch_cmd(gpus: int, port: int, argv) -> list:
    """The torchrun command of a --gpus N run: N ranks of this script on one node."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *argv]


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def algorithmic_bytes(ptr_host, items, r, s_f=4, s_v=4, s_i=4, s_p=8):
    """SURVEY.md §8(d) per-unit bytes x the units one launch processes:
    gather s*r*s_f + V s*(s_i+s_v) + ptr s_p + moving row 2*r*s_f per item."""
    sizes = np.diff(ptr_host)[items]
    nnz = int(sizes.sum())
    return nnz * r * s_f + nnz * (s_i + s_v) + len(items) * (s_p + 2 * r * s_f)


def kernel_name(kinfo) -> str:
    """Source name of a fast-kernel ladder entry (kernel_id, capacity, lanes, npl)."""
    _, cap, lanes, npl = kinfo
    if cap < 0:
        return "solve_coop_kernel"
    if lanes <= 32:
        return f"solve_warp_kernel<{lanes}, {npl}>"
    if lanes <= 256:
        return f"solve_block_kernel<{lanes}, {npl}>"
    return f"solve_cluster_kernel ({lanes // 256} CTAs per subproblem)"


def iteration_bytes(n, m, nnz, r, s_f=4, s_v=4):
    """Whole outer iteration: both half-steps."""
    def half(n_fix, n_mov):
        return nnz * r * s_f + nnz * (4 + s_v) + (n_mov + 1) * 8 + 2 * n_mov * r * s_f + n_fix * r * s_f
    return half(n, m) + half(m, n)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        if self.index < 0:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------
SAMPLE_EDGES = [0, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 16384, 65536, 1 << 62]


def cpu_reference_sample(V, w, f, spec, ids, seconds: float, threads: int, pick_seed: int = 123, vt=None):
    """Time the reference algorithm on the host cores at a given state.

    The reference's own per-column code path (oracle port of
    _kernels.sweep_range, _kernels.py:123-144, with its dense length-N_fix
    maintained product) solves a stratified sample of subproblems of both
    sides at the state (w, f, ids) -- the factors and visit order of the
    iteration being timed.  Every sampled column's thread CPU time is
    recorded; the side's serial cost is sum_b mean_b * |bucket b|, and the
    iteration time is the serial cost / threads (ideal parallel scaling over
    the host cores, which flatters the reference).  Returns (updates/s,
    seconds per iteration, subproblems sampled, Newton steps per visit)."""
    import oracle

    oracle.build()
    r = spec.rank
    reg = spec.reg
    if vt is None:
        vt = oracle.transpose_csc(V.n_rows, V.n_cols, V.col_ptr, V.row_idx, V.values)[:3]
    pt, rt, vtv = vt
    sides = [("F", V.col_ptr, V.row_idx, V.values, w, f, reg.alpha2, reg.beta2),
             ("W", pt, rt, vtv, f, w, reg.alpha1, reg.beta1)]
    rng = np.random.default_rng(pick_seed)
    total_cpu = 0.0
    sampled = 0
    newton = 0
    per_side = seconds * threads / 2.0  # thread-seconds of sampling per side
    for name, ptr, idx, val, fixed, moving, a, b in sides:
        sizes = np.diff(ptr)
        sums = oracle.row_sums(fixed)
        buckets = [np.nonzero((sizes > lo) & (sizes <= hi))[0] for lo, hi in zip(SAMPLE_EDGES[:-1], SAMPLE_EDGES[1:])]
        buckets = [q for q in [np.nonzero(sizes == 0)[0]] + buckets if len(q)]
        mov = np.ascontiguousarray(moving).copy()  # sampled columns are solved in place
        # calibration: a few members of every bucket (all in one threaded call)
        calib = [np.sort(rng.choice(q, size=min(len(q), 4), replace=False)) for q in buckets]
        st, secs = oracle.sweep_cols_timed(ptr, idx, val, fixed, sums, mov, np.concatenate(calib), ids, a, b,
                                           n_workers=threads)
        est, pos = [], 0
        for c in calib:
            est.append(max(float(np.mean(secs[pos:pos + len(c)])), 1e-7))
            pos += len(c)
        # allocation: every bucket gets an equal share of the thread-seconds
        share = per_side / len(buckets)
        picks = []
        for q, c, e in zip(buckets, calib, est):
            rest = np.setdiff1d(q, c, assume_unique=True)
            k = int(min(len(rest), max(0, share / e - len(c))))
            picks.append(np.sort(rng.choice(rest, size=k, replace=False)) if k > 0 else rest[:0])
        cols = np.concatenate(picks) if picks else np.zeros(0, np.int64)
        # longest first so no thread finishes last with a long column
        cols = cols[np.argsort(-sizes[cols], kind="stable")]
        st2, secs2 = oracle.sweep_cols_timed(ptr, idx, val, fixed, sums, mov, cols, ids, a, b, n_workers=threads)
        by_col = dict(zip(np.concatenate(calib).tolist(), secs.tolist()))
        by_col.update(zip(cols.tolist(), secs2.tolist()))
        for q, c, p in zip(buckets, calib, picks):
            members = np.concatenate([c, p])
            t = np.array([by_col[int(j)] for j in members])
            total_cpu += float(t.mean()) * len(q)
            sampled += len(members)
        newton += int(st[2] + st2[2])
    iter_s = total_cpu / threads
    return 2.0 * V.nnz * r / iter_s, iter_s, sampled, newton / max(1, sampled * r)


# ----------------------------------------------------------------------
def setup_dist(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def load_config(name, device_matrix=False):
    """(spec, V, w0, f0, generation seconds).  C1-C4 are generated on the host
    (synth.generate).  C5's matrix (565M nonzeros) only exists on the device
    (synth.generate_device): V is the DeviceMatrix when device_matrix is set,
    else its host copy."""
    from paper_1604_04026_b200 import synth

    spec = synth.CONFIGS[name]
    t0 = time.perf_counter()
    if name == "C5":
        V = synth.generate_device(spec)
        if not device_matrix:
            V = V.to_host()
    else:
        V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec)
    return spec, V, w0, f0, time.perf_counter() - t0


def ids_at(seed: int, r: int, iteration: int) -> np.ndarray:
    """The reference's visit order of outer iteration `iteration` (1-based):
    the iteration-th rng.permutation(r) of default_rng(seed) (solver.py:276,287)."""
    rng = np.random.default_rng(seed)
    for _ in range(iteration):
        ids = rng.permutation(r).astype(np.int64)
    return ids


def run_reference(args):
    """--impl reference: the reference algorithm on the host CPU (rank 0 only).

    Warm-up: `warmup` full outer iterations of the reference algorithm from
    the config's initial factors (oracle, support-t variant -- bitwise the
    reference's iterates, at a fraction of the dense cost), which brings the
    state to the one the GPU arm times (iteration warmup+1).  Each timed
    step is then one stratified sample of the reference's per-column code
    path (dense maintained product) at that state (cpu_reference_sample)."""
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    spec, V, w0, f0, _ = load_config(args.config)
    threads = oracle.cores()
    r, reg = spec.rank, spec.reg
    t0 = time.perf_counter()
    if args.warmup > 0:
        st = oracle.drive(V.col_ptr, V.row_idx, V.values, spec.n, spec.m, w0, f0, r, reg.alpha1, reg.alpha2,
                          reg.beta1, reg.beta2, args.warmup, spec.seed, n_workers=threads, log=False)
        w, f = st["w"], st["f"]
    else:
        w, f = w0, f0
    warm_s = time.perf_counter() - t0
    ids = ids_at(spec.seed, r, args.warmup + 1)
    vt = oracle.transpose_csc(V.n_rows, V.n_cols, V.col_ptr, V.row_idx, V.values)[:3]
    vals, times, nsv = [], [], []
    sampled = 0
    for k in range(args.steps):
        v, t_iter, n_s, steps_per_visit = cpu_reference_sample(V, w, f, spec, ids, args.cpu_seconds, threads,
                                                               pick_seed=1000 + k, vt=vt)
        vals.append(v)
        times.append(t_iter)
        nsv.append(steps_per_visit)
        sampled += n_s
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(times)) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "outer_iters_per_sec": 1.0 / float(np.mean(times)),
        "config": {"workload": spec.name, "n": spec.n, "m": spec.m, "nnz": V.nnz, "rank": spec.rank,
                   "reg": vars(spec.reg)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"iteration {args.warmup + 1} state (after {args.warmup} full reference "
                                   f"iterations, {warm_s:.0f} s); per step a stratified sample "
                                   f"({sampled // max(1, args.steps)} subproblems, both sides, "
                                   f"~{args.cpu_seconds:.0f} s on {threads} threads) of the reference "
                                   f"sweep_range port (dense maintained product), per-column thread CPU "
                                   f"time extrapolated by bucket population / {threads} cores",
                         "iteration": args.warmup + 1,
                         "newton_steps_per_visit": float(np.mean(nsv)),
                         "step_values": [float(x) for x in vals]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1604_04026_b200 import NmfConfig, factorize, FactorPair, DenseFactor, SparseMatrix
    from paper_1604_04026_b200.plan import DevicePlan

    world, rank, local = setup_dist(args)
    group = dist.group.WORLD if world > 1 else None
    spec, V, w0, f0, gen_s = load_config(args.config, device_matrix=True)
    precision = spec.precision
    dev = torch.device("cuda", local)
    plan = DevicePlan(V, spec.rank, precision, local, group)
    if not isinstance(V, SparseMatrix):  # C5: host copy for the e2e / CPU legs (outside any timing)
        V = V.to_host()
        torch.cuda.empty_cache()
    plan.graph_after = 1  # timed steps replay captured graphs (captured during warm-up)
    r = spec.rank
    reg = spec.reg
    rng = np.random.default_rng(spec.seed)
    ids = rng.permutation(r).astype(np.int64)
    plan.set_factors(w0, f0, order=ids)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    kernel_ms = {}   # (side, kernel_id) -> list of ms
    launch_count = [0]

    def step(events, mid=None):
        nonlocal ids
        ids_next = rng.permutation(r).astype(np.int64)
        plan.half_step("F", ids, alpha=reg.alpha2, beta=reg.beta2, events=events)
        if mid is not None:
            mid.record(stream)
        plan.half_step("W", ids, ids_next, alpha=reg.alpha1, beta=reg.beta1, events=events)
        ids = ids_next

    for _ in range(args.warmup):  # same (instrumented or not) graphs as the timed steps
        step(None if args.no_kernel_events else [])
    torch.cuda.synchronize(dev)
    # the state of the first timed iteration, for the CPU baseline (read
    # outside the timed region)
    cpu_state = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        w_st, f_st = plan.get_factors()
        cpu_state = (w_st, f_st, ids.copy())
    if world > 1:
        dist.barrier()

    plan.take_stats()
    step_ms = []
    half_ms = []  # (F half-step incl. its exchange, W half-step incl. its exchange) per timed step
    step_kernel_ms = []
    with ClockSampler(-1 if args.no_clocks else local) as clocks:
        for _ in range(args.steps):
            if not args.no_flush:
                flush.zero_()
            ev = None if args.no_kernel_events else []
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            em = torch.cuda.Event(enable_timing=True)
            # ~1 ms device sleep outside [e0, e1]: the host enqueues the whole
            # step before the device reaches e0, so host latency after the
            # per-step synchronize is not counted as device time
            torch.cuda._sleep(2_000_000)
            e0.record(stream)
            step(ev, em)
            e1.record(stream)
            # per-kernel events are CUDA-graph nodes re-recorded by each replay:
            # read them before the next step (device time is unaffected)
            torch.cuda.synchronize(dev)
            step_ms.append(e0.elapsed_time(e1))
            half_ms.append((e0.elapsed_time(em), em.elapsed_time(e1)))
            ksum = 0.0
            for (side, kid, a, b) in ev or []:
                kms = a.elapsed_time(b)
                ksum += kms
                kernel_ms.setdefault((side, kid), []).append(kms)
                launch_count[0] += 1
            if ev:
                step_kernel_ms.append(ksum)
    launch_count[0] += plan.aux_launches_per_step * args.steps
    st = plan.take_stats()
    # Per-kernel durations for the kernel table and the roofline: in the timed
    # steps the buckets run concurrently, so a kernel's event span includes
    # time shared with its neighbours.  A short instrumented pass with the
    # buckets launched one at a time (same trajectory, continuing) gives each
    # kernel's own duration.
    kernel_ms = {}
    k_steps = max(2, min(args.steps, 4))
    if not args.no_kernel_events:
        plan.concurrent = False
        step([])  # capture the serialized graphs
        for _ in range(k_steps):
            if not args.no_flush:
                flush.zero_()
            ev = []
            step(ev)
            torch.cuda.synchronize(dev)
            for (side, kid, a, b) in ev:
                kernel_ms.setdefault((side, kid), []).append(a.elapsed_time(b))
        plan.concurrent = True
        plan.take_stats()
    total_ms = float(np.sum(step_ms))
    # per-rank half-step times, the solver kernels' serialized time and the
    # exchange volume (every rank sends its rows of the moving factor and, in
    # fp32 mode, its entries' maintained products to every peer)
    me = {"rank": rank, "f_half_ms": float(np.mean([h[0] for h in half_ms])),
          "w_half_ms": float(np.mean([h[1] for h in half_ms])),
          "kernel_ms_serialized": float(sum(np.sum(v) for v in kernel_ms.values())) / max(1, min(args.steps, 4))
          if kernel_ms else None}
    xb = {}
    for side_name in ("F", "W"):
        sp = plan.sides[side_name]
        mine = sp.owned_items(rank)
        ent = int(np.diff(sp.ptr_host)[mine].sum())
        per_peer = len(mine) * plan.rp * (4 if plan.fp32 else 8) + (ent * 8 if plan.fp32 else 0)
        xb[side_name] = {"items": int(len(mine)), "entries": ent, "bytes_sent": per_peer * (world - 1)}
    me["exchange_per_half_step"] = xb
    ranks_report = [me]
    if world > 1:
        ranks_report = [None] * world
        dist.all_gather_object(ranks_report, me)
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    updates = 2.0 * V.nnz * r
    value = updates / (ms_per_step * 1e-3)

    # dominant kernel and its roofline
    peak, peak_kind = peaks()
    if not kernel_ms:
        kernel_ms[("F", -2)] = [0.0]
    kinfo_default = (-2, 0, 0, 0)
    dom = max(kernel_ms.items(), key=lambda kv: np.sum(kv[1]))
    (dside, dkid), dms = dom
    sp = plan.sides[dside]
    start, count = next(((s, c) for k, s, c in sp.buckets if k == dkid), (0, 0))
    items = sp.items[start:start + count].cpu().numpy()
    dbytes = algorithmic_bytes(sp.ptr_host, items, r)
    avg_s = float(np.mean(dms)) * 1e-3
    achieved = dbytes / avg_s / 1e9 if avg_s > 0 else 0.0
    kinfo = next((k for k in plan.fast_kernels if k[0] == dkid), (dkid, 0, 0, 0))
    traffic = None
    prof = REPO / "profiles" / "traffic.json"
    if prof.exists():
        try:
            tr = json.loads(prof.read_text())
            traffic = tr.get(f"{spec.name}:{dside}:{dkid}")
        except ValueError:
            traffic = None
    it_bytes = iteration_bytes(spec.n, spec.m, V.nnz, r)
    # share of the dominant kernel within the serialized pass (one regime:
    # both numbers from the buckets launched one at a time)
    serial_ms = float(sum(np.sum(v) for (sd, k), v in kernel_ms.items() if k >= -1))
    kernel_table = {
        f"{s}:{k}": {"ms_per_step": float(np.sum(v)) / k_steps,
                     "lanes": next((x for x in plan.fast_kernels if x[0] == k), kinfo_default)[2]}
        for (s, k), v in sorted(kernel_ms.items(), key=lambda kv: -np.sum(kv[1])) if k >= -1
    }

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 arithmetic on f32 storage",
            "data": "synthetic",
            "outer_iters_per_sec": 1e3 / ms_per_step,
            "config": {"workload": spec.name, "n": spec.n, "m": spec.m, "nnz": V.nnz, "rank": r,
                       "reg": vars(spec.reg), "precision": precision,
                       "parallelism": f"dp{world} (subproblems split by modelled device time; exchange: "
                                      + ("fused peer stores over NVLink (CUDA IPC), NCCL barrier"
                                         if plan.fused_exchange else "NCCL all-gather" if world > 1 else "none")
                                      + ")",
                       "l2": "flushed (256 MB write) before every timed step; V + maintained products "
                             "(~2.2 GB per half-step) exceed L2",
                       "gen_seconds": round(gen_s, 1)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": f"{kernel_name(kinfo)}, side {dside}, {count} subproblems",
                         "kernel_share_of_serialized_step": float(np.sum(dms)) / serial_ms if serial_ms else None,
                         "algorithmic_bytes_per_launch": dbytes,
                         "step_achieved_gbs": it_bytes / (ms_per_step * 1e-3) / 1e9,
                         "step_frac": it_bytes / (ms_per_step * 1e-3) / 1e9 / peak,
                         "step_algorithmic_bytes": it_bytes,
                         # the other measured bound of the step: every entry and 4-coordinate
                         # chunk is one 16-byte cp.async lane request; a fully divergent warp instruction
                         # costs 33.4 L1/TEX cycles per SM (profiles/r05_gather_microbench.md)
                         "l1tex_gather_floor_ms": 2.0 * V.nnz * ((r + 3) // 4) / 32.0 * 33.4 / (148 * 1.965e9) * 1e3
                         / world,
                         "l1tex_gather_frac": (2.0 * V.nnz * ((r + 3) // 4) / 32.0 * 33.4 / (148 * 1.965e9) * 1e3
                                               / world) / ms_per_step},
            "kernels": kernel_table,
            "kernel_timing": "kernels/roofline: per-launch durations from an instrumented pass with the buckets "
                             "launched one at a time (continuing the same trajectory); the timed steps run "
                             "independent buckets concurrently on parallel streams",
            "solver_stats_per_step": {"newton_steps": st.inner_iters / args.steps,
                                      "newton_steps_per_visit": st.inner_iters / args.steps
                                      / ((spec.n + spec.m) * r),
                                      "cap_hits": st.cap_hits, "degenerate": st.degenerate},
            "gpu_launches": launch_count[0],
            "ranks": ranks_report,
            "step_ms": [round(x, 3) for x in step_ms],
            "step_kernel_ms": [round(x, 3) for x in step_kernel_ms] if step_kernel_ms else None,
            "clocks": clocks.summary(),
        }

    # e2e: public API from host buffers, rank-local.  The device-timed plan
    # is released first (its memory stays in torch's cache for the e2e plan,
    # as for any repeated call; nothing is handed back to the driver while a
    # peer rank may still map it)
    del plan
    gc.collect()  # closes this rank's peer mappings (fused exchange)
    if world > 1:
        dist.barrier()
    if not args.no_e2e and not args.profile:
        cfg = NmfConfig(rank=r, reg=reg, max_outer_iters=args.steps, rel_obj_tol=0.0, seed=spec.seed,
                        log_objectives=False, precision=precision, device=local, shard=world > 1)
        pair = FactorPair(DenseFactor(w0), DenseFactor(f0))
        # median of E2E_JOBS complete jobs: a single host-side stall (seen up
        # to ~1 s on the shared box hosts) would otherwise set the number
        job_s = []
        for _ in range(args.e2e_jobs or (1 if spec.name == "C5" else E2E_JOBS)):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            res = factorize(V, cfg, factors0=pair)
            torch.cuda.synchronize(dev)
            s = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([s], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                s = float(t.item())
            job_s.append(s)
        e2e_s = float(np.median(job_s))
        h2d = V.col_ptr.nbytes + V.row_idx.nbytes + V.values.nbytes + w0.nbytes + f0.nbytes
        d2h = w0.nbytes + f0.nbytes  # the downloaded factors have the initial factors' shapes
        if line is not None:
            line["e2e"] = {"value": updates * res.iterations_run / e2e_s, "unit": UNIT,
                           "h2d_bytes_per_step": int(h2d / max(1, res.iterations_run)),
                           "d2h_bytes_per_step": int(d2h / max(1, res.iterations_run)),
                           "seconds": e2e_s, "job_seconds": [round(x, 4) for x in job_s],
                           "iterations": res.iterations_run,
                           "includes": "upload of host CSC + factors, device CSR build and bucketing, "
                                       "iterations, download of both factors"}

    if line is not None and cpu_state is not None:
        import oracle

        threads = oracle.cores()
        w_st, f_st, ids_st = cpu_state
        vt = oracle.transpose_csc(V.n_rows, V.n_cols, V.col_ptr, V.row_idx, V.values)[:3]
        vals, times, nsv, sampled = [], [], [], 0
        for k in range(args.cpu_samples):
            v, t_iter, n_s, spv = cpu_reference_sample(V, w_st, f_st, spec, ids_st, args.cpu_seconds, threads,
                                                       pick_seed=1000 + k, vt=vt)
            vals.append(v)
            times.append(t_iter)
            nsv.append(spv)
            sampled += n_s
        line["cpu_baseline"] = {
            "value": float(np.mean(vals)), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"state of timed iteration {args.warmup + 1} (the GPU's factors after warm-up); "
                      f"{args.cpu_samples} stratified samples ({sampled // max(1, args.cpu_samples)} subproblems "
                      f"each, both sides, ~{args.cpu_seconds:.0f} s on {threads} threads) of the reference "
                      f"sweep_range port (dense maintained product), per-column thread CPU time extrapolated "
                      f"by bucket population / {threads} cores: {float(np.mean(times)):.1f} s per outer iteration",
            "iteration": args.warmup + 1,
            "newton_steps_per_visit": float(np.mean(nsv)),
            "gpu_newton_steps_per_visit": line["solver_stats_per_step"]["newton_steps_per_visit"],
            "step_values": [float(x) for x in vals]}
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(relaunch_distributed(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
