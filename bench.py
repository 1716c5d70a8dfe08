#!/usr/bin/env python
"""Benchmark of the SRCD hot path (one outer iteration = F half-step + W half-step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Default workload: BASELINE.json config C4 (102,660 x 300,000, ~68M nnz,
r=100, alpha1=alpha2=0.01, fp32 storage / fp64 arithmetic) -- the config the
metric "outer iterations/sec and nnz*r coordinate updates/sec at 1/2/4/8
B200" is specified on.  Synthetic data of that shape (synth.py), U(0,1)
initial factors rounded to fp32.  Under torchrun (N>1) each rank owns an
nnz-balanced range of subproblems per side and the updated factor rows are
all-gathered over NCCL after each half-step (strong scaling: fixed C4).

value      nnz*r coordinate updates/s = 2*nnz*r / step time, data resident in HBM,
           device time (CUDA events, max over ranks), L2 flushed between steps.
e2e        the same metric through the public API (factorize with HOST numpy
           inputs: upload, device CSR build, bucketing, K iterations, download);
           the median of E2E_JOBS (5) complete jobs, each job's seconds listed.
roofline   the dominant solver kernel: SURVEY.md §8(d) algorithmic bytes of the
           launch / its CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the reference algorithm (oracle port of _kernels.sweep_range, dense
           maintained product as in the reference) on the host cores, on a
           stratified sample of subproblems, extrapolated to a full iteration.
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
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="target CPU-baseline sample budget")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu legs)")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-kernel-events", action="store_true")
    return ap.parse_args()


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
def cpu_reference_sample(V, w0, f0, spec, seconds: float, threads: int):
    """Time the reference algorithm (oracle port of _kernels.sweep_range with
    the reference's dense length-n maintained product) on a stratified sample
    of subproblems per nnz bucket and side, using `threads` host threads;
    extrapolate to one outer iteration.  Returns (updates/s, sample text)."""
    import oracle

    oracle.build()
    r = spec.rank
    reg = spec.reg
    pt, rt, vt, _ = oracle.transpose_csc(V.n_rows, V.n_cols, V.col_ptr, V.row_idx, V.values)
    sides = [("F", V.col_ptr, V.row_idx, V.values, w0, f0, reg.alpha2, reg.beta2),
             ("W", pt, rt, vt, f0, w0, reg.alpha1, reg.beta1)]
    ids = np.random.default_rng(spec.seed).permutation(r)
    edges = [0, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 1 << 62]
    rng = np.random.default_rng(123)
    total_time = 0.0
    sampled = 0
    per_side_budget = seconds / 2
    for name, ptr, idx, val, fixed, moving, a, b in sides:
        sizes = np.diff(ptr)
        sums = oracle.row_sums(fixed)
        buckets = [np.nonzero((sizes > lo) & (sizes <= hi))[0] for lo, hi in zip(edges[:-1], edges[1:])]
        buckets = [np.nonzero(sizes == 0)[0]] + buckets
        # calibrate: one column of the median bucket
        est = []
        for members in buckets:
            if len(members) == 0:
                est.append(0.0)
                continue
            j = int(members[len(members) // 2])
            t0 = time.perf_counter()
            _run_cols(oracle, ptr, idx, val, fixed, sums, moving, [j], ids, a, b, 1)
            est.append(time.perf_counter() - t0)
        side_time = 0.0
        for members, e in zip(buckets, est):
            if len(members) == 0:
                continue
            # sample count: all members of small buckets, else what fits the budget share
            share = per_side_budget / max(1, sum(1 for q in buckets if len(q)))
            k = int(min(len(members), max(threads, share * threads / max(e, 1e-6))))
            pick = np.sort(rng.choice(members, size=k, replace=False))
            t0 = time.perf_counter()
            _run_cols(oracle, ptr, idx, val, fixed, sums, moving, pick, ids, a, b, threads)
            dt = time.perf_counter() - t0
            side_time += dt * len(members) / k
            sampled += k
        total_time += side_time
    updates = 2.0 * V.nnz * r
    return updates / total_time, total_time, sampled


def _run_cols(oracle, ptr, idx, val, fixed, sums, moving, cols, ids, a, b, threads):
    """sweep_range over an explicit column subset (sub-CSC), threads over columns."""
    cols = np.asarray(cols, dtype=np.int64)
    sizes = ptr[cols + 1] - ptr[cols]
    sub_ptr = np.zeros(len(cols) + 1, dtype=np.int64)
    np.cumsum(sizes, out=sub_ptr[1:])
    sel = np.concatenate([np.arange(ptr[j], ptr[j + 1]) for j in cols]) if len(cols) else np.zeros(0, np.int64)
    mov = np.ascontiguousarray(moving[:, cols])
    oracle.sweep(sub_ptr, idx[sel], val[sel], fixed, sums, mov, ids, a, b, n_workers=threads, variant="dense")


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


def load_config(name):
    from paper_1604_04026_b200 import synth

    spec = synth.CONFIGS[name]
    t0 = time.perf_counter()
    V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec)
    return spec, V, w0, f0, time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the reference algorithm on the host CPU (rank 0 only)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    spec, V, w0, f0, _ = load_config(args.config)
    threads = oracle.cores()
    per_step = max(2.0, min(args.cpu_seconds, 60.0) / max(1, args.steps + args.warmup) * 2)
    for _ in range(args.warmup):
        cpu_reference_sample(V, w0, f0, spec, per_step, threads)
    vals, times = [], []
    for _ in range(args.steps):
        v, t_iter, sampled = cpu_reference_sample(V, w0, f0, spec, per_step, threads)
        vals.append(v)
        times.append(t_iter)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(times)) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "outer_iters_per_sec": 1.0 / float(np.mean(times)),
        "config": {"workload": spec.name, "n": spec.n, "m": spec.m, "nnz": V.nnz, "rank": spec.rank,
                   "reg": vars(spec.reg)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"stratified sample ({sampled} subproblems/step, both sides) of the "
                                   f"reference sweep_range port (dense maintained product), extrapolated "
                                   f"to a full outer iteration"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1604_04026_b200 import NmfConfig, factorize, FactorPair, DenseFactor
    from paper_1604_04026_b200.plan import DevicePlan

    world, rank, local = setup_dist(args)
    group = dist.group.WORLD if world > 1 else None
    spec, V, w0, f0, gen_s = load_config(args.config)
    precision = spec.precision
    dev = torch.device("cuda", local)
    plan = DevicePlan(V, spec.rank, precision, local, group)
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

    def step(events):
        nonlocal ids
        ids_next = rng.permutation(r).astype(np.int64)
        plan.half_step("F", ids, alpha=reg.alpha2, beta=reg.beta2, events=events)
        plan.half_step("W", ids, ids_next, alpha=reg.alpha1, beta=reg.beta1, events=events)
        ids = ids_next

    for _ in range(args.warmup):  # same (instrumented or not) graphs as the timed steps
        step(None if args.no_kernel_events else [])
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    plan.take_stats()
    step_ms = []
    step_kernel_ms = []
    with ClockSampler(-1 if args.no_clocks else local) as clocks:
        for _ in range(args.steps):
            if not args.no_flush:
                flush.zero_()
            ev = None if args.no_kernel_events else []
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            # ~1 ms device sleep outside [e0, e1]: the host enqueues the whole
            # step before the device reaches e0, so host latency after the
            # per-step synchronize is not counted as device time
            torch.cuda._sleep(2_000_000)
            e0.record(stream)
            step(ev)
            e1.record(stream)
            # per-kernel events are CUDA-graph nodes re-recorded by each replay:
            # read them before the next step (device time is unaffected)
            torch.cuda.synchronize(dev)
            step_ms.append(e0.elapsed_time(e1))
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
    if world > 1:
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
                       "parallelism": f"dp{world} (nnz-balanced subproblem ranges, NCCL all-gather)",
                       "l2": "flushed (256 MB write) before every timed step; V + maintained products "
                             "(~2.2 GB per half-step) exceed L2",
                       "gen_seconds": round(gen_s, 1)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": f"solve_fast L={kinfo[2]} NPL={kinfo[3]} side={dside}",
                         "kernel_share_of_step": float(np.sum(dms)) / k_steps / ms_per_step if world == 1 else None,
                         "algorithmic_bytes_per_launch": dbytes,
                         "step_achieved_gbs": it_bytes / (ms_per_step * 1e-3) / 1e9,
                         "step_frac": it_bytes / (ms_per_step * 1e-3) / 1e9 / peak,
                         "step_algorithmic_bytes": it_bytes},
            "kernels": kernel_table,
            "kernel_timing": "kernels/roofline: per-launch durations from an instrumented pass with the buckets "
                             "launched one at a time (continuing the same trajectory); the timed steps run "
                             "independent buckets concurrently on parallel streams",
            "solver_stats_per_step": {"newton_steps": st.inner_iters / args.steps,
                                      "newton_steps_per_visit": st.inner_iters / args.steps
                                      / ((spec.n + spec.m) * r),
                                      "cap_hits": st.cap_hits, "degenerate": st.degenerate},
            "gpu_launches": launch_count[0],
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
        for _ in range(E2E_JOBS):
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

    if line is not None and not args.no_cpu and not args.profile and world == 1:
        import oracle

        threads = oracle.cores()
        v, t_iter, sampled = cpu_reference_sample(V, w0, f0, spec, args.cpu_seconds, threads)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{sampled} subproblems (stratified by nnz bucket, both sides) of "
                                          f"the reference sweep_range port with its dense maintained "
                                          f"product, extrapolated: {t_iter:.1f} s per outer iteration"}
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
