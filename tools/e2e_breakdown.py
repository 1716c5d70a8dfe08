"""Wall-clock breakdown of factorize() from host arrays (the bench's e2e leg)."""
import gc
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_04026_b200 import synth  # noqa: E402
from paper_1604_04026_b200.plan import DevicePlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
spec = synth.CONFIGS[name]
V = synth.generate(spec)
w0, f0 = synth.initial_factors(spec)
torch.zeros(1, device="cuda")
torch.cuda.synchronize()


_gc_t0 = [0.0]


def _gc_cb(phase, info):
    if phase == "start":
        _gc_t0[0] = time.perf_counter()
    elif time.perf_counter() - _gc_t0[0] > 0.005:
        print(f"    gc gen{info['generation']} collected {info['collected']} in "
              f"{1e3 * (time.perf_counter() - _gc_t0[0]):.1f} ms", flush=True)


if os.environ.get("E2E_GC_TRACE"):
    gc.callbacks.append(_gc_cb)


def tick(label, t0):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"{label:28s} {1e3 * (t1 - t0):8.1f} ms", flush=True)
    return t1


for rep in range(2):
    print(f"--- run {rep}")
    t = t0 = time.perf_counter()
    plan = DevicePlan(V, spec.rank, spec.precision)
    t = tick("DevicePlan (upload, CSR, buckets)", t)
    rng = np.random.default_rng(spec.seed)
    ids = rng.permutation(spec.rank)
    plan.set_factors(w0, f0, order=ids)
    t = tick("set_factors", t)
    reg = spec.reg
    for it in range(1, iters + 1):
        nxt = rng.permutation(spec.rank)
        plan.half_step("F", ids, alpha=reg.alpha2, beta=reg.beta2, iteration=it)
        plan.half_step("W", ids, nxt, alpha=reg.alpha1, beta=reg.beta1, iteration=it)
        ids = nxt
        t = tick(f"iteration {it}", t)
        plan.objective(reg.alpha1, reg.alpha2, reg.beta1, reg.beta2)
        t = tick("  objective", t)
    plan.get_factors()
    t = tick("get_factors", t)
    print(f"total {1e3 * (t - t0):.1f} ms")
    del plan  # as factorize: the next job's plan reuses this one's cached memory
    gc.collect()
