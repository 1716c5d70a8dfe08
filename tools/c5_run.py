"""C5 (141,043 x 8.2M, ~480M nonzeros) end to end on one GPU: device-side
generation, plan build, U(0,1) factors drawn on the device, timed
iterations.  Usage: python tools/c5_run.py [iters] [config]"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_04026_b200 import synth  # noqa: E402
from paper_1604_04026_b200.plan import DevicePlan  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
name = sys.argv[2] if len(sys.argv) > 2 else "C5"
spec = synth.CONFIGS[name]
torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
out = {"config": name}
t0 = time.perf_counter()
V = synth.generate_device(spec)
torch.cuda.synchronize()
out["generate_s"] = time.perf_counter() - t0
out["nnz"] = V.nnz
t0 = time.perf_counter()
plan = DevicePlan(V, spec.rank, spec.precision)
torch.cuda.synchronize()
out["plan_s"] = time.perf_counter() - t0
del V
r = spec.rank
g = torch.Generator(device="cuda").manual_seed(spec.seed)
ids = np.random.default_rng(spec.seed).permutation(r)
for fname, n_items in (("W", plan.n), ("F", plan.m)):  # U(0,1), fp32, visit order == storage order
    plan.factors[fname][:, :r] = torch.rand(n_items, r, generator=g, device="cuda", dtype=plan.factors[fname].dtype)
    plan.order[fname] = ids.copy()
plan.t_current = None
out["peak_gb_after_plan"] = torch.cuda.max_memory_allocated() / 1e9
rng = np.random.default_rng(spec.seed + 1)
reg = spec.reg
ms, kls = [], []
kernels = {}
for it in range(1, iters + 1):
    nxt = rng.permutation(r)
    ev = [] if it == iters else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.half_step("F", ids, alpha=reg.alpha2, beta=reg.beta2, events=ev)
    plan.half_step("W", ids, nxt, alpha=reg.alpha1, beta=reg.beta1, events=ev)
    e1.record()
    torch.cuda.synchronize()
    for side, kid, a, b in ev or []:
        kernels[f"{side}:{kid}"] = round(a.elapsed_time(b), 3)
    ids = nxt
    ms.append(e0.elapsed_time(e1))
    kls.append(plan.objective(reg.alpha1, reg.alpha2, reg.beta1, reg.beta2)[1])
out["ms_per_iteration"] = ms
out["last_iteration_kernels_ms"] = dict(sorted(kernels.items(), key=lambda kv: -kv[1]))
out["total_objective"] = kls
out["updates_per_s_last"] = 2.0 * plan.nnz * r / (ms[-1] * 1e-3)
out["peak_gb"] = torch.cuda.max_memory_allocated() / 1e9
st = plan.take_stats()
out["newton_steps_per_visit"] = st.inner_iters / iters / ((plan.n + plan.m) * r)
print(json.dumps(out))
