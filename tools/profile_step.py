"""Host/device time breakdown of one outer iteration (diagnostics)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_04026_b200 import synth  # noqa: E402
from paper_1604_04026_b200.plan import DevicePlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = synth.CONFIGS[name]
V = synth.generate(spec)
w0, f0 = synth.initial_factors(spec)
plan = DevicePlan(V, spec.rank, spec.precision)
rng = np.random.default_rng(spec.seed)
ids = rng.permutation(spec.rank)
plan.set_factors(w0, f0, order=ids)
reg = spec.reg


def step():
    global ids
    nxt = rng.permutation(spec.rank)
    plan.half_step("F", ids, alpha=reg.alpha2, beta=reg.beta2)
    plan.half_step("W", ids, nxt, alpha=reg.alpha1, beta=reg.beta1)
    ids = nxt


for _ in range(2):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    step()
torch.cuda.synchronize()
pr.disable()
print(f"{steps} steps wall {1e3 * (time.perf_counter() - t0) / steps:.1f} ms/step")
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
