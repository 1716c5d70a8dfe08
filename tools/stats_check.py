"""Per-iteration solver statistics of the device plan (diagnostics)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from gpu_drivers import gpu_drive  # noqa: E402
from paper_1604_04026_b200 import synth  # noqa: E402

name = sys.argv[1]
m = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "full" else None
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 6
spec = synth.CONFIGS[name]
if m:
    spec = spec.scaled(m=m)
V = synth.generate(spec)
w0, f0 = synth.initial_factors(spec)
res = gpu_drive(V, w0, f0, spec.rank, spec.reg, iters, spec.seed, precision=spec.precision, hashes=False)
for i, s in enumerate(res["stats"]):
    print(i + 1, list(map(int, s)), res["kl"][i], flush=True)
print("sparsity W, F:", res["plan"].objective()[2:])
