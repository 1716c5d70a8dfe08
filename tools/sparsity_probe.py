"""Zero structure of the fixed factors at steady state, weighted by entries."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from gpu_drivers import gpu_drive  # noqa: E402
from paper_1604_04026_b200 import synth  # noqa: E402

spec = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
V = synth.generate(spec)
w0, f0 = synth.initial_factors(spec)
res = gpu_drive(V, w0, f0, spec.rank, spec.reg, int(sys.argv[2]) if len(sys.argv) > 2 else 8, spec.seed,
                precision="fp32", log=False, hashes=False)
w, f = res["w"], res["f"]
wnz = (w != 0).sum(axis=0)  # per feature
fnz = (f != 0).sum(axis=0)  # per document
cols = np.repeat(np.arange(V.n_cols), np.diff(V.col_ptr))
ew = wnz[V.row_idx]  # F-side entries: fixed row = W row of the feature
ef = fnz[cols]       # W-side entries: fixed row = F row of the document
for name, e, fac in (("F-side (fixed W)", ew, wnz), ("W-side (fixed F)", ef, fnz)):
    print(f"{name}: items zero-row {np.mean(fac == 0):.3f}; entries with zero fixed row {np.mean(e == 0):.3f}; "
          f"mean nnz of fixed row per entry {e.mean():.2f}/{spec.rank}; p50 {np.median(e)}, p90 {np.percentile(e, 90)}")
xw = (w != 0).sum(axis=0); xf = (f != 0).sum(axis=0)
print("moving-side nonzeros per item: W", xw.mean(), "F", xf.mean())
