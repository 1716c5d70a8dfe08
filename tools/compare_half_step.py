"""One F and one W half-step of the fp32 kernels against the fp32 oracle from
the same state, with the differing subproblems grouped by nnz bucket (i.e. by
kernel).  Usage: python tools/compare_half_step.py [config] [m]"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_1604_04026_b200 import synth  # noqa: E402
from paper_1604_04026_b200.plan import DevicePlan  # noqa: E402
from test_gpu_fast import _compare_half_step  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 8000
spec = synth.CONFIGS[name].scaled(m=m)
V = synth.generate(spec)
w0, f0 = synth.initial_factors(spec)
plan = DevicePlan(V, spec.rank, "fp32")
ids = np.random.default_rng(0).permutation(spec.rank)
plan.set_factors(w0, f0, order=ids)
caps = np.array([c if c > 0 else 1 << 40 for _, c, _, _ in plan.fast_kernels])
for which, a, b in (("F", spec.reg.alpha2, spec.reg.beta2), ("W", spec.reg.alpha1, spec.reg.beta1)):
    mg, mo, tg, to, sg, so = _compare_half_step(plan, which, ids, a, b)
    bad = np.where(np.any(mg != mo, axis=1))[0]
    sz = np.diff(plan.sides[which].ptr_host)
    bucket = np.searchsorted(caps, sz)
    print(f"{which}: exact {np.mean(mg == mo):.6f}; subproblems differing {len(bad)} of {len(sz)}; "
          f"stats gpu {sg} oracle {so.tolist()}")
    for k in sorted(set(bucket.tolist())):
        nb = int(np.sum(bucket[bad] == k))
        if nb:
            print(f"  kernel {k} (capacity {caps[k]}): {nb} of {int(np.sum(bucket == k))} differ")
