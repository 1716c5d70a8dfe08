import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle
from paper_1604_04026_b200 import synth
from paper_1604_04026_b200.plan import DevicePlan
from test_gpu_fast import _compare_half_step
spec = synth.CONFIGS['C4'].scaled(m=8000)
V = synth.generate(spec); w0, f0 = synth.initial_factors(spec)
plan = DevicePlan(V, spec.rank, "fp32")
ids = np.random.default_rng(0).permutation(spec.rank)
plan.set_factors(w0, f0, order=ids)
mg, mo, tg, to, sg, so = _compare_half_step(plan, "F", ids, spec.reg.alpha2, spec.reg.beta2)
print("F exact", np.mean(mg == mo))
mg, mo, tg, to, sg, so = _compare_half_step(plan, "W", ids, spec.reg.alpha1, spec.reg.beta1)
rows_bad = np.where(np.any(mg != mo, axis=1))[0]
sz = np.diff(plan.sides["W"].ptr_host)
print("W rows differing", len(rows_bad), "of", len(sz), "exact", np.mean(mg == mo))
caps = [c for _, c, _, _ in plan.fast_kernels]
b_all = np.searchsorted(np.array([c if c > 0 else 1 << 40 for c in caps]), sz)
b_bad = b_all[rows_bad]
for k in sorted(set(b_all.tolist())):
    print(f"  bucket {k} cap {caps[k]}: rows {np.sum(b_all == k)} bad {np.sum(b_bad == k)}")
print("stats gpu", sg, "oracle", so)
# first bad row details
if len(rows_bad):
    i = rows_bad[0]
    print("row", i, "size", sz[i], "gpu", mg[i, :8], "orc", mo[i, :8])
