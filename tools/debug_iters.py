"""Per-half-step, per-bucket comparison of the fp32 kernels against the fp32
oracle over several iterations (GPU state reset to the oracle each half-step)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
from paper_1604_04026_b200 import synth  # noqa: E402
from paper_1604_04026_b200.plan import DevicePlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
spec = synth.CONFIGS[name].scaled(m=m)
V = synth.generate(spec)
w0, f0 = synth.initial_factors(spec)
r, rp = spec.rank, (spec.rank + 3) // 4 * 4
plan = DevicePlan(V, r, "fp32")
rng = np.random.default_rng(spec.seed)
ids = rng.permutation(r)
plan.set_factors(w0, f0, order=ids)
reg = spec.reg
for it in range(5):
    nxt = rng.permutation(r)
    for which, a, b in (("F", reg.alpha2, reg.beta2), ("W", reg.alpha1, reg.beta1)):
        side = plan.sides[which]
        fixed_name = "W" if which == "F" else "F"
        need = "csr" if which == "F" else "csc"
        if plan.t_current != need:
            plan._init_t(need)
        t0 = plan.t[need].cpu().numpy()[side.tmap.cpu().numpy()]
        fixed = plan.factors[fixed_name].cpu().numpy()
        mov = plan.factors[which].cpu().numpy()
        o_mov = plan.order[which]
        perm_in = np.argsort(o_mov)[ids]
        mov_vis = np.zeros_like(mov)
        mov_vis[:, :r] = mov[:, perm_in]
        sums = fixed.astype(np.float64).sum(axis=0)
        sums = plan.row_sums_pos(fixed_name, torch.zeros(rp, dtype=torch.float64, device=plan.dev)).cpu().numpy()
        mo, to = mov_vis.copy(), t0.copy()
        so = oracle.sweep_fp32(side.ptr.cpu().numpy(), side.idx.cpu().numpy(), side.val.cpu().numpy(), fixed, rp, r,
                               sums, mo, to, None, a, b)
        plan.half_step(which, ids, nxt if which == "W" else None, alpha=a, beta=b)
        sg = plan.take_stats()
        out_order = ids if which == "F" else nxt
        got = plan.factors[which].cpu().numpy()
        got_vis = got[:, np.argsort(out_order)[ids]]
        bad = np.any(got_vis != mo[:, :r], axis=1)
        sizes = np.diff(side.ptr_host)
        items = side.items.cpu().numpy()
        kid_of = np.zeros(side.n_mov, dtype=int)
        for kid, st, cnt in side.buckets:
            kid_of[items[st:st + cnt]] = kid
        tg = plan.t["csc" if which == "F" else "csr"].cpu().numpy()[: plan.nnz]
        tbad = np.abs(tg - to) > 1e-9 * np.abs(to)
        print(f"it{it+1} {which}: bad items {bad.sum()} / {len(bad)}; by kernel",
              dict(zip(*np.unique(kid_of[bad], return_counts=True))) if bad.any() else {},
              "t bad", int(tbad.sum()), "stats gpu", [sg.cap_hits, sg.inner_iters], "oracle", so.tolist(), flush=True)
        # reset the GPU state to the oracle's result to isolate the next half-step
        fixed_t = torch.from_numpy(np.ascontiguousarray(mo[:, np.argsort(ids)] if False else mo))
        reset = np.zeros_like(got)
        reset[:, np.argsort(out_order)[ids]] = mo[:, :r]
        plan.factors[which].copy_(torch.from_numpy(reset))
        plan.t["csc" if which == "F" else "csr"][: plan.nnz].copy_(torch.from_numpy(to))
    ids = nxt
