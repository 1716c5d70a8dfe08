"""Compare GPU vs fp32-oracle solver stats on C4-scaled iteration 1, F side,
and bisect to a single column whose stats differ."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import paper_1604_04026_b200 as kb  # noqa: E402
from paper_1604_04026_b200 import synth  # noqa: E402
from paper_1604_04026_b200.plan import DevicePlan  # noqa: E402

spec = synth.CONFIGS["C4"].scaled(m=int(sys.argv[1]) if len(sys.argv) > 1 else 3000)
V = synth.generate(spec)
w0, f0 = synth.initial_factors(spec)
ids = np.random.default_rng(spec.seed).permutation(spec.rank)


def run(cols):
    cols = np.asarray(cols)
    sizes = V.col_ptr[cols + 1] - V.col_ptr[cols]
    ptr = np.zeros(len(cols) + 1, dtype=np.int64)
    np.cumsum(sizes, out=ptr[1:])
    sel = np.concatenate([np.arange(V.col_ptr[j], V.col_ptr[j + 1]) for j in cols])
    Vs = kb.SparseMatrix(V.n_rows, len(cols), ptr, V.row_idx[sel], V.values[sel])
    plan = DevicePlan(Vs, spec.rank, "fp32")
    plan.set_factors(w0, f0[:, cols], order=ids)
    side = plan.sides["F"]
    need = "csr"
    plan._init_t(need)
    t0 = plan.t[need].cpu().numpy()[side.tmap.cpu().numpy()]
    fixed = plan.factors["W"].cpu().numpy()
    mov = plan.factors["F"].cpu().numpy()
    sums = plan.row_sums_pos("W", torch.zeros(plan.rp, dtype=torch.float64, device=plan.dev)).cpu().numpy()
    mo, to = mov.copy(), t0.copy()
    so = oracle.sweep_fp32(side.ptr.cpu().numpy(), side.idx.cpu().numpy(), side.val.cpu().numpy(), fixed,
                           plan.rp, plan.r, sums, mo, to, None, spec.reg.alpha2, spec.reg.beta2)
    plan.half_step("F", ids, alpha=spec.reg.alpha2, beta=spec.reg.beta2)
    sg = plan.take_stats()
    mg = plan.factors["F"].cpu().numpy()
    return [sg.cap_hits, sg.degenerate, sg.inner_iters, sg.passes], so.tolist(), np.array_equal(mg, mo)


cols = np.arange(spec.m)
g, o, eq = run(cols)
print("all cols gpu", g, "oracle", o, "factors equal", eq, flush=True)
while len(cols) > 1 and g[2] != o[2]:
    half = cols[: len(cols) // 2]
    g2, o2, _ = run(half)
    if g2[2] != o2[2]:
        cols = half
        g, o = g2, o2
    else:
        cols = cols[len(cols) // 2:]
        g, o, _ = run(cols)
    print(len(cols), g, o, flush=True)
print("culprit columns", cols[:10], "sizes", [int(V.col_ptr[j + 1] - V.col_ptr[j]) for j in cols[:10]])
