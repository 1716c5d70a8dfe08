"""Kernel-safety workload: every solver kernel family run on the CHECKED
build of the library, results compared with the CPU oracle, and the
device-side check counters required to stay at zero.

    python tools/build_variant.py checked -DKLNMF_CHECKED
    KLNMF_LIB=_variants/checked/libklnmf.so python tools/checked_run.py [repeats]

The checked build (csrc/solve_fast.cu, KLNMF_CHECKED) bounds-checks every
gather offset, item id, maintained-product index, spill record and result
store, and asserts the inter-CTA protocols: a cooperative reduction slot is
never overwritten before every reader has read it (tags never run ahead),
the arrival counter never runs two rounds ahead, and every cluster inbox
round holds exactly the current round's partial from every peer (a
(round, sender) tag travels with each st.async push).  compute-sanitizer is
not available on this GPU pool, so these checks stand in for memcheck /
racecheck / synccheck on the hand-written protocols.

Families: solve_exact_kernel (fp64 mode), every warp / block / cluster
capacity of the fp32 ladder (one column per bucket), the cooperative
long-row kernel including its spill path (a column longer than the whole
GPU's on-chip capacity), in the shared and the counter coordinate order,
plus the objective, row-sum, transpose and layout kernels the plan runs.
Small ranks keep the instrumented run short.
"""
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

import oracle  # noqa: E402  (test infrastructure: the checker)


def ladder_matrix(rng, n, sizes):
    import paper_1604_04026_b200 as kb

    rows, cols = [], []
    for j, s in enumerate(sizes):
        rows.append(np.sort(rng.choice(n, size=s, replace=False)))
        cols.append(np.full(s, j))
    rows = np.concatenate(rows)
    vals = rng.integers(1, 6, size=rows.shape[0]).astype(np.float64)
    return kb.SparseMatrix.from_coo(n, len(sizes), rows, np.concatenate(cols), vals)


def fp32_pass(V, r, order, rng, label):
    import torch

    from paper_1604_04026_b200.plan import DevicePlan
    from test_gpu_fast import _check, _compare_half_step

    w0 = rng.random((r, V.n_rows)).astype(np.float32).astype(np.float64)
    w0[rng.random(w0.shape) < 0.5] = 0.0
    f0 = rng.random((r, V.n_cols)).astype(np.float32).astype(np.float64)
    plan = DevicePlan(V, r, "fp32", order=order, order_seed=11)
    plan.use_graphs = False
    ids = rng.permutation(r)
    plan.set_factors(w0, f0, order=ids)
    kid = plan._stream_kernel_id()
    used = sorted({k for s in plan.sides.values() for k, _, c in s.buckets if c > 0})
    it = 3 if order == "counter" else None
    for which in ("F", "W"):
        mg, mo, tg, to, _, _ = _compare_half_step(plan, which, ids, 0.01, 0.05, iteration=it)
        _check(mg, mo, tg, to, f"{label} {which}")
    plan.objective(0.01, 0.01, 0.05, 0.05)
    torch.cuda.synchronize()
    print(f"{label}: order={order} kernels {used} (coop id {kid}) ok", flush=True)
    del plan
    torch.cuda.empty_cache()


def read_checks(reset=False):
    import ctypes

    from paper_1604_04026_b200 import _lib

    lib = _lib.load()
    if not hasattr(lib, "klnmf_debug_checks"):
        raise SystemExit("not the checked build: set KLNMF_LIB=_variants/checked/libklnmf.so")
    out = (ctypes.c_ulonglong * 2)()
    if lib.klnmf_debug_checks(out, int(reset)) != 0:
        raise RuntimeError("klnmf_debug_checks failed")
    return int(out[0]), int(out[1])


def main():
    import torch

    from paper_1604_04026_b200 import synth
    from paper_1604_04026_b200.plan import DevicePlan

    torch.cuda.set_device(0)
    t0 = time.time()
    repeats = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    read_checks(reset=True)
    for rep in range(repeats):
        workload(rep)
        n, code = read_checks()
        print(f"repeat {rep}: check violations {n} (first code {code})", flush=True)
        assert n == 0, (n, code)
    # full-size W side of scaled C4 through the cluster and cooperative kernels
    spec = synth.CONFIGS["C4"].scaled(m=100000)
    V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec)
    plan = DevicePlan(V, spec.rank, "fp32")
    ids = np.random.default_rng(2).permutation(spec.rank)
    plan.set_factors(w0, f0, order=ids)
    for it in range(3):
        plan.half_step("F", ids, alpha=0.01, beta=0.0)
        plan.half_step("W", ids, alpha=0.01, beta=0.0)
    torch.cuda.synchronize()
    n, code = read_checks()
    print(f"scaled C4, 3 iterations: check violations {n} (first code {code})", flush=True)
    assert n == 0, (n, code)
    print(f"checked workload ok in {time.time() - t0:.1f} s: 0 violations", flush=True)


def workload(rep):
    import torch

    from paper_1604_04026_b200 import _lib, synth
    from paper_1604_04026_b200.plan import DevicePlan

    rng = np.random.default_rng(2024 + rep)

    # fp64 exact mode (solve_exact_kernel, exact row sums, layout, objective)
    spec = synth.CONFIGS["C1"].scaled(m=200, n=400)
    V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec)
    ids = np.random.default_rng(1).permutation(spec.rank)
    plan = DevicePlan(V, spec.rank, "fp64")
    plan.set_factors(w0, f0, order=ids)
    plan.half_step("F", ids)
    plan.half_step("W", ids)
    wg, fg = plan.get_factors()
    plan.objective()
    w, f = w0.copy(), f0.copy()
    oracle.sweep(V.col_ptr, V.row_idx, V.values, w, oracle.row_sums(w), f, ids, 0.0, 0.0)
    pt, rt, vt, _ = oracle.transpose_csc(V.n_rows, V.n_cols, V.col_ptr, V.row_idx, V.values)
    oracle.sweep(pt, rt, vt, f, oracle.row_sums(f), w, ids, 0.0, 0.0)
    assert np.array_equal(fg, f) and np.array_equal(wg, w)
    print("fp64 exact: ok", flush=True)
    del plan

    # fp32: one column per capacity of the ladder (warp, block, cluster, coop)
    caps = [c for _, c, _, _ in _lib.fast_kernels(8) if c > 0]
    sizes = [max(1, c - c // 7) for c in caps] + [caps[-1] + 5000]
    V = ladder_matrix(rng, caps[-1] + 20000, sizes)
    for order in ("shared", "counter"):
        fp32_pass(V, 8, order, rng, "fp32 ladder")

    # fp32 spill path: a column beyond every CTA's on-chip capacity together
    per_cta, n_ctas, _ = _lib.coop_info(8)
    cap = per_cta * n_ctas
    V = ladder_matrix(rng, cap + cap // 8 + 1000, [cap + cap // 8, 70000, 3])
    fp32_pass(V, 7, "shared", rng, "fp32 spill")
    fp32_pass(V, 7, "counter", rng, "fp32 spill")


if __name__ == "__main__":
    main()
