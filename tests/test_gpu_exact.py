"""fp64 exact mode on the GPU vs the reference (golden fixtures) and the
pinned oracle: bit-identical factors, stats and trajectories."""

import numpy as np
import pytest

import oracle
from conftest import load_cases, load_golden
from gpu_drivers import gpu_drive, sha

pytestmark = pytest.mark.gpu

SWEEP = load_cases("sweep_small.npz")


@pytest.mark.parametrize("case", range(len(SWEEP)))
def test_sweep_drop_in_bit_exact(cuda_ok, case):
    """klnmf_sweep_range (host drop-in) reproduces _kernels.sweep_range."""
    import paper_1604_04026_b200 as kb

    c = SWEEP[case]
    n_fix = int(c["n_fix"])
    n_mov = c["moving_in"].shape[1]
    V = kb.SparseMatrix(n_fix, n_mov, c["col_ptr"], c["row_idx"], c["values"])
    moving = kb.DenseFactor(c["moving_in"].copy())
    tol = kb.Tolerances(float(c["eps_grad"]), float(c["eps_x"]), float(c["eps_div"]), int(c["inner_cap"]))
    st = kb.sweep(V, kb.DenseFactor(c["at"]), moving, c["sum_a"], c["ids"], float(c["alpha"]),
                  float(c["beta"]), tol=tol)
    assert np.array_equal(moving.values, c["moving_out"])
    assert [st.cap_hits, st.degenerate, st.inner_iters, st.passes] == list(c["stats"])


@pytest.mark.parametrize("n_workers", [3, 8])
@pytest.mark.parametrize("case", range(0, len(SWEEP), 5))
def test_sweep_drop_in_concurrent_workers(cuda_ok, case, n_workers):
    """The reference drives sweep_range from a thread pool, one disjoint
    column chunk per worker (solver.py:197-214); through the drop-in the
    concurrent calls must each touch only their own columns, so the result
    is bit-identical to the reference for any worker count."""
    import paper_1604_04026_b200 as kb

    c = SWEEP[case]
    n_fix = int(c["n_fix"])
    n_mov = c["moving_in"].shape[1]
    V = kb.SparseMatrix(n_fix, n_mov, c["col_ptr"], c["row_idx"], c["values"])
    moving = kb.DenseFactor(c["moving_in"].copy())
    tol = kb.Tolerances(float(c["eps_grad"]), float(c["eps_x"]), float(c["eps_div"]), int(c["inner_cap"]))
    st = kb.sweep(V, kb.DenseFactor(c["at"]), moving, c["sum_a"], c["ids"], float(c["alpha"]),
                  float(c["beta"]), tol=tol, n_workers=n_workers)
    assert np.array_equal(moving.values, c["moving_out"])
    assert [st.cap_hits, st.degenerate, st.inner_iters, st.passes] == list(c["stats"])


def test_sweep_range_writes_only_its_columns(cuda_ok):
    """klnmf_sweep_range(j_lo, j_hi) leaves every other column of `moving`
    untouched, even if the host copy changes during the call's lifetime
    (another worker writing its chunk)."""
    from paper_1604_04026_b200 import _lib

    c = next(c for c in SWEEP if c["moving_in"].shape[1] >= 6 and c["col_ptr"][-1] > 0)
    n_fix = int(c["n_fix"])
    mv = c["moving_in"].copy()
    r, n_mov = mv.shape
    lo, hi = n_mov // 3, 2 * n_mov // 3
    sentinel = np.full_like(mv, np.nan)
    sentinel[:, lo:hi] = mv[:, lo:hi]
    stats = np.zeros(4, dtype=np.int64)
    ids = np.ascontiguousarray(c["ids"], dtype=np.int64)
    args = [np.ascontiguousarray(c[k]) for k in ("col_ptr", "row_idx", "values", "at", "sum_a")]
    _lib.call("klnmf_sweep_range", *[a.ctypes.data for a in args], sentinel.ctypes.data, lo, hi, ids.ctypes.data,
              float(c["alpha"]), float(c["beta"]), float(c["eps_grad"]), float(c["eps_x"]), float(c["eps_div"]),
              int(c["inner_cap"]), r, n_fix, n_mov, stats.ctypes.data)
    assert np.isnan(sentinel[:, :lo]).all() and np.isnan(sentinel[:, hi:]).all()
    assert np.array_equal(sentinel[:, lo:hi], c["moving_out"][:, lo:hi])


@pytest.mark.parametrize("case", range(len(load_cases("objective_small.npz"))))
def test_full_objective(cuda_ok, case):
    import paper_1604_04026_b200 as kb

    c = load_cases("objective_small.npz")[case]
    n = int(c["n_rows"])
    m = c["f"].shape[1]
    V = kb.SparseMatrix(n, m, c["col_ptr"], c["row_idx"], c["values"])
    kl, total = kb.full_objective(V, kb.DenseFactor(c["w"]), kb.DenseFactor(c["f"]),
                                  kb.RegConfig(*map(float, c["reg"])), eps_div=float(c["eps_div"]))
    # GPU log differs from libm by <= 1 ulp and the entry sum is a fixed tree
    assert kl == pytest.approx(float(c["kl"]), rel=1e-12, abs=1e-12)
    assert total == pytest.approx(float(c["total"]), rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("case", range(len(load_cases("row_sums.npz"))))
def test_row_sums_drop_in_bit_exact(cuda_ok, case):
    from paper_1604_04026_b200 import _lib

    c = load_cases("row_sums.npz")[case]
    x = np.ascontiguousarray(c["x"])
    out = np.zeros(x.shape[0])
    _lib.call("klnmf_row_sums", x.ctypes.data, x.shape[0], x.shape[1], out.ctypes.data)
    assert np.array_equal(out, c["sums"])


def _c1():
    from paper_1604_04026_b200 import synth

    spec = synth.CONFIGS["C1"]
    V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec)
    return spec, V, w0, f0


def test_c1_trajectory_bit_exact(cuda_ok):
    """30 outer iterations on C1 (fp64 oracle mode): every iterate equals the
    reference's bit for bit (factor hashes), stats equal, objective within
    1e-12 (GPU log + tree sum)."""
    g = load_golden("c1_trajectory.npz")
    spec, V, w0, f0 = _c1()
    res = gpu_drive(V, w0, f0, spec.rank, spec.reg, 30, spec.seed, precision="fp64")
    assert np.array_equal(res["ids"], g["ids"])
    assert list(res["w_sha"]) == list(g["w_sha"])
    assert list(res["f_sha"]) == list(g["f_sha"])
    assert np.array_equal(res["stats"], g["stats"])
    np.testing.assert_allclose(res["kl"], g["kl"], rtol=1e-12)
    np.testing.assert_allclose(res["total"], g["total"], rtol=1e-12)


def test_c1_half_step_vs_oracle(cuda_ok):
    """Per-half-step parity from the reference state after iteration 1."""
    from paper_1604_04026_b200.plan import DevicePlan

    g = load_golden("c1_trajectory.npz")
    spec, V, _, _ = _c1()
    w1, f1 = g["w_it1"], g["f_it1"]
    ids = g["ids"][1]
    plan = DevicePlan(V, spec.rank, "fp64")
    plan.set_factors(w1, f1, order=ids)
    plan.half_step("F", ids)
    wg, fg = plan.get_factors()
    f_or = f1.copy()
    oracle.sweep(V.col_ptr, V.row_idx, V.values, w1, oracle.row_sums(w1), f_or, ids, 0.0, 0.0)
    assert np.array_equal(fg, f_or)
    plan.half_step("W", ids)
    wg, fg = plan.get_factors()
    assert sha(wg) == str(g["w_sha"][1]) and sha(fg) == str(g["f_sha"][1])


FACT = load_cases("factorize_small.npz")


@pytest.mark.parametrize("case", range(len(FACT)))
def test_factorize_matches_reference(cuda_ok, case):
    import paper_1604_04026_b200 as kb

    c = FACT[case]
    V = kb.SparseMatrix(int(c["n"]), int(c["m"]), c["col_ptr"], c["row_idx"], c["values"])
    cfg = kb.NmfConfig(rank=int(c["rank"]), reg=kb.RegConfig(*map(float, c["reg"])),
                       max_outer_iters=int(c["iters"]), rel_obj_tol=float(c["rel_obj_tol"]), seed=int(c["seed"]))
    res = kb.factorize(V, cfg)
    assert res.iterations_run == int(c["iterations_run"])
    assert res.converged == bool(c["converged"])
    assert np.array_equal(res.factors.w.values, c["w"])
    assert np.array_equal(res.factors.f.values, c["f"])
    np.testing.assert_allclose(res.log.column("kl_objective"), c["kl"], rtol=1e-12)
    np.testing.assert_allclose(res.log.column("total_objective"), c["total"], rtol=1e-12)
    assert np.array_equal(res.log.column("sparsity_w"), c["sparsity_w"])
    assert np.array_equal(res.log.column("sparsity_f"), c["sparsity_f"])
    assert [res.stats.cap_hits, res.stats.degenerate, res.stats.inner_iters] == list(c["stats"][:3])
