"""fp32-mode edge cases: extreme ranks, empty subproblems, rejected inputs."""
import numpy as np
import pytest

from test_gpu_fast import _check, _check_stats, _compare_half_step

pytestmark = pytest.mark.gpu


def _random(rng, n, m, density, empty_cols=()):
    import paper_1604_04026_b200 as kb

    mask = rng.random((n, m)) < density
    mask[:, list(empty_cols)] = False
    rows, cols = np.nonzero(mask)
    return kb.SparseMatrix.from_coo(n, m, rows, cols, rng.integers(1, 9, size=rows.shape[0]).astype(np.float64))


@pytest.mark.parametrize("r", [1, 2, 5, 256])
def test_extreme_ranks_vs_oracle(cuda_ok, r):
    from paper_1604_04026_b200.plan import DevicePlan

    rng = np.random.default_rng(r)
    V = _random(rng, 300, 200, 0.2, empty_cols=(0, 7))
    w0 = rng.random((r, 300)).astype(np.float32).astype(np.float64)
    f0 = rng.random((r, 200)).astype(np.float32).astype(np.float64)
    plan = DevicePlan(V, r, "fp32")
    ids = rng.permutation(r)
    plan.set_factors(w0, f0, order=ids)
    for which in ("F", "W"):
        mg, mo, tg, to, sg, so = _compare_half_step(plan, which, ids, 0.01, 0.02)
        _check(mg, mo, tg, to, f"r={r} {which}")
        _check_stats(sg, so)
    # empty columns are driven to exact zeros (pkg/tests/test_subproblem.py:171-178)
    F = plan.get_factors()[1]
    assert np.all(F[:, 0] == 0.0) and np.all(F[:, 7] == 0.0)


def test_rank_above_fp32_limit_is_rejected(cuda_ok):
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(1)
    V = _random(rng, 60, 40, 0.3)
    with pytest.raises((ValueError, RuntimeError), match="256"):
        kb.factorize(V, kb.NmfConfig(rank=257, max_outer_iters=1, precision="fp32"))


def test_fp32_needs_positive_eps_div(cuda_ok):
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(2)
    V = _random(rng, 60, 40, 0.3)
    with pytest.raises(ValueError, match="eps_div"):
        kb.factorize(V, kb.NmfConfig(rank=4, max_outer_iters=1, precision="fp32",
                                     tol=kb.Tolerances(eps_div=0.0)))
    # the exact mode accepts it (the reference's arithmetic, division by zero included)
    res = kb.factorize(V, kb.NmfConfig(rank=4, max_outer_iters=2, precision="fp64",
                                       tol=kb.Tolerances(eps_div=0.0), log_objectives=False))
    assert res.iterations_run == 2


def test_single_column_and_single_row(cuda_ok):
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(3)
    for n, m in ((1, 50), (50, 1)):
        V = _random(rng, n, m, 0.9)
        res = kb.factorize(V, kb.NmfConfig(rank=3, max_outer_iters=4, rel_obj_tol=0.0, precision="fp32"))
        tot = [rec.total_objective for rec in res.log.records]
        # monotone within rounding (an exact fit ends at ~0 +- 1e-14)
        assert all(b <= a + 1e-8 * max(1.0, abs(a)) for a, b in zip(tot, tot[1:])), tot
