"""Defining properties of one KL subproblem (the reference's
pkg/tests/test_subproblem.py TestSolveColumn, restated for the GPU path):
closed-form cases of solve_column through the exact kernel
(klnmf_sweep_range_passes), and the empty-column behaviour of the fp32 plan.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_identity_fixed_factor_returns_the_data(cuda_ok):
    # A = I makes the problem separable with the closed form x_k = v_k
    from paper_1604_04026_b200.subproblem import solve_column

    x, _ = solve_column(np.array([0, 1], dtype=np.int64), np.array([2.0, 3.0]), np.eye(2), np.ones(2),
                        np.array([1.0, 1.0]), 0.0, 0.0, [0, 1])
    assert np.allclose(x, [2.0, 3.0], rtol=1e-8)


def test_empty_column_is_driven_exactly_to_zero(cuda_ok):
    # v = 0: the objective is sum_a . x, minimised at x = 0 (reached exactly,
    # not asymptotically: the projected step clamps at the bound)
    from paper_1604_04026_b200.subproblem import solve_column

    rng = np.random.default_rng(7)
    A = rng.uniform(0.2, 1.0, size=(5, 3))
    none = np.array([], dtype=np.int64)
    x, _ = solve_column(none, none.astype(np.float64), np.ascontiguousarray(A.T), A.sum(axis=0),
                        rng.uniform(0.5, 1.5, size=3), 0.0, 0.0, [1, 2, 0])
    assert np.array_equal(x, np.zeros(3))


def test_zero_curvature_still_reaches_the_bound(cuda_ok):
    # alpha = 0 and no data: h = 0 exactly, g = sum_a > 0, so the h <= 0
    # branch must move each coordinate to zero, and that is not a degeneracy
    from paper_1604_04026_b200.subproblem import solve_column

    none = np.array([], dtype=np.int64)
    x, stats = solve_column(none, none.astype(np.float64), np.ones((2, 3)), np.full(2, 3.0),
                            np.array([0.4, 0.9]), 0.0, 0.0, [0, 1])
    assert np.array_equal(x, np.zeros(2))
    assert stats.degenerate == 0


def test_scalar_minimiser(cuda_ok):
    # r = 1, V = [[2]], fixed factor [[1]]: the minimiser of 1*x - 2 log x is 2
    from paper_1604_04026_b200.subproblem import solve_column

    x, _ = solve_column(np.array([0], dtype=np.int64), np.array([2.0]), np.array([[1.0]]), np.array([1.0]),
                        np.array([1.0]), 0.0, 0.0, [0])
    assert x[0] == pytest.approx(2.0, rel=1e-8)


def test_l1_run_reactivates_zero_coordinates(cuda_ok):
    # starting from x = 0 with an L1 weight below the data pull, every
    # coordinate must become active again (g < -eps_grad at zero)
    from paper_1604_04026_b200.subproblem import solve_column

    x, _ = solve_column(np.array([0, 1], dtype=np.int64), np.array([4.0, 5.0]), np.eye(2), np.ones(2),
                        np.zeros(2), 0.0, 0.5, [0, 1])
    assert np.all(x > 0.0)
    # with A = I and beta the closed form is v_k / (1 + beta)
    assert np.allclose(x, [4.0 / 1.5, 5.0 / 1.5], rtol=1e-6)


def test_fp32_plan_empty_columns_are_exactly_zero(cuda_ok):
    # the fp32 kernels keep the same semantics: an empty column of V (alpha =
    # 0) ends its half-step at exact zeros whatever the bucket kernel
    import paper_1604_04026_b200 as kb
    from paper_1604_04026_b200.plan import DevicePlan

    rng = np.random.default_rng(3)
    n, m, r = 400, 300, 12
    mask = rng.random((n, m)) < 0.1
    empty = [0, 5, 150, 299]
    mask[:, empty] = False
    rows, cols = np.nonzero(mask)
    V = kb.SparseMatrix.from_coo(n, m, rows, cols, rng.integers(1, 9, size=rows.shape[0]).astype(np.float64))
    w0 = rng.random((r, n)).astype(np.float32).astype(np.float64)
    f0 = rng.random((r, m)).astype(np.float32).astype(np.float64) + 0.1
    plan = DevicePlan(V, r, "fp32")
    ids = rng.permutation(r)
    plan.set_factors(w0, f0, order=ids)
    plan.half_step("F", ids, alpha=0.0, beta=0.0)
    _, f = plan.get_factors()
    assert np.array_equal(f[:, empty], np.zeros((r, len(empty))))
    nonempty = np.setdiff1d(np.arange(m), empty)
    assert np.all(f[:, nonempty].sum(axis=0) > 0.0)
