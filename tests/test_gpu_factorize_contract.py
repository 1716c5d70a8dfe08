"""factorize's contract on the GPU backend (the reference's
pkg/tests/test_solver.py TestFactorize, restated): stop rules, the caller's
initial factors left untouched, monotone descent, exact recovery of a planted
rank-1 product, nonnegativity, convergence flag and memory accounting --
in the exact fp64 mode (the reference's tolerances) and, where the property
is precision independent, in the fp32 mode (tolerance stated per test)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sparse_counts(seed, n, m, density):
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(seed)
    rows, cols = np.nonzero(rng.random((n, m)) < density)
    return kb.SparseMatrix.from_coo(n, m, rows, cols, (1 + rng.poisson(2.0, size=rows.shape[0])).astype(np.float64))


def _planted(n, m, r, seed):
    # V = W^T F with strictly positive factors on a dense pattern: exactly
    # representable, so the KL data term can reach ~0
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(seed)
    w = rng.uniform(0.5, 1.5, size=(r, n))
    f = rng.uniform(0.5, 1.5, size=(r, m))
    p = w.T @ f
    rows, cols = np.nonzero(p > 0.0)
    return kb.SparseMatrix.from_coo(n, m, rows, cols, p[rows, cols])


def test_zero_iterations_hand_back_a_copy(cuda_ok):
    import paper_1604_04026_b200 as kb

    V = _sparse_counts(1, 20, 30, 0.3)
    pair = kb.init_factors(20, 30, 3, seed=4, mean_v=1.0)
    res = kb.factorize(V, kb.NmfConfig(rank=3, max_outer_iters=0), factors0=pair)
    assert res.iterations_run == 0 and len(res.log) == 0 and not res.converged
    assert np.array_equal(res.factors.w.values, pair.w.values)
    assert res.factors.w.values is not pair.w.values and res.factors.f.values is not pair.f.values


def test_zero_time_budget_runs_nothing(cuda_ok):
    import paper_1604_04026_b200 as kb

    res = kb.factorize(_sparse_counts(2, 20, 30, 0.3),
                       kb.NmfConfig(rank=2, max_outer_iters=50, time_budget_seconds=0.0))
    assert res.iterations_run == 0


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_initial_factors_not_mutated(cuda_ok, precision):
    import paper_1604_04026_b200 as kb

    V = _sparse_counts(3, 20, 30, 0.3)
    pair = kb.init_factors(20, 30, 3, seed=5, mean_v=1.0)
    w0, f0 = pair.w.values.copy(), pair.f.values.copy()
    res = kb.factorize(V, kb.NmfConfig(rank=3, max_outer_iters=5, precision=precision), factors0=pair)
    assert np.array_equal(pair.w.values, w0) and np.array_equal(pair.f.values, f0)
    assert not np.array_equal(res.factors.w.values, w0)


@pytest.mark.parametrize("precision,slack", [("fp64", 1e-8), ("fp32", 1e-6)])
def test_objective_monotone(cuda_ok, precision, slack):
    # fp64: the reference's absolute 1e-8; fp32: relative 1e-6 (fp32 storage
    # rounds every coordinate after its Newton step)
    import paper_1604_04026_b200 as kb

    V = _sparse_counts(8, 20, 30, 0.3)
    res = kb.factorize(V, kb.NmfConfig(rank=4, max_outer_iters=40, rel_obj_tol=0.0, seed=1, precision=precision))
    objs = np.array(res.log.column("total_objective"))
    bound = slack if precision == "fp64" else slack * objs[:-1]
    assert np.all(np.diff(objs) <= bound)


@pytest.mark.parametrize("precision,bound", [("fp64", 1e-6), ("fp32", 1e-6)])
def test_planted_rank1_recovery(cuda_ok, precision, bound):
    import paper_1604_04026_b200 as kb

    V = _planted(25, 35, 1, seed=6)
    res = kb.factorize(V, kb.NmfConfig(rank=1, max_outer_iters=30, rel_obj_tol=0.0, seed=2, precision=precision))
    assert res.log.records[-1].kl_objective <= bound * V.nnz


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_nonnegative_under_l1(cuda_ok, precision):
    import paper_1604_04026_b200 as kb

    res = kb.factorize(_sparse_counts(9, 20, 30, 0.3),
                       kb.NmfConfig(rank=3, max_outer_iters=10, seed=3, precision=precision,
                                    reg=kb.RegConfig(beta1=0.2, beta2=0.2)))
    assert np.all(res.factors.w.values >= 0.0) and np.all(res.factors.f.values >= 0.0)
    assert np.all(np.isfinite(res.factors.w.values)) and np.all(np.isfinite(res.factors.f.values))


def test_convergence_flag(cuda_ok):
    import paper_1604_04026_b200 as kb

    res = kb.factorize(_planted(10, 14, 1, seed=12), kb.NmfConfig(rank=1, max_outer_iters=100, rel_obj_tol=1e-9,
                                                                   seed=4))
    assert res.converged and res.iterations_run < 100


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_memory_accounting_is_sparse(cuda_ok, precision):
    # every tracked buffer is O(nnz) or O((n + m) r): nothing near a dense n*m array
    import paper_1604_04026_b200 as kb

    V = _sparse_counts(15, 40, 60, 0.1)
    ledger = kb.MemoryLedger()
    kb.factorize(V, kb.NmfConfig(rank=4, max_outer_iters=5, precision=precision), ledger=ledger)
    assert ledger.peak_bytes > 0
    assert ledger.max_single_bytes < 8 * V.shape[0] * V.shape[1]


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_unlogged_run_queues_ahead_and_matches_the_logged_one(cuda_ok, precision):
    # without a log or a time budget factorize does not wait for the device
    # between iterations (solver.py: sync_each); the iterates must not change.
    # Enough iterations for the half-step graphs to be captured and replayed
    # while earlier iterations are still in flight.
    import paper_1604_04026_b200 as kb

    V = _sparse_counts(11, 300, 500, 0.2)
    pair = kb.init_factors(300, 500, 8, seed=6, mean_v=1.0)
    kw = dict(rank=8, max_outer_iters=9, rel_obj_tol=0.0, precision=precision, seed=3)
    logged = kb.factorize(V, kb.NmfConfig(log_objectives=True, **kw), factors0=pair)
    quiet = kb.factorize(V, kb.NmfConfig(log_objectives=False, **kw), factors0=pair)
    assert quiet.iterations_run == logged.iterations_run == 9 and len(quiet.log) == 0
    assert np.array_equal(quiet.factors.w.values, logged.factors.w.values)
    assert np.array_equal(quiet.factors.f.values, logged.factors.f.values)
    assert (quiet.stats.inner_iters, quiet.stats.cap_hits, quiet.stats.degenerate) == (
        logged.stats.inner_iters, logged.stats.cap_hits, logged.stats.degenerate)
    assert quiet.solve_seconds > 0.0
