"""GPU baseline kernels: the MU update, KKT
violations and multi-pass solve_column through the C ABI, bit-exact against
fixtures recorded from the reference, plus the reference's MU tests
(pkg/tests/test_multiplicative.py) and KKT-certificate tests
(pkg/tests/test_subproblem.py) restated on the device."""
import ctypes
import json

import numpy as np
import pytest

from conftest import load_cases

pytestmark = pytest.mark.gpu


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def test_mu_update_range_bit_exact(cuda_ok):
    from paper_1604_04026_b200 import _lib

    for c in load_cases("mu_small.npz"):
        mov = np.ascontiguousarray(c["moving_in"].copy())
        fixed = np.ascontiguousarray(c["fixed"])
        r, n_fix = fixed.shape
        _lib.call("klnmf_mu_update_range", _p(c["col_ptr"]), _p(c["row_idx"]), _p(c["values"]), _p(fixed),
                  _p(mov), _p(np.ascontiguousarray(c["sum_fixed"])), float(c["eps_mu"]), 0, mov.shape[1], r, n_fix,
                  mov.shape[1])
        assert np.array_equal(mov, c["moving_out"])


def test_kkt_violations_bit_exact(cuda_ok):
    import paper_1604_04026_b200 as kb

    for c in load_cases("kkt_small.npz"):
        tol = kb.Tolerances(eps_x=float(c["eps_x"]))
        ptr = c["col_ptr"]
        for j in range(c["x"].shape[1]):
            out = kb.kkt_violations(c["row_idx"][ptr[j]:ptr[j + 1]], c["values"][ptr[j]:ptr[j + 1]], c["at"],
                                    c["sum_a"], c["x"][:, j], float(c["alpha"]), float(c["beta"]), tol)
            assert np.array_equal(out, c["out"][:, j])


def test_multipass_solve_column_bit_exact(cuda_ok):
    import paper_1604_04026_b200 as kb

    for c in load_cases("solve_column_small.npz"):
        tol = kb.Tolerances(eps_x=float(c["eps_x"]))
        x, st = kb.solve_column(c["v_idx"], c["v_val"], c["at"], c["sum_a"], c["x0"], float(c["alpha"]),
                                float(c["beta"]), c["ids"], tol, max_passes=int(c["max_passes"]))
        assert np.array_equal(x, c["x"])
        assert [st.cap_hits, st.degenerate, st.inner_iters, st.passes] == c["stats"].tolist()


def test_solve_column_kkt_certificate(cuda_ok):
    """Run to stationarity; the exit point carries the certificate
    (pkg/tests/test_subproblem.py:247-263: violations <= 1e-12 at eps_x tiny)."""
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(4)
    for trial in range(6):
        n, r = 40, 5
        at = rng.uniform(0.0, 2.0, size=(r, n))
        idx = np.sort(rng.choice(n, size=15, replace=False))
        val = rng.uniform(0.5, 5.0, size=15)
        sums = at.sum(axis=1)
        tol = kb.Tolerances(eps_x=1e-8)
        x, st = kb.solve_column(idx, val, at, sums, rng.uniform(0.1, 1.0, size=r), 0.01 * trial, 0.0,
                                rng.permutation(r), tol, max_passes=500)
        assert st.passes < 500
        viol = kb.kkt_violations(idx, val, at, sums, x, 0.01 * trial, 0.0, tol)
        assert np.all(viol <= 1e-12), viol


def _matrix(rng, n, m, density):
    import paper_1604_04026_b200 as kb

    mask = rng.random((n, m)) < density
    rows, cols = np.nonzero(mask)
    return kb.SparseMatrix.from_coo(n, m, rows, cols, np.round(rng.uniform(0.5, 6.0, size=rows.shape[0])))


def test_mu_factorize_matches_reference_run(cuda_ok):
    import paper_1604_04026_b200 as kb

    z = np.load(__import__("conftest").GOLDEN / "mu_factorize.npz")
    V = kb.SparseMatrix(int(z["n_rows"]), int(z["col_ptr"].shape[0] - 1), z["col_ptr"], z["row_idx"], z["values"])
    res = kb.mu_factorize(V, kb.NmfConfig(rank=int(z["rank"]), max_outer_iters=int(z["iters"]), rel_obj_tol=0.0,
                                          seed=int(z["seed"])))
    assert np.array_equal(res.factors.w.values, z["w"])
    assert np.array_equal(res.factors.f.values, z["f"])
    kl = np.array([rec.kl_objective for rec in res.log.records])
    assert np.allclose(kl, z["kl"], rtol=1e-12, atol=0.0)


def test_mu_objective_monotone_and_positive(cuda_ok):
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(1)
    V = _matrix(rng, 25, 40, 0.3)
    res = kb.mu_factorize(V, kb.NmfConfig(rank=4, max_outer_iters=25, rel_obj_tol=0.0, seed=2))
    objs = [rec.total_objective for rec in res.log.records]
    assert res.iterations_run == 25
    assert all(b <= a + 1e-8 for a, b in zip(objs, objs[1:]))
    # an empty column shrinks by ~eps/rowsum per iteration but stays positive
    # over the reference test's 10 iterations (test_multiplicative.py:47-56)
    V = kb.SparseMatrix.from_coo(25, 41, *_with_empty_column(V))
    res = kb.mu_factorize(V, kb.NmfConfig(rank=4, max_outer_iters=10, rel_obj_tol=0.0, seed=2))
    assert np.all(res.factors.w.values > 0.0) and np.all(res.factors.f.values > 0.0)
    assert res.factors.w.sparsity() == 0.0 and res.factors.f.sparsity() == 0.0


def _with_empty_column(V):
    cols = np.repeat(np.arange(V.n_cols), np.diff(V.col_ptr))
    return V.row_idx, cols, V.values


def test_mu_iterate_matches_factorize_and_validates(cuda_ok):
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(3)
    V = _matrix(rng, 18, 30, 0.8)
    pair = kb.init_factors(18, 30, 4, 8, mean_v=1.0)
    state = kb.MuState(pair.copy())
    vt = V.transpose()
    for _ in range(5):
        kb.mu_iterate(V, state, vt)
    res = kb.mu_factorize(V, kb.NmfConfig(rank=4, max_outer_iters=5, rel_obj_tol=0.0, log_objectives=False),
                          factors0=pair.copy())
    assert np.array_equal(state.factors.w.values, res.factors.w.values)
    assert np.array_equal(state.factors.f.values, res.factors.f.values)
    with pytest.raises(ValueError):
        kb.MuState(kb.FactorPair(kb.DenseFactor(np.array([[0.0, 1.0]])), kb.DenseFactor(np.array([[1.0, 1.0]]))))
    empty = kb.SparseMatrix(3, 3, np.zeros(4, dtype=np.int64), np.array([], dtype=np.int64), np.array([]))
    with pytest.raises(ValueError, match="empty"):
        kb.mu_factorize(empty, kb.NmfConfig(rank=2))


def test_planted_mu_converges(cuda_ok):
    """Rank-1 dense planted product: KL -> 0 (pkg/tests/test_multiplicative.py:58-65)."""
    import paper_1604_04026_b200 as kb

    rng = np.random.default_rng(5)
    w, f = rng.uniform(0.5, 1.5, size=(1, 15)), rng.uniform(0.5, 1.5, size=(1, 20))
    dense = w.T @ f
    rows, cols = np.nonzero(dense)
    V = kb.SparseMatrix.from_coo(15, 20, rows, cols, dense[rows, cols])
    res = kb.mu_factorize(V, kb.NmfConfig(rank=1, max_outer_iters=200, rel_obj_tol=0.0, seed=6,
                                          log_objectives=False))
    kl, _ = kb.full_objective(V, res.factors.w, res.factors.f, kb.RegConfig())
    assert kl <= 1e-4 * V.nnz


def test_race_driver(cuda_ok, tmp_path):
    from paper_1604_04026_b200 import cli

    rc = cli.main(["race", "--config", "C1@m=200", "--rank", "4", "--budget", "0.5", "--precision", "fp32",
                   "--out", str(tmp_path)])
    assert rc == 0
    rows = (tmp_path / "race.csv").read_text().splitlines()
    assert rows[0] == "algorithm,elapsed_seconds,kl_objective"
    assert {r.split(",")[0] for r in rows[1:]} == {"srcd", "mu"}
    s = json.loads((tmp_path / "summary.json").read_text())
    assert set(s["final_kl"]) == {"srcd", "mu"}
    assert s["final_kl"]["srcd"] < s["initial_kl_objective"] and s["final_kl"]["mu"] < s["initial_kl_objective"]
