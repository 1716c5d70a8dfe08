"""Host-side API mirror (no GPU): the reference's config, storage and log
types with the same validation (solver.py:37-131, sparse.py:48-206,
subproblem.py:28-81); ported from the reference's own unit tests."""

import numpy as np
import pytest

import paper_1604_04026_b200 as kb


class TestConfigs:
    @pytest.mark.parametrize("kwargs", [{"rank": 0}, {"max_outer_iters": -1}, {"rel_obj_tol": -0.1},
                                        {"n_workers": 0}, {"precision": "fp16"}])
    def test_invalid(self, kwargs):
        with pytest.raises(ValueError):
            kb.NmfConfig(**kwargs)

    def test_negative_reg_rejected(self):
        with pytest.raises(ValueError):
            kb.RegConfig(alpha1=-1.0)

    def test_defaults_match_reference(self):
        cfg = kb.NmfConfig()
        assert (cfg.rank, cfg.max_outer_iters, cfg.rel_obj_tol, cfg.seed, cfg.n_workers) == (10, 100, 1e-6, 0, 1)
        assert cfg.precision == "fp64" and cfg.log_objectives

    def test_tolerance_defaults(self):
        tol = kb.Tolerances()
        assert (tol.eps_grad, tol.eps_x, tol.eps_div, tol.inner_iter_cap) == (1e-10, 0.1, 1e-16, 128)

    @pytest.mark.parametrize("kwargs", [{"eps_grad": 0.0}, {"eps_x": 1.5}, {"eps_div": -1e-3},
                                        {"inner_iter_cap": 0}])
    def test_tolerances_invalid(self, kwargs):
        with pytest.raises(ValueError):
            kb.Tolerances(**kwargs)


class TestLog:
    def test_invariants(self):
        log = kb.ConvergenceLog()
        with pytest.raises(ValueError):
            log.append(kb.IterationRecord(2, 1.0, 1.0, 1.0, 0.0, 0.0))
        log.append(kb.IterationRecord(1, 1.0, 1.0, 1.0, 0.0, 0.0))
        with pytest.raises(ValueError):
            log.append(kb.IterationRecord(2, 1.0, 1.0, 1.0, 0.0, 0.0))
        log.append(kb.IterationRecord(2, 2.0, 0.5, 0.5, 0.1, 0.2))
        assert len(log) == 2
        assert np.array_equal(log.column("kl_objective"), [1.0, 0.5])


class TestSparse:
    def test_from_coo_sorted_and_zeros_dropped(self):
        m = kb.SparseMatrix.from_coo(3, 2, [2, 0, 1, 0], [1, 1, 0, 0], [1.0, 2.0, 0.0, 4.0])
        assert m.nnz == 3
        assert m.col_ptr.tolist() == [0, 1, 3]
        assert m.row_idx.tolist() == [0, 0, 2]

    def test_duplicate_rejected(self):
        with pytest.raises(kb.DuplicateEntryError):
            kb.SparseMatrix.from_coo(2, 2, [0, 0], [1, 1], [1.0, 2.0])

    def test_negative_rejected(self):
        with pytest.raises(ValueError):
            kb.SparseMatrix.from_coo(2, 2, [0], [0], [-1.0])

    def test_unsorted_rows_rejected(self):
        with pytest.raises(ValueError, match="strictly increasing"):
            kb.SparseMatrix(3, 1, [0, 2], [2, 1], [1.0, 1.0])

    def test_rows_may_restart_between_columns(self):
        m = kb.SparseMatrix(3, 3, [0, 2, 2, 4], [1, 2, 0, 1], [1.0, 1.0, 1.0, 1.0])
        assert m.nnz == 4

    @pytest.mark.parametrize("seed", range(4))
    def test_transpose_involution_bit_exact(self, seed):
        rng = np.random.default_rng(seed)
        mask = rng.random((7, 9)) < 0.4
        r, c = np.nonzero(mask)
        m = kb.SparseMatrix.from_coo(7, 9, r, c, rng.uniform(0.1, 3.0, size=r.shape[0]))
        tt = m.transpose().transpose()
        assert np.array_equal(tt.col_ptr, m.col_ptr) and np.array_equal(tt.row_idx, m.row_idx)
        assert np.array_equal(tt.values, m.values)
        assert np.array_equal(m.transpose().to_dense(), m.to_dense().T)

    def test_dense_factor_validation_and_sums(self):
        with pytest.raises(ValueError):
            kb.DenseFactor(np.array([[-1.0]]))
        f = kb.DenseFactor(np.array([[1.0, 0.0], [2.0, 3.0]]))
        assert f.row_sums().tolist() == [1.0, 5.0]
        assert f.sparsity() == 0.25


def test_init_factors_reference_stream():
    a = kb.init_factors(5, 7, 3, seed=42, mean_v=2.0)
    rng = np.random.default_rng(42)
    s = 2.0 * np.sqrt(2.0 / 3)
    assert np.array_equal(a.w.values, s * (1.0 - rng.random((3, 5))))
    assert np.array_equal(a.f.values, s * (1.0 - rng.random((3, 7))))


def test_memory_ledger():
    led = kb.MemoryLedger()
    led.track("a", np.zeros(10))
    with pytest.raises(ValueError):
        led.track("a", np.zeros(1))
    led.track("b", np.zeros(5))
    assert led.peak_bytes == 120
    led.release("a")
    assert led.live_bytes == 40


def test_synth_configs_shapes():
    spec = kb.synth.CONFIGS["C1"] if hasattr(kb, "synth") else None
    from paper_1604_04026_b200 import synth

    spec = synth.CONFIGS["C3"].scaled(m=300, n=2000)
    V = synth.generate(spec)
    assert V.shape == (2000, 300) and V.nnz > 0
    assert np.all(V.values >= 1.0) and np.all(V.values == np.round(V.values))
    V2 = synth.generate(spec)
    assert np.array_equal(V.row_idx, V2.row_idx)


def test_fp32_plan_rejects_32bit_offset_overflow():
    # fp32 kernels address the fixed factor with 32-bit offsets: a shape whose
    # items x padded rank reaches 2^31 must be refused loudly, not wrap
    import types

    import pytest

    from paper_1604_04026_b200.plan import DevicePlan

    huge = types.SimpleNamespace(shape=(30_000_000, 10))
    with pytest.raises(ValueError, match="2\\^31"):
        DevicePlan(huge, 100, "fp32")


@pytest.mark.parametrize("bad", [1e-40, 1e39])
def test_fp32_plan_rejects_values_outside_normal_fp32(bad):
    # a positive fp64 value that is subnormal/zero or inf in fp32 would make
    # the entry state 1/v infinite and spread NaN: refused before any upload
    from paper_1604_04026_b200.plan import DevicePlan

    V = kb.SparseMatrix(3, 2, np.array([0, 2, 3]), np.array([0, 2, 1]), np.array([1.0, bad, 2.0]))
    with pytest.raises(ValueError, match="fp32 range"):
        DevicePlan(V, 4, "fp32")


def test_order_key_accepts_any_default_rng_seed():
    # the reference accepts any seed default_rng does (solver.py:276); only
    # the counter order needs a 64-bit key, derived deterministically
    from paper_1604_04026_b200.solver import _order_key

    assert _order_key(7) == 7 and _order_key(np.int64(9)) == 9
    for seed in (None, [1, 2, 3], np.random.SeedSequence(5), 2**70):
        k = _order_key(seed)
        assert 0 <= k < 2**64
        if seed is not None:
            assert k == _order_key(seed)
