"""Pin the CPU oracle against the reference's own outputs (golden fixtures
made by tests/golden/make_golden.py from /root/reference).  Bit-exact."""

import numpy as np
import pytest

import oracle
from conftest import load_cases, load_golden
from paper_1604_04026_b200 import synth

SWEEP = load_cases("sweep_small.npz")


@pytest.mark.parametrize("variant", ["dense", "support"])
@pytest.mark.parametrize("case", range(len(SWEEP)))
def test_sweep_range_bit_exact(case, variant):
    c = SWEEP[case]
    mov = c["moving_in"].copy()
    st = oracle.sweep(c["col_ptr"], c["row_idx"], c["values"], c["at"], c["sum_a"], mov, c["ids"],
                      float(c["alpha"]), float(c["beta"]), float(c["eps_grad"]), float(c["eps_x"]),
                      float(c["eps_div"]), int(c["inner_cap"]), n_workers=1, variant=variant)
    assert np.array_equal(mov, c["moving_out"])
    assert np.array_equal(st, c["stats"])


def test_sweep_worker_invariance():
    c = SWEEP[3]
    outs = []
    for workers in (1, 2, 4):
        mov = c["moving_in"].copy()
        oracle.sweep(c["col_ptr"], c["row_idx"], c["values"], c["at"], c["sum_a"], mov, c["ids"],
                     float(c["alpha"]), float(c["beta"]), n_workers=workers)
        outs.append(mov)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("case", range(len(load_cases("objective_small.npz"))))
def test_objective_bit_exact(case):
    c = load_cases("objective_small.npz")[case]
    data = oracle.kl_data_term(c["col_ptr"], c["row_idx"], c["values"], c["w"], c["f"], float(c["eps_div"]))
    assert data == float(c["data"])
    kl, total = oracle.full_objective(c["col_ptr"], c["row_idx"], c["values"], c["w"], c["f"],
                                      *map(float, c["reg"]), eps_div=float(c["eps_div"]))
    assert kl == float(c["kl"])
    assert total == float(c["total"])


@pytest.mark.parametrize("case", range(len(load_cases("row_sums.npz"))))
def test_row_sums_pairwise_bit_exact(case):
    c = load_cases("row_sums.npz")[case]
    assert np.array_equal(oracle.row_sums(c["x"]), c["sums"])


def test_c1_generator_matches_golden():
    g = load_golden("c1_trajectory.npz")
    V = synth.generate(synth.CONFIGS["C1"])
    import hashlib

    h = hashlib.sha256()
    for a in (V.col_ptr, V.row_idx, V.values):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(g["v_sha"])


def test_c1_trajectory_bit_exact():
    """30 outer iterations of the reference loop on C1: every iterate's
    factors hash-equal and every objective bit-equal (support-t variant)."""
    g = load_golden("c1_trajectory.npz")
    spec = synth.CONFIGS["C1"]
    V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec)
    res = oracle.drive(V.col_ptr, V.row_idx, V.values, spec.n, spec.m, w0, f0, spec.rank, 0, 0, 0, 0,
                       30, spec.seed)
    assert np.array_equal(res["ids"], g["ids"])
    assert list(res["w_sha"]) == list(g["w_sha"])
    assert list(res["f_sha"]) == list(g["f_sha"])
    assert np.array_equal(res["kl"], g["kl"])
    assert np.array_equal(res["total"], g["total"])
    assert np.array_equal(res["stats"], g["stats"])
