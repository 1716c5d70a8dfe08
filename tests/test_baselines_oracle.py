"""The oracle's restatements of the baseline kernels (mu_update_range,
kkt_violation, multi-pass solve_column) against fixtures recorded from the
reference itself (tests/golden/make_golden.py "baselines"), bit for bit."""
import numpy as np

import oracle
from conftest import load_cases


def test_mu_update_range_matches_reference():
    for c in load_cases("mu_small.npz"):
        mov = c["moving_in"].copy()
        oracle.mu_update_range(c["col_ptr"], c["row_idx"], c["values"], c["fixed"], mov, c["sum_fixed"],
                               float(c["eps_mu"]), 0, mov.shape[1])
        assert np.array_equal(mov, c["moving_out"])


def test_kkt_violation_matches_reference():
    for c in load_cases("kkt_small.npz"):
        out = oracle.kkt_violation(c["col_ptr"], c["row_idx"], c["values"], c["at"], c["sum_a"], c["x"],
                                   float(c["alpha"]), float(c["beta"]), eps_x=float(c["eps_x"]))
        assert np.array_equal(out, c["out"])


def test_multipass_solve_column_matches_reference():
    for c in load_cases("solve_column_small.npz"):
        x = c["x0"].copy()
        st = oracle.solve_column(c["v_idx"], c["v_val"], c["at"], c["sum_a"], x, c["ids"], float(c["alpha"]),
                                 float(c["beta"]), eps_x=float(c["eps_x"]), max_passes=int(c["max_passes"]))
        assert np.array_equal(x, c["x"])
        assert np.array_equal(st, c["stats"])
