"""libklnmf.so loads (no GPU needed) and exports every symbol include/klnmf.h declares."""

import ctypes
import re
from pathlib import Path

from paper_1604_04026_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "klnmf.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(klnmf_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared() == sorted(_lib.EXPORTS)
    assert set(_lib.EXPORTS) == set(_lib._SIGS)


def test_library_loads_and_exports():
    lib = _lib.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.klnmf_abi_version() == 1
    assert lib.klnmf_fast_kernel_count() >= 2


def test_fast_kernel_table_is_bucketed():
    ks = _lib.fast_kernels()
    caps = [c for _, c, _, _ in ks]
    assert caps[-1] == -1  # the last bucket is unbounded (cooperative long-row kernel)
    assert all(a < b for a, b in zip(caps[:-1], caps[1:-1]))


def test_struct_layout_matches_header():
    # klnmf_solve_args_t: 6 side fields + 12 pointers/ints, alignment 8
    assert ctypes.sizeof(_lib.Side) == 48
    # side, 12 pointers, r/rp, 5 doubles, inner_cap, stats, order mode/side, order seed, order_iter,
    # max_passes/n_peers, peer pointers, t_scatter (+ padding)
    assert ctypes.sizeof(_lib.SolveArgs) == 48 + 8 * 12 + 8 + 8 * 5 + 8 + 8 + 8 + 8 + 8 + 8 + 16 + 8 + 16  # ... t_scatter (padded), fixed_mask, slice_words
    # and as the C compiler lays it out
    lib = _lib.load()
    assert lib.klnmf_sizeof_solve_args() == ctypes.sizeof(_lib.SolveArgs)
    assert lib.klnmf_sizeof_side() == ctypes.sizeof(_lib.Side)


def test_errors_are_raised_loudly_without_a_device():
    import pytest

    with pytest.raises(RuntimeError):
        _lib.call("klnmf_solve_fast", ctypes.byref(_lib.SolveArgs()), 999, None)
