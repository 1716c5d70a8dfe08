"""Counter-based coordinate order (north-star (c)) on the CPU: the oracle's
Philox4x32-10 against the generator's published known-answer vectors, and the
library's host copy of the device generator (klnmf_chunk_order, the same
source the kernels compile) against the oracle restatement."""
import ctypes

import numpy as np
import pytest

import oracle

# Philox4x32-10 known-answer vectors published with the Random123 library
# (Salmon et al., SC'11): (counter, key) -> output.
KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF, 0xFFFFFFFF),
     (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(ctr, key, want):
    assert tuple(int(x) for x in oracle.philox4x32_10(ctr, key)) == want


def _lib_order(seed, it, item, side, n):
    from paper_1604_04026_b200 import _lib

    out = (ctypes.c_uint8 * max(n, 1))()
    _lib.call("klnmf_chunk_order", seed, it, item, side, n, out)
    return np.frombuffer(out, dtype=np.uint8)[:n].copy()


def test_library_orders_match_oracle():
    rng = np.random.default_rng(3)
    for _ in range(300):
        seed = int(rng.integers(0, 2**63))
        it, item, side = (int(x) for x in rng.integers(0, 2**31, size=3))
        side &= 1
        n = int(rng.integers(0, 65))
        a = _lib_order(seed, it, item, side, n)
        b = oracle.chunk_order(seed, it, item, side, n)
        assert np.array_equal(a, b)
        assert np.array_equal(np.sort(a), np.arange(n))


def test_orders_vary_per_subproblem_iteration_and_side():
    n = 25
    base = oracle.chunk_order(5, 1, 100, 0, n)
    assert not np.array_equal(base, oracle.chunk_order(5, 1, 101, 0, n))
    assert not np.array_equal(base, oracle.chunk_order(5, 2, 100, 0, n))
    assert not np.array_equal(base, oracle.chunk_order(5, 1, 100, 1, n))
    assert not np.array_equal(base, oracle.chunk_order(6, 1, 100, 0, n))
    assert np.array_equal(base, oracle.chunk_order(5, 1, 100, 0, n))


def test_order_positions_are_uniform():
    """Each chunk lands in each visit slot ~uniformly over subproblems."""
    n, items = 8, 8000
    counts = np.zeros((n, n))
    for j in range(items):
        o = oracle.chunk_order(77, 4, j, 0, n)
        counts[np.arange(n), o] += 1
    expected = items / n
    chi2 = ((counts - expected) ** 2 / expected).sum()
    # 49 degrees of freedom; p ~ 1e-6 at ~105
    assert chi2 < 105, chi2


def test_counter_order_is_fp32_only():
    from paper_1604_04026_b200 import NmfConfig

    with pytest.raises(ValueError):
        NmfConfig(precision="fp64", order="counter")
    with pytest.raises(ValueError):
        NmfConfig(precision="fp32", order="random")
    NmfConfig(precision="fp32", order="counter")


def _lib_perm4(seed, it, item, side, pos):
    from paper_1604_04026_b200 import _lib

    out = (ctypes.c_uint8 * 4)()
    _lib.call("klnmf_chunk_perm4", seed, it, item, side, pos, out)
    return np.frombuffer(out, dtype=np.uint8).copy()


def test_library_in_chunk_orders_match_oracle():
    rng = np.random.default_rng(5)
    for _ in range(500):
        seed = int(rng.integers(0, 2**63))
        it, item = (int(x) for x in rng.integers(0, 2**31, size=2))
        side, pos = int(rng.integers(0, 2)), int(rng.integers(0, 64))
        a = _lib_perm4(seed, it, item, side, pos)
        assert np.array_equal(a, oracle.chunk_perm4(seed, it, item, side, pos))
        assert np.array_equal(np.sort(a), np.arange(4))


def test_in_chunk_orders_cover_all_24_uniformly():
    """Each subproblem gets its own order inside every chunk: over many
    subproblems all 24 permutations of a chunk's coordinates occur ~equally."""
    from collections import Counter

    items = 24000
    c = Counter(tuple(oracle.chunk_perm4(9, 3, j, 1, 7)) for j in range(items))
    assert len(c) == 24
    expected = items / 24
    chi2 = sum((v - expected) ** 2 / expected for v in c.values())
    assert chi2 < 60, chi2  # 23 degrees of freedom; p ~ 5e-5 at 60
    # and orders differ between chunks of one subproblem
    assert len({tuple(oracle.chunk_perm4(9, 3, 11, 1, p)) for p in range(25)}) > 5
