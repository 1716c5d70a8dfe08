"""Multi-rank protocol of the sharded solver on CPU (gloo, world size 2).

The GPU path shards every half-step into contiguous nnz-balanced ranges of
subproblems and all-gathers the updated factor rows (and, in fp32 mode, the
maintained products of the updated entries) with plan.allgather_ranges.  Only
one GPU exists in this environment, so the protocol is exercised here with the
pinned oracle as the per-rank solver: the sharded result must equal the
single-process result bit for bit (the reference's worker-count invariance,
tests/test_solver.py:162-173 in the reference, carried over to ranks).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1604_04026_b200 import synth
from paper_1604_04026_b200.plan import allgather_ranges, nnz_balanced_ranges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_allgather(rank, world, port, q):
    _init(rank, world, port)
    try:
        rng = np.random.default_rng(0)
        full2 = rng.random((37, 5)).astype(np.float32)
        full1 = rng.random(101)
        ranges2 = [(0, 10), (10, 37)] if world == 2 else [(0, 37)]
        ranges1 = [(0, 70), (70, 101)] if world == 2 else [(0, 101)]
        b2 = torch.zeros(37, 5)
        b1 = torch.zeros(101, dtype=torch.float64)
        lo, hi = ranges2[rank]
        b2[lo:hi] = torch.from_numpy(full2[lo:hi])
        lo, hi = ranges1[rank]
        b1[lo:hi] = torch.from_numpy(full1[lo:hi])
        allgather_ranges(b2, ranges2, dist.group.WORLD)
        allgather_ranges(b1, ranges1, dist.group.WORLD)
        q.put((rank, np.array_equal(b2.numpy(), full2), np.array_equal(b1.numpy(), full1)))
    finally:
        dist.destroy_process_group()


def _worker_sharded_iterations(rank, world, port, q):
    """Two outer iterations, each half-step sharded over the ranks."""
    _init(rank, world, port)
    try:
        spec = synth.CONFIGS["C1"].scaled(m=240, n=500)
        V = synth.generate(spec)
        w0, f0 = synth.initial_factors(spec)
        pt, rt, vt, _ = oracle.transpose_csc(V.n_rows, V.n_cols, V.col_ptr, V.row_idx, V.values)
        w = torch.from_numpy(np.ascontiguousarray(w0.T).copy())  # item-major like the device layout
        f = torch.from_numpy(np.ascontiguousarray(f0.T).copy())
        rng = np.random.default_rng(spec.seed)
        for _ in range(2):
            ids = rng.permutation(spec.rank)
            for ptr, idx, val, fixed, moving in ((V.col_ptr, V.row_idx, V.values, w, f),
                                                 (pt, rt, vt, f, w)):
                ranges = nnz_balanced_ranges(ptr, world)
                lo, hi = ranges[rank]
                # this rank's subproblems only: a sub-CSC of columns lo..hi
                sub_ptr = ptr[lo:hi + 1] - ptr[lo]
                sel = slice(int(ptr[lo]), int(ptr[hi]))
                mov = np.ascontiguousarray(moving.numpy().T[:, lo:hi])
                fx = np.ascontiguousarray(fixed.numpy().T)
                oracle.sweep(sub_ptr, idx[sel], val[sel], fx, oracle.row_sums(fx), mov, ids, 0.0, 0.0)
                moving[lo:hi] = torch.from_numpy(mov.T)
                allgather_ranges(moving, ranges, dist.group.WORLD)
        q.put((rank, w.numpy().copy(), f.numpy().copy()))
    finally:
        dist.destroy_process_group()


def _run(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_nnz_balanced_ranges_properties():
    rng = np.random.default_rng(3)
    sizes = rng.zipf(1.5, size=1000).clip(max=5000)
    ptr = np.concatenate([[0], np.cumsum(sizes)])
    for parts in (1, 2, 3, 8):
        rs = nnz_balanced_ranges(ptr, parts)
        assert rs[0][0] == 0 and rs[-1][1] == 1000
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        loads = [ptr[hi] - ptr[lo] for lo, hi in rs]
        assert max(loads) <= ptr[-1] / parts + sizes.max()


@pytest.mark.skipif(not dist.is_gloo_available(), reason="gloo backend unavailable")
def test_allgather_ranges_gloo():
    out = _run(_worker_allgather, 2)
    assert all(ok2 and ok1 for _, ok2, ok1 in out)


@pytest.mark.skipif(not dist.is_gloo_available(), reason="gloo backend unavailable")
def test_sharded_half_steps_bitwise_rank_invariant():
    single = _run(_worker_sharded_iterations, 1)[0]
    pair = _run(_worker_sharded_iterations, 2)
    for _, w, f in pair:
        assert np.array_equal(w, single[1])
        assert np.array_equal(f, single[2])


def _c5_like_row_sizes():
    """Row lengths with C5's shape: Zipf(1.0)
    feature popularity over 141,043 rows, 8.2M documents, ~565M nonzeros,
    longest rows ~7M (a row cannot exceed the document count)."""
    i = np.arange(1, 141_044, dtype=np.float64)
    m = 8.2e6
    lo, hi = 0.1, 100.0
    for _ in range(60):  # expected tokens of the top feature per document
        c = np.sqrt(lo * hi)
        tot = (m * -np.expm1(-c / i)).sum()
        lo, hi = (c, hi) if tot < 5.65e8 else (lo, c)
    return np.maximum(1, (m * -np.expm1(-c / i))).astype(np.int64)


def test_cost_balanced_ranges_properties():
    from paper_1604_04026_b200.plan import cost_balanced_ranges, subproblem_cost

    rng = np.random.default_rng(4)
    sizes = rng.zipf(1.3, size=5000).clip(max=2_000_000)
    ptr = np.concatenate([[0], np.cumsum(sizes)])
    cost = subproblem_cost(sizes)
    for parts in (1, 2, 3, 8):
        rs = cost_balanced_ranges(ptr, parts)
        assert rs[0][0] == 0 and rs[-1][1] == len(sizes)
        assert all(a[1] == b[0] and a[0] <= a[1] for a, b in zip(rs, rs[1:]))
        loads = [cost[lo:hi].sum() for lo, hi in rs]
        assert max(loads) <= cost.sum() / parts + cost.max()


def test_cost_balancing_c5_w_side_at_8_ranks():
    """C5's W side (rows, Zipf head first): nnz-balanced ranges give the first
    rank the long rows (spill path, ~2-5x the per-entry cost), cost-balanced
    ranges keep the modelled per-rank time within 10% of the mean at P=8
    (DESIGN.md §6)."""
    from paper_1604_04026_b200.plan import (cost_balanced_ranges, dealt_assignment, nnz_balanced_ranges,
                                            subproblem_cost)

    sizes = _c5_like_row_sizes()
    assert 5.5e8 < sizes.sum() < 5.8e8 and 6e6 < sizes.max() < 8.2e6
    ptr = np.concatenate([[0], np.cumsum(sizes)])
    cost = subproblem_cost(sizes)

    def imbalance(rs):
        loads = np.array([cost[lo:hi].sum() for lo, hi in rs])
        return loads.max() / loads.mean()

    def imbalance_items(owned):
        loads = np.array([cost[o].sum() for o in owned])
        return loads.max() / loads.mean()

    by_nnz = imbalance(nnz_balanced_ranges(ptr, 8))
    by_cost = imbalance(cost_balanced_ranges(ptr, 8))
    owned = dealt_assignment(ptr, 8)
    dealt = imbalance_items(owned)
    print(f"C5 W side, P=8: max/mean modelled rank time nnz-balanced {by_nnz:.3f}, "
          f"cost-balanced ranges {by_cost:.3f}, dealt {dealt:.3f}")
    assert by_cost < by_nnz
    assert dealt <= 1.10
    assert np.array_equal(np.sort(np.concatenate(owned)), np.arange(len(sizes)))


def test_dealt_assignment_properties():
    from paper_1604_04026_b200.plan import dealt_assignment, subproblem_cost

    rng = np.random.default_rng(8)
    for parts in (1, 2, 3, 8):
        sizes = rng.zipf(1.2, size=3000).clip(max=3_000_000)
        ptr = np.concatenate([[0], np.cumsum(sizes)])
        owned = dealt_assignment(ptr, parts)
        assert len(owned) == parts
        allv = np.concatenate(owned)
        assert np.array_equal(np.sort(allv), np.arange(len(sizes)))  # a partition
        assert all(np.all(np.diff(o) > 0) for o in owned)  # ascending
        c = subproblem_cost(sizes)
        loads = np.array([c[o].sum() for o in owned])
        assert loads.max() <= c.sum() / parts + c.max()
