"""The sharded multi-rank path on the GPU: two ranks (processes) sharing one
GPU over a gloo process group run factorize(shard=True) -- nnz-balanced
subproblem ranges per rank, the updated factor rows and maintained products
exchanged after every half-step, stats all-reduced -- and must reproduce the
single-process run BIT FOR BIT (the reference's worker invariance,
pkg/tests/test_solver.py:162-173, across ranks).  Both exchanges are covered:
the fused one (fp32 default: the kernels store their results into the peer's
copies through CUDA-IPC mappings, then a barrier) and the all-gather.  The
kernels of the two ranks never wait on each other: the synchronisation is a
host-side collective between launches."""
import os
import pickle
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, precision, order, fused, out):
    os.environ["KLNMF_FUSED_EXCHANGE"] = "0" if fused is False else "1"
    import torch
    import torch.distributed as dist

    import paper_1604_04026_b200 as kb
    from paper_1604_04026_b200 import plan as plan_mod
    from paper_1604_04026_b200 import synth

    mapped = []
    setup = plan_mod.DevicePlan._setup_peers

    def recording_setup(self):
        setup(self)
        mapped.append(self.fused_exchange)

    plan_mod.DevicePlan._setup_peers = recording_setup
    if fused == "fail" and rank == 1:
        # this rank cannot map its peer: every rank must fall back together
        from paper_1604_04026_b200 import _lib

        real_call = _lib.call

        def failing_call(name, *args):
            if name == "klnmf_ipc_open":
                raise RuntimeError("klnmf_ipc_open failed (test)")
            return real_call(name, *args)

        _lib.call = failing_call
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        spec = synth.CONFIGS["C3"].scaled(m=4000)
        V = synth.generate(spec)
        w0, f0 = synth.initial_factors(spec, round_fp32=True)
        cfg = kb.NmfConfig(rank=spec.rank, reg=spec.reg, max_outer_iters=4, rel_obj_tol=0.0, seed=spec.seed,
                           precision=precision, order=order, shard=True)
        res = kb.factorize(V, cfg, kb.FactorPair(kb.DenseFactor(w0), kb.DenseFactor(f0)))
        if rank == 0:
            with open(out, "wb") as fh:
                pickle.dump({"w": res.factors.w.values, "f": res.factors.f.values,
                             "total": [rec.total_objective for rec in res.log.records],
                             "stats": (res.stats.cap_hits, res.stats.degenerate, res.stats.inner_iters),
                             "fused": mapped}, fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("precision,order,fused", [("fp32", "shared", True), ("fp32", "counter", True),
                                                   ("fp32", "shared", False), ("fp32", "shared", "fail"),
                                                   ("fp64", "shared", False)])
def test_two_ranks_match_one(cuda_ok, tmp_path, precision, order, fused):
    import torch.multiprocessing as mp

    import paper_1604_04026_b200 as kb
    from paper_1604_04026_b200 import synth

    out = str(tmp_path / "rank0.pkl")
    mp.start_processes(_worker, args=(2, _free_port(), precision, order, fused, out), nprocs=2, join=True,
                       start_method="spawn")
    with open(out, "rb") as fh:
        two = pickle.load(fh)
    # the fused exchange is the fp32 path's; fp64 and the opt-out all-gather;
    # a rank that cannot map its peer sends every rank to the all-gather
    expect = {True: [True], False: [], "fail": [False]}[fused] if precision == "fp32" else []
    assert two["fused"] == expect
    spec = synth.CONFIGS["C3"].scaled(m=4000)
    V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec, round_fp32=True)
    cfg = kb.NmfConfig(rank=spec.rank, reg=spec.reg, max_outer_iters=4, rel_obj_tol=0.0, seed=spec.seed,
                       precision=precision, order=order)
    one = kb.factorize(V, cfg, kb.FactorPair(kb.DenseFactor(w0), kb.DenseFactor(f0)))
    assert np.array_equal(two["w"], one.factors.w.values)
    assert np.array_equal(two["f"], one.factors.f.values)
    assert two["total"] == [rec.total_objective for rec in one.log.records]
    assert two["stats"] == (one.stats.cap_hits, one.stats.degenerate, one.stats.inner_iters)
