"""Host logic of the fused sharded exchange (plan.DevicePlan._setup_peers) on
CPU: two gloo ranks exchange their buffers' IPC handles, map every peer
allocation once and build the peer-pointer tables the kernels store through;
if any rank cannot map its peers, every rank falls back to the all-gather
together.  The CUDA-IPC calls are replaced by a recording fake (no GPU here);
the device path itself is tests/test_gpu_sharded.py."""
import ctypes
import os
import pickle
import socket
import types

import pytest

pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fail_rank, out):
    import torch
    import torch.distributed as dist

    from paper_1604_04026_b200 import _lib
    from paper_1604_04026_b200.plan import DevicePlan

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    calls = []

    def fake_call(name, *args):
        calls.append(name)
        if name == "klnmf_ipc_export":
            ptr, handle, off = args
            # W and F share one allocation (offsets 0 / 4096), t's arrays another
            alloc = "fac" if ptr in (1000, 5096) else "t"
            tag = f"r{rank}-{alloc}".encode().ljust(64, b"\0")
            ctypes.memmove(handle, tag, 64)
            off._obj.value = {1000: 0, 5096: 4096, 9000: 0, 9800: 800}[ptr]
        elif name == "klnmf_ipc_open":
            handle, base = args
            if rank == fail_rank:
                raise RuntimeError("klnmf_ipc_open failed (test)")
            peer, alloc = bytes(handle).rstrip(b"\0").decode().split("-")
            base._obj.value = (1 << 40) * (1 + int(peer[1:])) + (0 if alloc == "fac" else 1 << 30)

    _lib.call = fake_call

    def tensor_at(addr):
        return types.SimpleNamespace(data_ptr=lambda: addr)

    plan = types.SimpleNamespace(
        factors={"W": tensor_at(1000), "F": tensor_at(5096)}, t={"csc": tensor_at(9000), "csr": tensor_at(9800)},
        world=world, rank_id=rank, group=None, dev=torch.device("cpu"), _peers=None, _ipc_bases=[])
    try:
        DevicePlan._setup_peers(plan)
        peers = None if plan._peers is None else {k: v.tolist() for k, v in plan._peers.items()}
        with open(f"{out}.{rank}", "wb") as fh:
            pickle.dump({"peers": peers, "bases": plan._ipc_bases, "calls": calls}, fh)
    finally:
        dist.destroy_process_group()


def _run(tmp_path, fail_rank):
    import torch.multiprocessing as mp

    out = str(tmp_path / "res")
    mp.start_processes(_worker, args=(2, _free_port(), fail_rank, out), nprocs=2, join=True, start_method="spawn")
    res = []
    for r in range(2):
        with open(f"{out}.{r}", "rb") as fh:
            res.append(pickle.load(fh))
    return res


def test_peer_tables(tmp_path):
    res = _run(tmp_path, fail_rank=-1)
    for rank, r in enumerate(res):
        peer = 1 - rank
        fac = (1 << 40) * (1 + peer)
        tb = fac + (1 << 30)
        assert r["peers"] == {"W": [fac], "F": [fac + 4096], "csc": [tb], "csr": [tb + 800]}
        # one mapping per peer allocation, not per buffer
        assert r["calls"].count("klnmf_ipc_open") == 2
        assert sorted(r["bases"]) == sorted([fac, tb])


def test_one_rank_failing_sends_every_rank_to_allgather(tmp_path):
    res = _run(tmp_path, fail_rank=1)
    assert [r["peers"] for r in res] == [None, None]
    # the rank that mapped its peer releases the mappings again
    assert res[0]["calls"].count("klnmf_ipc_close") == res[0]["calls"].count("klnmf_ipc_open") == 2
    assert res[0]["bases"] == [] and res[1]["bases"] == []
