"""bench.py's launcher contract on the CPU: --gpus N outside torchrun
re-launches N ranks through torch.distributed.run (or fails loudly when
fewer GPUs are visible), and the CPU-baseline sampler's extrapolation."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import bench  # noqa: E402


def test_launch_cmd_is_one_rank_per_gpu():
    cmd = bench.launch_cmd(8, 29555, ["--gpus", "8", "--steps", "3"])
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "8", "--steps", "3"][-3:]
    assert cmd[cmd.index("--master-port=29555")] and Path(cmd[-5]).name == "bench.py"


def test_gpus_beyond_visible_devices_fails_loudly():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode != 0
    assert "only 0 CUDA device" in json.loads(p.stdout.strip().splitlines()[-1])["error"]


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "4"], capture_output=True, text=True,
                       env=env, timeout=300)
    assert p.returncode != 0 and "WORLD_SIZE=2" in p.stderr


def test_ids_at_is_the_reference_stream():
    rng = np.random.default_rng(4)
    seq = [rng.permutation(10) for _ in range(3)]
    assert np.array_equal(bench.ids_at(4, 10, 3), seq[2])


def test_cpu_sample_extrapolates_per_column_time():
    # a small C1-shaped problem: the sampler's serial-cost estimate must be
    # close to the measured cost of solving every column (all buckets small
    # enough to be sampled whole -> exact up to timer noise)
    import oracle
    from paper_1604_04026_b200 import synth

    spec = synth.CONFIGS["C1"].scaled(m=200, n=300)
    V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec)
    ids = bench.ids_at(spec.seed, spec.rank, 1)
    v, it_s, sampled, spv = bench.cpu_reference_sample(V, w0, f0, spec, ids, seconds=5.0, threads=2)
    assert sampled == spec.m + spec.n  # every subproblem fits the budget
    assert v > 0 and it_s > 0 and spv > 0
    assert np.isclose(v, 2.0 * V.nnz * spec.rank / it_s)
