"""Full-size reference trajectories of the fp32 throughput configs (C3, C4, C5).

The reference algorithm (``factorize``'s loop, solver.py:283-317, with
``_kernels.sweep_range`` / ``kl_data_term``, _kernels.py:123-160) run for the
config's full iteration count on the pinned CPU oracle (``oracle.drive``,
variant "support": t kept on the column support only, which
tests/test_oracle_golden.py pins bit for bit to the reference itself).  The
starting point is the fp32-representable one both sides use
(``synth.initial_factors``); V holds integer counts, exact in fp32.

    python tests/golden/make_trajectories.py C3 C4      # host-generated matrices (here)
    python tests/golden/make_trajectories.py C5 --iters 3 --device --out DIR   # on a GPU box

C5's matrix only exists on the device (``synth.generate_device``), so its
fixture is made on a GPU box: the matrix is generated there, copied to the
host and solved by the oracle on the host cores; the file records the
matrix's checksum, which the GPU test re-checks before comparing.

The GPU tests (tests/test_gpu_trajectory.py) compare ``factorize``-equivalent
fp32 runs with these files at every outer iteration (north-star bar 1e-4).
"""

from __future__ import annotations

import argparse
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))

import oracle  # noqa: E402  (test infrastructure: the pinned restatement)
from paper_1604_04026_b200 import synth  # noqa: E402  (deterministic generators)


def matrix_sha(col_ptr, row_idx, values) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(col_ptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(row_idx, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(values, dtype=np.float64).tobytes())
    return h.hexdigest()


def make(name: str, iters: int | None, device: bool, out: Path) -> Path:
    spec = synth.CONFIGS[name]
    iters = iters or spec.iters
    t0 = time.time()
    if device:
        V = synth.generate_device(spec).to_host()
    else:
        V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec)
    print(f"{name}: n={spec.n} m={spec.m} nnz={V.nnz} generated in {time.time() - t0:.1f} s", flush=True)
    reg = spec.reg
    t0 = time.time()
    res = oracle.drive(V.col_ptr, V.row_idx, V.values, spec.n, spec.m, w0, f0, spec.rank, reg.alpha1,
                       reg.alpha2, reg.beta1, reg.beta2, iters, spec.seed, log=True)
    secs = time.time() - t0
    print(f"{name}: {iters} iterations in {secs:.1f} s; kl {res['kl'][0]:.9e} -> {res['kl'][-1]:.9e}", flush=True)
    path = out / f"{name.lower()}_traj_full.npz"
    np.savez_compressed(
        path, config=name, n=spec.n, m=spec.m, nnz=V.nnz, rank=spec.rank, seed=spec.seed, iters=iters,
        device_generated=device, matrix_sha=matrix_sha(V.col_ptr, V.row_idx, V.values),
        w0_sha=hashlib.sha256(w0.tobytes()).hexdigest(), f0_sha=hashlib.sha256(f0.tobytes()).hexdigest(),
        ids=res["ids"], kl=res["kl"], total=res["total"], stats=res["stats"],
        w_rowsum=oracle.row_sums(res["w"]), f_rowsum=oracle.row_sums(res["f"]),
        w_zeros=int(np.count_nonzero(res["w"] == 0.0)), f_zeros=int(np.count_nonzero(res["f"] == 0.0)),
        oracle_seconds=secs, oracle_cores=oracle.cores())
    print(f"wrote {path}", flush=True)
    return path


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--iters", type=int, default=None, help="default: the config's iteration count")
    ap.add_argument("--device", action="store_true", help="generate the matrix on the GPU (C5)")
    ap.add_argument("--out", type=Path, default=HERE)
    a = ap.parse_args(argv)
    a.out.mkdir(parents=True, exist_ok=True)
    for name in a.configs:
        make(name, a.iters, a.device or name == "C5", a.out)


if __name__ == "__main__":
    main()
