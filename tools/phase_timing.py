"""Per-phase clock cycles of the solver kernels (cluster, cooperative, warp)
on steady-state iterations, from the diagnostic build
(``python -m paper_1604_04026_b200.build --phase`` -> libklnmf_phase.so).

    python tools/phase_timing.py [cfg] [warm_iters] [timed_iters]

Thread 0 of every cluster / cooperative / block-kernel CTA and lane 0 of
every warp-kernel warp accumulate the cycles between phase marks; the table gives each phase's
share of that time and its mean per event (cycles per chunk reduction, per
re-evaluation reduction, per move).
"""
import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("KLNMF_LIB", str(ROOT / "paper_1604_04026_b200" / "libklnmf_phase.so"))
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1604_04026_b200 import _lib, synth  # noqa: E402
from paper_1604_04026_b200.plan import DevicePlan  # noqa: E402

PHASES = ["init", "gather", "pass", "chunk reduce", "scalar newton", "update/re-eval", "re-eval reduce", "final"]
COUNTS = ["chunk reductions", "re-eval reductions", "moves", "chunks"]

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 8
timed = int(sys.argv[3]) if len(sys.argv) > 3 else 2
spec = synth.CONFIGS[name]
V = synth.generate(spec)
w0, f0 = synth.initial_factors(spec)
lib = _lib.load()
fn = lib.klnmf_debug_phase
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((4, 16), dtype=np.uint64)

plan = DevicePlan(V, spec.rank, spec.precision)
rng = np.random.default_rng(spec.seed)
ids = rng.permutation(spec.rank)
plan.set_factors(w0, f0, order=ids)
reg = spec.reg
for it in range(1, warm + timed + 1):
    if it == warm + 1:
        torch.cuda.synchronize()
        assert fn(buf.ctypes.data, 1) == 0
    nxt = rng.permutation(spec.rank)
    plan.half_step("F", ids, alpha=reg.alpha2, beta=reg.beta2, iteration=it)
    plan.half_step("W", ids, nxt, alpha=reg.alpha1, beta=reg.beta1, iteration=it)
    ids = nxt
torch.cuda.synchronize()
assert fn(buf.ctypes.data, 0) == 0
for kind, label in ((0, "cluster kernels"), (1, "cooperative kernel"), (2, "warp kernels (per warp)"),
                    (3, "block kernels (per block)")):
    c = buf[kind].astype(np.float64)
    tot = c[:8].sum() + c[12]
    if tot == 0:
        continue
    print(f"--- {label}: {tot / 1e9:.3f} G CTA-cycles over {timed} iteration(s)")
    for i, p in enumerate(PHASES):
        print(f"  {p:16s} {100 * c[i] / tot:5.1f}%")
    if c[12]:
        print(f"  {'first reduction':16s} {100 * c[12] / tot:5.1f}%  (per subproblem start, includes waiting for the group)")
    for i, p in enumerate(COUNTS):
        print(f"  {p:20s} {c[8 + i]:.0f}")
    per = lambda cyc, n: cyc / n if n else float("nan")  # noqa: E731
    print(f"  cycles per chunk reduction   {per(c[3], c[8]):8.0f}")
    print(f"  cycles per re-eval reduction {per(c[6], c[9]):8.0f}")
    print(f"  cycles per gather            {per(c[1], c[11]):8.0f}")
    print(f"  cycles per pass              {per(c[2], c[8]):8.0f}")
    print(f"  cycles per move (update)     {per(c[5], c[10]):8.0f}")
