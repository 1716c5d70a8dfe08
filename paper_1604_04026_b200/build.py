"""Builds libklnmf.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a.

``python -m paper_1604_04026_b200.build`` or ``__graft_entry__.build()``.
The shared library lands next to this file so it travels with the repo
snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
OBJDIR = PKG / "_build"
LIB = PKG / "libklnmf.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", str(INCLUDE)]
# exact mode mirrors the reference's FMA-free numba codegen (SURVEY.md finding 3)
PER_FILE = {"solve_exact.cu": ["-fmad=false"]}
SOURCES = ["abi_host.cu", "solve_exact.cu", "solve_fast.cu", "factor_ops.cu", "sparse_build.cu", "host_io.cu", "mm_io.cu", "synth_gen.cu"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: cannot build libklnmf.so")
    return cand


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str | None = None) -> Path:
    """variant="phase": a diagnostic copy (libklnmf_phase.so) whose long-row
    kernels count clock cycles per phase (KLNMF_PHASE_TIMING, tools/phase_timing.py)."""
    objdir, lib, extra = OBJDIR, LIB, []
    if variant == "phase":
        objdir, lib, extra = PKG / "_build_phase", PKG / "libklnmf_phase.so", ["-DKLNMF_PHASE_TIMING"]
    elif variant is not None:
        raise ValueError(f"unknown build variant {variant!r}")
    return _build(objdir, lib, extra, force, verbose)


def _build(objdir: Path, lib: Path, extra, force: bool, verbose: bool) -> Path:
    objdir.mkdir(exist_ok=True)
    headers = [CSRC / "common.cuh", INCLUDE / "klnmf.h"]
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = objdir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers]):
            cmd = [nvcc(), *ARCH, *COMMON, *extra, *PER_FILE.get(src, []), "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _stale(lib, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-pthread", "-o", str(lib), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True,
                variant="phase" if "--phase" in sys.argv else None))
