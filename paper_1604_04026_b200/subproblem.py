"""Solver tolerance and statistics types (klnmf.subproblem, subproblem.py:28-81).

The semantics the device kernels honour: ``eps_grad`` bounds the gradient in
the inner-loop entry test, ``eps_x`` is the relative-step cutoff, ``eps_div``
guards the denominators (and the objective's log argument), and
``inner_iter_cap`` bounds Newton steps per coordinate visit (128 in the
reference code, subproblem.py:39).
"""

from __future__ import annotations

import dataclasses

import numpy as np

from . import _lib

__all__ = ["Tolerances", "SolveStats", "SubproblemWorkspace"]


@dataclasses.dataclass(frozen=True)
class Tolerances:
    eps_grad: float = 1e-10
    eps_x: float = 0.1
    eps_div: float = 1e-16
    inner_iter_cap: int = 128

    def __post_init__(self):
        if self.eps_grad <= 0.0 or self.eps_x <= 0.0 or self.eps_div < 0.0:
            raise ValueError("tolerances must be positive (eps_div may be 0)")
        if self.eps_x >= 1.0:
            raise ValueError("eps_x must be < 1")
        if self.inner_iter_cap < 1:
            raise ValueError("inner_iter_cap must be >= 1")


@dataclasses.dataclass
class SolveStats:
    """Counters summed over subproblem solves (subproblem.py:65-81)."""

    cap_hits: int = 0
    degenerate: int = 0
    inner_iters: int = 0
    passes: int = 0

    @classmethod
    def from_array(cls, arr) -> "SolveStats":
        return cls(
            cap_hits=int(arr[_lib.STAT_CAP_HITS]),
            degenerate=int(arr[_lib.STAT_DEGENERATE]),
            inner_iters=int(arr[_lib.STAT_INNER_ITERS]),
            passes=int(arr[_lib.STAT_PASSES]),
        )

    def add(self, other: "SolveStats") -> None:
        self.cap_hits += other.cap_hits
        self.degenerate += other.degenerate
        self.inner_iters += other.inner_iters
        self.passes += other.passes


@dataclasses.dataclass
class SubproblemWorkspace:
    """Kept for signature compatibility with sweep(..., workspaces=...)
    (subproblem.py:50-62).  The device path owns its scratch, so these host
    buffers are never touched by the solve."""

    ax: np.ndarray
    x: np.ndarray

    @classmethod
    def allocate(cls, n: int, r: int) -> "SubproblemWorkspace":
        return cls(np.zeros(n), np.zeros(r))

    def nbytes(self) -> int:
        return int(self.ax.nbytes + self.x.nbytes)
