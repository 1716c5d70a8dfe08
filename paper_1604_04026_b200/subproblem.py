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

__all__ = [
    "Tolerances",
    "SolveStats",
    "SubproblemWorkspace",
    "grad_and_hess",
    "newton_step",
    "solve_column",
    "subproblem_objective",
    "kkt_violations",
]


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


def _c64(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def grad_and_hess(k, v_indices, v_values, at, ax, sum_a, x_k, alpha, beta, eps_div=1e-16):
    """Gradient and Hessian diagonal of one coordinate (subproblem.py:84-110,
    _kernels._grad_hess): a host helper in the reference's operation order
    (serial over the entries), O(nnz(v))."""
    at = np.asarray(at, dtype=np.float64)
    g = float(sum_a[k]) + float(alpha) * float(x_k) + float(beta)
    h = float(alpha)
    row = at[int(k)]
    for i, v in zip(np.asarray(v_indices, dtype=np.int64).tolist(), np.asarray(v_values, np.float64).tolist()):
        a = float(row[i])
        if a != 0.0:
            q = a / (float(ax[i]) + eps_div)
            g -= v * q
            h += v * q * q
    return g, h


def newton_step(x_k, gradient, hessian_diag):
    """Projected Newton step max(0, x - g/h); (new_x, delta) (subproblem.py:113-122)."""
    if hessian_diag <= 0.0:
        return float(x_k), 0.0
    new_x = max(0.0, x_k - gradient / hessian_diag)
    return new_x, new_x - x_k


def _one_column(v_indices, v_values, n):
    v_indices = _c64(v_indices, np.int64)
    v_values = _c64(v_values)
    if v_indices.shape[0] and (v_indices.min() < 0 or v_indices.max() >= n):
        raise ValueError("column index out of range for the operator")
    return np.array([0, v_indices.shape[0]], dtype=np.int64), v_indices, v_values


def solve_column(v_indices, v_values, at, sum_a, x0, alpha, beta, ids, tol: Tolerances = Tolerances(),
                 workspace: SubproblemWorkspace | None = None, max_passes: int = 200):
    """Minimize D(v || Ax) + (alpha/2)||x||^2 + beta||x||_1 over x >= 0
    (subproblem.py:125-166): passes over the coordinates in order ``ids``
    repeat until none moves (the stationarity certificate) or max_passes.
    Runs the exact kernel on the GPU (klnmf_sweep_range_passes), bit-identical
    to the reference.  Returns (x, SolveStats)."""
    import ctypes

    at = _c64(at)
    r, n = at.shape
    x0 = np.asarray(x0, dtype=np.float64)
    if x0.shape != (r,):
        raise ValueError(f"x0 has shape {x0.shape}, expected ({r},)")
    if np.any(x0 < 0.0):
        raise ValueError("x0 must be nonnegative")
    ptr, v_indices, v_values = _one_column(v_indices, v_values, n)
    ids = _c64(ids, np.int64)
    if sorted(ids.tolist()) != list(range(r)):
        raise ValueError("ids must be a permutation of 0..r-1")
    if max_passes < 1:
        raise ValueError("max_passes must be >= 1")
    x = _c64(x0.reshape(r, 1)).copy()
    stats = np.zeros(_lib.STATS_LEN, dtype=np.int64)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.call("klnmf_sweep_range_passes", p(ptr), p(v_indices), p(v_values), p(at), p(_c64(sum_a)), p(x), 0, 1,
              p(ids), float(alpha), float(beta), tol.eps_grad, tol.eps_x, tol.eps_div, tol.inner_iter_cap,
              int(max_passes), r, n, 1, p(stats))
    return x[:, 0].copy(), SolveStats.from_array(stats)


def subproblem_objective(v_indices, v_values, at, x, alpha, beta, eps_div=1e-16):
    """D(v || Ax) + (alpha/2)||x||^2 + beta||x||_1 with 0 log 0 = 0
    (subproblem.py:169-181); a host helper in float64 (the dense sum of Ax is
    numpy's, not bit-identical to the reference's serial loop)."""
    at = _c64(at)
    x = _c64(x)
    ax = at.T @ x
    v_indices = _c64(v_indices, np.int64)
    v_values = _c64(v_values)
    data = float(ax.sum()) + float(np.sum(v_values * np.log(v_values / (ax[v_indices] + eps_div)) - v_values))
    return data + 0.5 * alpha * float(x @ x) + beta * float(np.abs(x).sum())


def kkt_violations(v_indices, v_values, at, sum_a, x, alpha, beta, tol: Tolerances = Tolerances()):
    """Per-coordinate stationarity violations at x (subproblem.py:184-201):
    bound coordinates need g >= -eps_grad, interior ones |g| <= max(eps_grad,
    eps_x * x_k * h_k).  Exact kernel on the GPU (klnmf_kkt_violation)."""
    import ctypes

    at = _c64(at)
    r, n = at.shape
    ptr, v_indices, v_values = _one_column(v_indices, v_values, n)
    x = _c64(np.asarray(x, dtype=np.float64).reshape(r, 1))
    out = np.zeros((r, 1))
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.call("klnmf_kkt_violation", p(ptr), p(v_indices), p(v_values), p(at), p(_c64(sum_a)), p(x), float(alpha),
              float(beta), tol.eps_grad, tol.eps_x, tol.eps_div, r, n, 1, p(out))
    return out[:, 0]
