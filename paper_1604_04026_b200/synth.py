"""Seeded planted-topic count matrices for the BASELINE.json configs C1-C5.

The reference's own generator (pkg/src/klnmf/synth.py) samples uniform cells
and cannot express these configs, so this is new.  Model
(BASELINE.json "configs"): T planted topics; topic-feature weights
phi_t ~ Dirichlet(c * n * pop) with c = 0.05 and pop the feature popularity
(uniform, or Zipf(s) normalised), so each topic is sparse and the corpus-wide
feature frequencies follow pop; instance-topic weights theta_j ~
Dirichlet(0.1); instance lengths ~ Poisson(mean) or lognormal with the stated
mean and sigma; tokens drawn multinomially and aggregated into integer counts
(V is features x instances, stored CSC: columns are instances).

Seeded synthetic inputs stand in for the paper's corpora,
which are not available; nnz is whatever the stated distributions give
(C2/C3 come out below BASELINE.json's "~" figures).
"""

from __future__ import annotations

import dataclasses

import numpy as np

from .sparse import SparseMatrix
from .solver import RegConfig

__all__ = ["ConfigSpec", "CONFIGS", "DeviceMatrix", "generate", "generate_coo", "generate_device", "initial_factors"]


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    name: str
    n: int                 # features (rows of V)
    m: int                 # instances (columns of V)
    topics: int
    zipf: float | None     # feature popularity exponent (None = uniform)
    length: tuple          # ("poisson", mean) or ("lognormal", mean, sigma)
    rank: int
    reg: RegConfig
    iters: int
    precision: str
    seed: int

    def scaled(self, m: int, n: int | None = None) -> "ConfigSpec":
        """Same generative model with fewer instances/features (tests)."""
        return dataclasses.replace(self, m=m, n=self.n if n is None else n)


CONFIGS = {
    "C1": ConfigSpec("C1", 2000, 1500, 10, None, ("poisson", 200.0), 10, RegConfig(), 30, "fp64", 1),
    "C2": ConfigSpec("C2", 6906, 3430, 10, 1.1, ("lognormal", 136.0, 1.0), 50, RegConfig(), 50, "fp32", 2),
    "C3": ConfigSpec("C3", 28102, 39861, 100, 1.05, ("lognormal", 160.0, 1.0), 100,
                     RegConfig(beta1=0.1, beta2=0.1), 50, "fp32", 3),
    "C4": ConfigSpec("C4", 102660, 300000, 200, 1.0, ("lognormal", 330.0, 0.8), 100,
                     RegConfig(alpha1=0.01, alpha2=0.01), 30, "fp32", 4),
    "C5": ConfigSpec("C5", 141043, 8200000, 500, 1.0, ("lognormal", 90.0, 1.2), 100,
                     RegConfig(beta2=0.1), 20, "fp32", 5),
}


def _popularity(n: int, s: float | None) -> np.ndarray:
    if s is None:
        return np.full(n, 1.0 / n)
    w = 1.0 / np.arange(1, n + 1, dtype=np.float64) ** s
    return w / w.sum()


def _lengths(rng, spec: ConfigSpec, m: int) -> np.ndarray:
    kind = spec.length[0]
    if kind == "poisson":
        return rng.poisson(spec.length[1], size=m).astype(np.int64)
    mean, sigma = spec.length[1], spec.length[2]
    mu = np.log(mean) - 0.5 * sigma * sigma
    return np.maximum(1, np.rint(rng.lognormal(mu, sigma, size=m))).astype(np.int64)


def generate_coo(spec: ConfigSpec, chunk: int = 50_000):
    """(rows, cols, counts) of V, columns ascending then rows ascending."""
    rng = np.random.default_rng(spec.seed)
    n, m, T = spec.n, spec.m, spec.topics
    conc = 0.05 * n * _popularity(n, spec.zipf)
    phi = rng.gamma(np.broadcast_to(conc, (T, n)))
    phi /= phi.sum(axis=1, keepdims=True)
    cdf = np.cumsum(phi, axis=1)
    cdf[:, -1] = 1.0
    theta = rng.gamma(0.1, size=(m, T))
    theta /= theta.sum(axis=1, keepdims=True)
    lengths = _lengths(rng, spec, m)
    rows_out, cols_out, vals_out = [], [], []
    for c0 in range(0, m, chunk):
        c1 = min(m, c0 + chunk)
        tc = rng.multinomial(lengths[c0:c1], theta[c0:c1])  # (chunk, T) token counts per topic
        docs, feats = [], []
        for t in range(T):
            cnt = tc[:, t]
            tot = int(cnt.sum())
            if tot == 0:
                continue
            docs.append(np.repeat(np.arange(c0, c1, dtype=np.int64), cnt))
            u = rng.random(tot)
            feats.append(np.minimum(np.searchsorted(cdf[t], u, side="right"), n - 1))
        if not docs:
            continue
        d = np.concatenate(docs)
        f = np.concatenate(feats)
        key, cnt = np.unique(d * n + f, return_counts=True)
        cols_out.append(key // n)
        rows_out.append(key % n)
        vals_out.append(cnt.astype(np.float64))
    rows = np.concatenate(rows_out) if rows_out else np.zeros(0, np.int64)
    cols = np.concatenate(cols_out) if cols_out else np.zeros(0, np.int64)
    vals = np.concatenate(vals_out) if vals_out else np.zeros(0)
    return rows, cols, vals


def generate(spec: ConfigSpec) -> SparseMatrix:
    """The config's V as a CSC SparseMatrix (entries already sorted)."""
    rows, cols, vals = generate_coo(spec)
    col_ptr = np.zeros(spec.m + 1, dtype=np.int64)
    np.cumsum(np.bincount(cols, minlength=spec.m), out=col_ptr[1:])
    return SparseMatrix(spec.n, spec.m, col_ptr, rows, vals)


def initial_factors(spec: ConfigSpec, round_fp32: bool | None = None):
    """W, F ~ Uniform(0,1) from default_rng(seed), W first (BASELINE.json configs).

    Rounded to fp32 for fp32 configs so both sides start from the same
    representable point."""
    rng = np.random.default_rng(spec.seed)
    w = rng.random((spec.rank, spec.n))
    f = rng.random((spec.rank, spec.m))
    if round_fp32 is None:
        round_fp32 = spec.precision == "fp32"
    if round_fp32:
        w = w.astype(np.float32).astype(np.float64)
        f = f.astype(np.float32).astype(np.float64)
    return w, f


@dataclasses.dataclass
class DeviceMatrix:
    """A CSC matrix resident on the GPU (col_ptr int64, row_idx int32, values
    float32/float64 torch tensors), as DevicePlan consumes it -- the C5-scale
    input never exists in host memory."""

    n_rows: int
    n_cols: int
    col_ptr: "object"
    row_idx: "object"
    values: "object"
    col_ptr_host: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_idx.shape[0])

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def to_host(self) -> SparseMatrix:
        return SparseMatrix(self.n_rows, self.n_cols, self.col_ptr_host.copy(),
                            self.row_idx.cpu().numpy().astype(np.int64), self.values.cpu().numpy().astype(np.float64))


def generate_device(spec: ConfigSpec, device=None, precision: str | None = None) -> DeviceMatrix:
    """The config's generative model drawn on the GPU (csrc/synth_gen.cu):
    same distributions as ``generate``, a different (counter-based) random
    stream, so a statistically equivalent -- not identical -- matrix."""
    import ctypes

    import torch

    from . import _lib

    precision = precision or spec.precision
    fp32 = precision == "fp32"
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        col_ptr = torch.empty(spec.m + 1, dtype=torch.int64, device=dev)
        nnz = ctypes.c_int64()
        rows_p, vals_p = ctypes.c_void_p(), ctypes.c_void_p()
        kind = 0 if spec.length[0] == "poisson" else 1
        sigma = spec.length[2] if kind == 1 else 0.0
        _lib.call("klnmf_synth_build", int(spec.seed), spec.n, spec.m, spec.topics,
                  float(spec.zipf) if spec.zipf is not None else 0.0, kind, float(spec.length[1]), float(sigma),
                  int(fp32), ctypes.byref(nnz), col_ptr.data_ptr(), ctypes.byref(rows_p), ctypes.byref(vals_p),
                  stream)
        k = nnz.value
        rows = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(k, 1), dtype=torch.float32 if fp32 else torch.float64, device=dev)
        _lib.call("klnmf_synth_fetch", rows_p, vals_p, k, int(fp32), rows.data_ptr(), vals.data_ptr(), stream)
        return DeviceMatrix(spec.n, spec.m, col_ptr, rows[:k], vals[:k], col_ptr.cpu().numpy())
