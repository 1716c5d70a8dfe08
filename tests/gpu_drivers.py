"""Fixed-iteration drivers of the device plan for the parity tests."""

from __future__ import annotations

import hashlib

import numpy as np


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gpu_drive(V, w0, f0, r, reg, iters, seed, precision="fp64", log=True, hashes=True, tol=None):
    """factorize's loop (solver.py:283-317) on a DevicePlan for exactly
    `iters` iterations; returns objectives, factor hashes and final factors."""
    from paper_1604_04026_b200.plan import DevicePlan
    from paper_1604_04026_b200.subproblem import Tolerances

    tol = tol or Tolerances()
    plan = DevicePlan(V, r, precision)
    rng = np.random.default_rng(seed)
    ids = rng.permutation(r).astype(np.int64)
    plan.set_factors(w0, f0, order=ids)
    out = {"kl": [], "total": [], "w_sha": [], "f_sha": [], "ids": [], "stats": []}
    for _ in range(iters):
        ids_next = rng.permutation(r).astype(np.int64)
        plan.half_step("F", ids, alpha=reg.alpha2, beta=reg.beta2, tol=tol)
        st_f = plan.take_stats()
        plan.half_step("W", ids, ids_next, alpha=reg.alpha1, beta=reg.beta1, tol=tol)
        st_w = plan.take_stats()
        out["ids"].append(ids)
        out["stats"].append([st_f.cap_hits, st_f.degenerate, st_f.inner_iters, st_f.passes,
                             st_w.cap_hits, st_w.degenerate, st_w.inner_iters, st_w.passes])
        if log:
            kl, total, _, _ = plan.objective(reg.alpha1, reg.alpha2, reg.beta1, reg.beta2, tol.eps_div)
            out["kl"].append(kl)
            out["total"].append(total)
        if hashes:
            w, f = plan.get_factors()
            out["w_sha"].append(sha(w))
            out["f_sha"].append(sha(f))
        ids = ids_next
    res = {k: np.array(v) for k, v in out.items()}
    res["w"], res["f"] = plan.get_factors()
    res["plan"] = plan
    return res
