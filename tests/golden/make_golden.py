"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``klnmf`` from /root/reference/pkg/src (read-only) and records
inputs and outputs of the reference's own hot-path functions:
``_kernels.sweep_range`` (via ``sweep``), ``_kernels.kl_data_term`` /
``full_objective``, ``DenseFactor.row_sums`` and ``factorize``, plus
fixed-iteration trajectories on configs C1 (fp64) and C2 (fp64 reference
run from fp32-rounded initial factors, the baseline of the fp32 mode).
The tests compare the oracle (bit-exact) and the CUDA path against these
files; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import klnmf  # noqa: E402  (the reference)
from klnmf import _kernels  # noqa: E402

from paper_1604_04026_b200 import synth  # noqa: E402  (generator only; deterministic numpy)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def random_case(rng, i):
    n_fix = int(rng.integers(1, 40))
    n_mov = int(rng.integers(1, 30))
    r = int(rng.integers(1, 9))
    density = float(rng.choice([0.0, 0.1, 0.4, 0.9]))
    mask = rng.random((n_fix, n_mov)) < density
    rows, cols = np.nonzero(mask)
    vals = np.round(rng.uniform(0.5, 6.0, size=rows.shape[0]))
    V = klnmf.SparseMatrix.from_coo(n_fix, n_mov, rows, cols, vals)
    at = rng.uniform(0.0, 2.0, size=(r, n_fix))
    at[rng.random(at.shape) < float(rng.choice([0.0, 0.3, 0.7]))] = 0.0
    mov = rng.uniform(0.0, 2.0, size=(r, n_mov))
    mov[rng.random(mov.shape) < float(rng.choice([0.0, 0.5]))] = 0.0
    alpha = float(rng.choice([0.0, 0.0, 0.1, 1.0]))
    beta = float(rng.choice([0.0, 0.0, 0.05, 0.5]))
    tol = klnmf.Tolerances(
        eps_grad=1e-10,
        eps_x=float(rng.choice([0.1, 0.1, 1e-3, 1e-8])),
        eps_div=float(rng.choice([1e-16, 1e-16, 1e-8])),
        inner_iter_cap=int(rng.choice([128, 128, 1, 3])),
    )
    ids = rng.permutation(r)
    fixed = klnmf.DenseFactor(at)
    sums = fixed.row_sums()
    moving = klnmf.DenseFactor(mov.copy())
    st = klnmf.sweep(V, fixed, moving, sums, ids, alpha, beta, tol=tol)
    return {
        "col_ptr": V.col_ptr, "row_idx": V.row_idx, "values": V.values, "n_fix": n_fix,
        "at": at, "sum_a": sums, "moving_in": mov, "ids": ids, "alpha": alpha, "beta": beta,
        "eps_grad": tol.eps_grad, "eps_x": tol.eps_x, "eps_div": tol.eps_div, "inner_cap": tol.inner_iter_cap,
        "moving_out": moving.values,
        "stats": np.array([st.cap_hits, st.degenerate, st.inner_iters, st.passes], dtype=np.int64),
    }


def save_cases(name, cases):
    flat = {"n_cases": np.array(len(cases))}
    for i, c in enumerate(cases):
        for k, v in c.items():
            flat[f"c{i}_{k}"] = np.asarray(v)
    np.savez_compressed(HERE / name, **flat)


def make_sweep_small():
    rng = np.random.default_rng(20240601)
    cases = [random_case(rng, i) for i in range(40)]
    save_cases("sweep_small.npz", cases)


def make_objective_small():
    rng = np.random.default_rng(7)
    cases = []
    for i in range(12):
        n, m, r = int(rng.integers(1, 30)), int(rng.integers(1, 30)), int(rng.integers(1, 7))
        mask = rng.random((n, m)) < float(rng.choice([0.05, 0.3, 0.8]))
        rows, cols = np.nonzero(mask)
        if rows.shape[0] == 0:
            rows, cols = np.array([0]), np.array([0])
        vals = np.round(rng.uniform(0.5, 9.0, size=rows.shape[0]))
        V = klnmf.SparseMatrix.from_coo(n, m, rows, cols, vals)
        w = rng.uniform(0.0, 1.5, size=(r, n))
        f = rng.uniform(0.0, 1.5, size=(r, m))
        w[rng.random(w.shape) < 0.3] = 0.0
        reg = klnmf.RegConfig(*[float(x) for x in rng.choice([0.0, 0.01, 0.5], size=4)])
        eps = float(rng.choice([1e-16, 1e-6]))
        kl, total = klnmf.full_objective(V, klnmf.DenseFactor(w), klnmf.DenseFactor(f), reg, eps_div=eps)
        data = _kernels.kl_data_term(V.col_ptr, V.row_idx, V.values, w, f, eps)
        cases.append({"col_ptr": V.col_ptr, "row_idx": V.row_idx, "values": V.values, "n_rows": n,
                      "w": w, "f": f, "reg": np.array([reg.alpha1, reg.alpha2, reg.beta1, reg.beta2]),
                      "eps_div": eps, "kl": kl, "total": total, "data": data})
    save_cases("objective_small.npz", cases)


def make_row_sums():
    rng = np.random.default_rng(11)
    cases = []
    for n in [1, 5, 7, 8, 9, 127, 128, 129, 255, 256, 1000, 1031, 4096, 10007, 30011]:
        r = int(rng.integers(1, 5)) if n <= 1031 else 1
        x = rng.random((r, n)) * float(10.0 ** rng.integers(-3, 4))
        x[rng.random(x.shape) < 0.2] = 0.0
        cases.append({"x": x, "sums": klnmf.DenseFactor(x).row_sums()})
    save_cases("row_sums.npz", cases)


def make_factorize_small():
    """The reference's factorize() on its own synthetic data, logged."""
    cases = []
    for seed, (n, m, r, reg, iters, tol) in enumerate([
        (20, 30, 3, klnmf.RegConfig(), 15, 0.0),
        (25, 50, 5, klnmf.RegConfig(alpha1=0.1, alpha2=0.05, beta1=0.02, beta2=0.2), 12, 0.0),
        (30, 45, 4, klnmf.RegConfig(beta1=0.2, beta2=0.2), 40, 1e-6),
    ]):
        V = klnmf.synthesize(klnmf.SyntheticSpec(n=n, m=m, r_true=3, sparsity=0.7, seed=seed))
        cfg = klnmf.NmfConfig(rank=r, reg=reg, max_outer_iters=iters, rel_obj_tol=tol, seed=seed + 1)
        res = klnmf.factorize(V, cfg)
        cases.append({"n": n, "m": m, "col_ptr": V.col_ptr, "row_idx": V.row_idx, "values": V.values,
                      "rank": r, "reg": np.array([reg.alpha1, reg.alpha2, reg.beta1, reg.beta2]),
                      "iters": iters, "rel_obj_tol": tol, "seed": seed + 1,
                      "w": res.factors.w.values, "f": res.factors.f.values,
                      "kl": res.log.column("kl_objective"), "total": res.log.column("total_objective"),
                      "sparsity_w": res.log.column("sparsity_w"), "sparsity_f": res.log.column("sparsity_f"),
                      "iterations_run": res.iterations_run, "converged": int(res.converged),
                      "stats": np.array([res.stats.cap_hits, res.stats.degenerate, res.stats.inner_iters,
                                         res.stats.passes])})
    save_cases("factorize_small.npz", cases)


def drive(V, w0, f0, r, reg, iters, seed, n_workers=8, keep=()):
    """The reference factorize loop driven through sweep() for a fixed
    iteration count (rel_obj_tol cannot stop it; SURVEY.md hazard P6)."""
    vt = V.transpose()
    w, f = klnmf.DenseFactor(w0.copy()), klnmf.DenseFactor(f0.copy())
    rng = np.random.default_rng(seed)
    out = {"ids": [], "kl": [], "total": [], "stats": [], "w_sha": [], "f_sha": []}
    snaps = {}
    for it in range(1, iters + 1):
        ids = rng.permutation(r).astype(np.int64)
        st_f = klnmf.sweep(V, w, f, w.row_sums(), ids, reg.alpha2, reg.beta2, n_workers=n_workers)
        st_w = klnmf.sweep(vt, f, w, f.row_sums(), ids, reg.alpha1, reg.beta1, n_workers=n_workers)
        kl, total = klnmf.full_objective(V, w, f, reg)
        out["ids"].append(ids)
        out["kl"].append(kl)
        out["total"].append(total)
        out["stats"].append([st_f.cap_hits, st_f.degenerate, st_f.inner_iters, st_f.passes,
                             st_w.cap_hits, st_w.degenerate, st_w.inner_iters, st_w.passes])
        out["w_sha"].append(sha(w.values))
        out["f_sha"].append(sha(f.values))
        if it in keep:
            snaps[f"w_it{it}"] = w.values.copy()
            snaps[f"f_it{it}"] = f.values.copy()
    res = {k: np.array(v) for k, v in out.items()}
    res.update(snaps)
    return res


def make_trajectory(name, spec, iters, keep=()):
    t0 = time.time()
    V = synth.generate(spec)
    w0, f0 = synth.initial_factors(spec, round_fp32=(spec.precision == "fp32"))
    res = drive(V, w0, f0, spec.rank, spec.reg, iters, spec.seed, keep=keep)
    res["v_sha"] = np.array(sha(V.col_ptr, V.row_idx, V.values))
    res["w0_sha"] = np.array(sha(w0))
    res["f0_sha"] = np.array(sha(f0))
    res["nnz"] = np.array(V.nnz)
    np.savez_compressed(HERE / name, **res)
    print(f"{name}: nnz={V.nnz} {time.time() - t0:.1f}s", flush=True)


def _small_matrix(rng, n, m, density):
    mask = rng.random((n, m)) < density
    rows, cols = np.nonzero(mask)
    return klnmf.SparseMatrix.from_coo(n, m, rows, cols, np.round(rng.uniform(0.5, 6.0, size=rows.shape[0])))


def make_mu_small():
    """_kernels.mu_update_range cases (empty columns included) and a short
    mu_factorize run (multiplicative.py)."""
    rng = np.random.default_rng(91)
    cases = []
    for i in range(20):
        n_fix, n_mov, r = int(rng.integers(1, 40)), int(rng.integers(1, 30)), int(rng.integers(1, 9))
        V = _small_matrix(rng, n_fix, n_mov, float(rng.choice([0.05, 0.3, 0.9])))
        fixed = rng.uniform(0.05, 2.0, size=(r, n_fix))
        mov = rng.uniform(0.05, 2.0, size=(r, n_mov))
        sums = klnmf.DenseFactor(fixed).row_sums()
        eps_mu = float(rng.choice([1e-16, 1e-8]))
        out = mov.copy()
        _kernels.mu_update_range(V.col_ptr, V.row_idx, V.values, fixed, out, sums, eps_mu, np.zeros(r), 0, n_mov)
        cases.append({"col_ptr": V.col_ptr, "row_idx": V.row_idx, "values": V.values, "n_fix": n_fix,
                      "fixed": fixed, "sum_fixed": sums, "moving_in": mov, "eps_mu": eps_mu, "moving_out": out})
    save_cases("mu_small.npz", cases)
    V = klnmf.synthesize(klnmf.SyntheticSpec(n=60, m=80, r_true=3, sparsity=0.8, seed=5))
    res = klnmf.mu_factorize(V, klnmf.NmfConfig(rank=4, max_outer_iters=12, rel_obj_tol=0.0, seed=6))
    np.savez_compressed(HERE / "mu_factorize.npz", col_ptr=V.col_ptr, row_idx=V.row_idx, values=V.values,
                        n_rows=V.n_rows, rank=4, seed=6, iters=12,
                        kl=np.array(res.log.column("kl_objective")),
                        total=np.array(res.log.column("total_objective")),
                        w=res.factors.w.values, f=res.factors.f.values)


def make_kkt_small():
    """subproblem.kkt_violations and multi-pass subproblem.solve_column."""
    rng = np.random.default_rng(92)
    kkt, solve = [], []
    for i in range(16):
        n_fix, n_mov, r = int(rng.integers(1, 40)), int(rng.integers(1, 12)), int(rng.integers(1, 9))
        V = _small_matrix(rng, n_fix, n_mov, float(rng.choice([0.1, 0.4, 0.9])))
        at = rng.uniform(0.0, 2.0, size=(r, n_fix))
        at[rng.random(at.shape) < 0.3] = 0.0
        sums = klnmf.DenseFactor(at).row_sums()
        x = rng.uniform(0.0, 2.0, size=(r, n_mov))
        x[rng.random(x.shape) < 0.4] = 0.0
        alpha = float(rng.choice([0.0, 0.1]))
        beta = float(rng.choice([0.0, 0.05]))
        tol = klnmf.Tolerances(eps_x=float(rng.choice([0.1, 1e-3])))
        out = np.stack([klnmf.kkt_violations(V.row_idx[V.col_ptr[j]:V.col_ptr[j + 1]],
                                             V.values[V.col_ptr[j]:V.col_ptr[j + 1]], at, sums, x[:, j],
                                             alpha, beta, tol) for j in range(n_mov)], axis=1)
        kkt.append({"col_ptr": V.col_ptr, "row_idx": V.row_idx, "values": V.values, "n_fix": n_fix, "at": at,
                    "sum_a": sums, "x": x, "alpha": alpha, "beta": beta, "eps_x": tol.eps_x, "out": out})
        j = int(rng.integers(0, n_mov))
        lo, hi = V.col_ptr[j], V.col_ptr[j + 1]
        ids = rng.permutation(r)
        max_passes = int(rng.choice([1, 3, 200]))
        xs, st = klnmf.solve_column(V.row_idx[lo:hi], V.values[lo:hi], at, sums, x[:, j], alpha, beta, ids, tol,
                                    max_passes=max_passes)
        solve.append({"v_idx": V.row_idx[lo:hi], "v_val": V.values[lo:hi], "at": at, "sum_a": sums,
                      "x0": x[:, j], "ids": ids, "alpha": alpha, "beta": beta, "eps_x": tol.eps_x,
                      "max_passes": max_passes, "x": xs,
                      "stats": np.array([st.cap_hits, st.degenerate, st.inner_iters, st.passes], dtype=np.int64)})
    save_cases("kkt_small.npz", kkt)
    save_cases("solve_column_small.npz", solve)


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"small", "c1", "c2", "baselines"}
    if "baselines" in which:
        make_mu_small()
        make_kkt_small()
        print("baseline fixtures done", flush=True)
    _kernels.warm_up()
    if "small" in which:
        make_sweep_small()
        make_objective_small()
        make_row_sums()
        make_factorize_small()
        print("small fixtures done", flush=True)
    if "c1" in which:
        make_trajectory("c1_trajectory.npz", synth.CONFIGS["C1"], 30, keep=(1, 2))
    if "c2" in which:
        make_trajectory("c2_trajectory.npz", synth.CONFIGS["C2"], 50)
