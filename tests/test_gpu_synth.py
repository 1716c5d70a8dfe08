"""Device-side corpus generator: valid CSC,
deterministic, and the same generative model as the host generator
(statistics, not the identical matrix: the random streams differ)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check_csc(V):
    ptr = V.col_ptr_host
    assert ptr[0] == 0 and ptr[-1] == V.nnz and np.all(np.diff(ptr) >= 0)
    rows = V.row_idx.cpu().numpy().astype(np.int64)
    vals = V.values.cpu().numpy()
    assert rows.min() >= 0 and rows.max() < V.n_rows
    cols = np.repeat(np.arange(V.n_cols), np.diff(ptr))
    key = cols * V.n_rows + rows
    assert np.all(np.diff(key) > 0)  # strictly increasing rows per column, columns ascending
    assert np.all(vals >= 1.0) and np.all(vals == np.round(vals))
    return rows, vals


@pytest.mark.parametrize("name,m", [("C1", 1500), ("C2", 3430), ("C4", 20000)])
def test_device_generator_matches_host_model(cuda_ok, name, m):
    from paper_1604_04026_b200 import synth

    spec = synth.CONFIGS[name].scaled(m=m)
    D = synth.generate_device(spec)
    rows, vals = _check_csc(D)
    H = synth.generate(spec)
    # same model: corpus size, tokens and column-length distribution agree closely
    assert abs(D.nnz - H.nnz) / H.nnz < 0.05, (D.nnz, H.nnz)
    assert abs(vals.sum() - H.values.sum()) / H.values.sum() < 0.05
    dl, hl = np.diff(D.col_ptr_host), np.diff(H.col_ptr)
    for q in (0.1, 0.5, 0.9):
        assert abs(np.quantile(dl, q) - np.quantile(hl, q)) <= 0.1 * np.quantile(hl, q) + 2
    # feature popularity: the share of the 1% most frequent features
    def top_share(r, n):
        c = np.sort(np.bincount(r, minlength=n))[::-1]
        return c[: max(1, n // 100)].sum() / c.sum()
    assert abs(top_share(rows, spec.n) - top_share(H.row_idx, spec.n)) < 0.05


def test_device_generator_deterministic_and_plan_ready(cuda_ok):
    import torch

    from paper_1604_04026_b200 import synth
    from paper_1604_04026_b200.plan import DevicePlan

    spec = synth.CONFIGS["C3"].scaled(m=5000)
    a, b = synth.generate_device(spec), synth.generate_device(spec)
    assert torch.equal(a.col_ptr, b.col_ptr) and torch.equal(a.row_idx, b.row_idx)
    assert torch.equal(a.values, b.values)
    w0, f0 = synth.initial_factors(spec)
    plan = DevicePlan(a, spec.rank, "fp32")  # straight from device memory
    ids = np.random.default_rng(0).permutation(spec.rank)
    plan.set_factors(w0, f0, order=ids)
    kl0 = plan.objective()[0]
    plan.half_step("F", ids, alpha=spec.reg.alpha2, beta=spec.reg.beta2)
    plan.half_step("W", ids, alpha=spec.reg.alpha1, beta=spec.reg.beta1)
    assert plan.objective()[0] < kl0
    host = a.to_host()
    assert host.nnz == a.nnz and np.array_equal(host.col_ptr, a.col_ptr_host)
