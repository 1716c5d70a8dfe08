"""Native MatrixMarket reader against the
reference's acceptance rules (pkg/tests/test_sparse.py:133-200 restated) and
round trips.  CPU only: the reader is host code in libklnmf.so."""
import numpy as np
import pytest

from paper_1604_04026_b200 import (
    DenseFactor,
    DuplicateEntryError,
    MatrixMarketError,
    SparseMatrix,
    load_matrix_market,
    save_matrix_market,
    save_tsv,
)


def write_mm(path, n, m, triples, header="%%MatrixMarket matrix coordinate real general"):
    lines = [header, f"{n} {m} {len(triples)}"] + [f"{i} {j} {v}" for i, j, v in triples]
    path.write_text("\n".join(lines) + "\n")


def random_sparse(rng, n, m, density=0.3):
    mask = rng.random((n, m)) < density
    rows, cols = np.nonzero(mask)
    return SparseMatrix.from_coo(n, m, rows, cols, rng.uniform(0.1, 5.0, size=rows.shape[0]))


def test_identity_file(tmp_path):
    write_mm(tmp_path / "id.mtx", 2, 2, [(1, 1, 1.0), (2, 2, 3.0)])
    m = load_matrix_market(tmp_path / "id.mtx")
    assert m.nnz == 2 and m.col_ptr.tolist() == [0, 1, 2] and m.to_dense()[1, 1] == 3.0


def test_integer_field_and_case_insensitive_header(tmp_path):
    (tmp_path / "i.mtx").write_text("%%MatrixMarket MATRIX Coordinate INTEGER general\n2 2 1\n1 2 7\n")
    assert load_matrix_market(tmp_path / "i.mtx").to_dense()[0, 1] == 7.0


def test_comments_blank_lines_and_whitespace(tmp_path):
    (tmp_path / "c.mtx").write_text(
        "%%MatrixMarket matrix coordinate real general\n% a comment\n  % indented comment\n2 3 2\n"
        "\n1 1 1.5\n   % between\n\t2  3\t 2.5e0  \r\n")
    m = load_matrix_market(tmp_path / "c.mtx")
    assert m.nnz == 2 and m.to_dense()[1, 2] == 2.5


@pytest.mark.parametrize("triples,match", [
    ([(1, 1, -1.0)], "negative"),
    ([(1, 1, 0.0)], "zero"),
    ([(3, 1, 1.0)], "out of bounds"),
    ([(1, 0, 1.0)], "out of bounds"),
])
def test_rejected_values(tmp_path, triples, match):
    write_mm(tmp_path / "x.mtx", 2, 2, triples)
    with pytest.raises(MatrixMarketError, match=match):
        load_matrix_market(tmp_path / "x.mtx")


def test_negative_message_matches_reference_format(tmp_path):
    write_mm(tmp_path / "n.mtx", 2, 2, [(1, 2, -2.5)])
    with pytest.raises(MatrixMarketError, match=r"negative entry -2\.5 at \(1, 2\)"):
        load_matrix_market(tmp_path / "n.mtx")


def test_duplicate_rejected(tmp_path):
    write_mm(tmp_path / "d.mtx", 2, 2, [(1, 1, 1.0), (1, 1, 2.0)])
    with pytest.raises(DuplicateEntryError):
        load_matrix_market(tmp_path / "d.mtx")


@pytest.mark.parametrize("text,match", [
    ("%%MatrixMarket matrix array real general\n2 2\n1.0\n", "header"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 1.0\n", "header"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 0x1p0\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "expected 2"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 x 1\n1 1 1.0\n", "size line"),
    ("", "header"),
])
def test_malformed_rejected(tmp_path, text, match):
    (tmp_path / "m.mtx").write_text(text)
    with pytest.raises(MatrixMarketError, match=match):
        load_matrix_market(tmp_path / "m.mtx")


def test_first_error_in_file_order(tmp_path):
    write_mm(tmp_path / "o.mtx", 3, 3, [(1, 1, 1.0), (2, 2, -1.0), (9, 9, 1.0)])
    with pytest.raises(MatrixMarketError, match="negative"):
        load_matrix_market(tmp_path / "o.mtx")


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        load_matrix_market(tmp_path / "nope.mtx")


def test_nan_rejected_by_matrix_validation(tmp_path):
    write_mm(tmp_path / "nan.mtx", 2, 2, [(1, 1, "nan")])
    with pytest.raises(ValueError):
        load_matrix_market(tmp_path / "nan.mtx")


@pytest.mark.parametrize("seed", range(4))
def test_round_trip_identical(tmp_path, seed):
    rng = np.random.default_rng(seed)
    m = random_sparse(rng, int(rng.integers(1, 30)), int(rng.integers(1, 30)))
    save_matrix_market(m, tmp_path / "r.mtx")
    back = load_matrix_market(tmp_path / "r.mtx")
    assert np.array_equal(back.col_ptr, m.col_ptr)
    assert np.array_equal(back.row_idx, m.row_idx)
    assert np.array_equal(back.values, m.values)  # repr() round-trips every double


def test_large_file_parallel_parse_matches(tmp_path):
    """Several MB so the reader splits the body across threads."""
    rng = np.random.default_rng(7)
    n, m = 5000, 4000
    rows = rng.integers(0, n, size=400000)
    cols = rng.integers(0, m, size=400000)
    key = np.unique(rows * m + cols)
    rows, cols = key // m, key % m
    vals = rng.integers(1, 9, size=key.shape[0]).astype(np.float64) / 4
    ref = SparseMatrix.from_coo(n, m, rows, cols, vals)
    save_matrix_market(ref, tmp_path / "big.mtx")
    back = load_matrix_market(tmp_path / "big.mtx")
    assert back.nnz == ref.nnz
    assert np.array_equal(back.col_ptr, ref.col_ptr) and np.array_equal(back.row_idx, ref.row_idx)
    assert np.array_equal(back.values, ref.values)


def test_factor_outputs(tmp_path):
    f = DenseFactor(np.array([[0.0, 1.5], [2.0, 0.0]]))
    save_matrix_market(f, tmp_path / "f.mtx")
    back = load_matrix_market(tmp_path / "f.mtx")
    assert np.array_equal(back.to_dense(), f.values)
    save_tsv(f, tmp_path / "f.tsv")
    assert np.array_equal(np.loadtxt(tmp_path / "f.tsv", delimiter="\t"), f.values)
