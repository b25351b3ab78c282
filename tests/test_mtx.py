"""MatrixMarket ingestion (reference sparse.py:205-264; the reference's own
test cases, tests/test_sparse.py:25-100, restated), plus a cross-check
against the reference parser when /root/reference is importable here."""

import os
import sys

import numpy as np
import pytest

import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import MtxFormatError, coo_to_csr, parse_mtx

FIG_MTX = """%%MatrixMarket matrix coordinate real general
4 4 6
1 2 7.0
1 4 5.0
2 1 3.0
2 3 2.0
3 2 4.0
4 4 1.0
"""


def test_running_example_csr():
    m = coo_to_csr(parse_mtx(FIG_MTX))
    assert m.values.tolist() == [7, 5, 3, 2, 4, 1]
    assert m.col_idx.tolist() == [1, 3, 0, 2, 1, 3]
    assert m.row_start.tolist() == [0, 2, 4, 5, 6]


def test_symmetric_mirrors_off_diagonal():
    coo = parse_mtx("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 2.0\n2 1 3.0\n")
    assert set(zip(coo.row_idx.tolist(), coo.col_idx.tolist(), coo.values.tolist())) == {
        (0, 0, 2.0), (1, 0, 3.0), (0, 1, 3.0)}


def test_pattern_and_integer_fields():
    coo = parse_mtx("%%MatrixMarket matrix coordinate pattern general\n3 3 1\n3 1\n")
    assert (coo.row_idx[0], coo.col_idx[0], coo.values[0]) == (2, 0, 1.0)
    assert parse_mtx("%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 7\n").values[0] == 7.0


def test_comments_and_blank_lines_skipped():
    text = "%%MatrixMarket matrix coordinate real general\n% a comment\n\n2 2 1\n% another\n2 2 9.0\n"
    assert parse_mtx(text).nnz == 1


@pytest.mark.parametrize("text", [
    "no banner\n1 1 0\n",
    "%%MatrixMarket matrix array real general\n1 1\n1.0\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n2 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n1.5 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n",
])
def test_rejects_malformed(text):
    with pytest.raises(MtxFormatError):
        parse_mtx(text)


def test_duplicates_rejected_as_mtx_error():
    with pytest.raises(MtxFormatError):
        coo_to_csr(parse_mtx("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1 1 2.0\n"))


def test_read_mtx_roundtrip_through_encoder(tmp_path):
    p = tmp_path / "fig.mtx"
    p.write_text(FIG_MTX)
    m = P.read_mtx(str(p))
    c = P.encode_matrix(m)
    assert P.size_bytes(c) > 0 and c.nnz == 6


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
def test_matches_reference_parser():
    sys.path.insert(0, REF)
    try:
        import csrdtans as R
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(3)
    for sym in ("general", "symmetric"):
        n, k = 50, 200
        r = rng.integers(1, n + 1, k)
        c = rng.integers(1, n + 1, k)
        if sym == "symmetric":
            r, c = np.maximum(r, c), np.minimum(r, c)
        key = np.unique(r * 1000 + c)
        r, c = key // 1000, key % 1000
        lines = [f"%%MatrixMarket matrix coordinate real {sym}", f"{n} {n} {len(r)}"]
        lines += [f"{a} {b} {rng.standard_normal():.17g}" for a, b in zip(r, c)]
        text = "\n".join(lines) + "\n"
        a, b = parse_mtx(text), R.parse_mtx(text)
        for f in ("row_idx", "col_idx", "values"):
            assert np.array_equal(getattr(a, f), getattr(b, f))


def test_save_load_mmap_roundtrip(tmp_path):
    """save() streams byte-identical CDTA bytes; load() memory-maps them."""
    from paper_2603_01915_b200 import synth
    m = synth.laplacian_2d(120)
    c = P.encode_matrix(m)
    path = tmp_path / "lap.cdta"
    n = P.save(c, str(path))
    data = path.read_bytes()
    assert n == len(data) and data == P.serialize(c)
    c2 = P.load(str(path))
    assert c2 == c
    assert not c2.stream.flags.owndata  # a view of the mapping, not a copy


def test_sort_symmetric_by_degree_is_pap():
    from paper_2603_01915_b200 import synth
    m = synth.rmat(9, 3000, seed=2)
    b, perm = P.sort_symmetric_by_degree(m)
    import scipy.sparse as sp
    A = sp.csr_matrix((m.values, m.col_idx, m.row_start), shape=(m.rows, m.cols))
    B = sp.csr_matrix((b.values, b.col_idx, b.row_start), shape=(b.rows, b.cols))
    p = perm.astype(np.int64)
    assert (A[p][:, p] != B).nnz == 0
    nnz_row = np.diff(b.row_start)
    assert np.all(np.diff(nnz_row) <= 0)  # rows by descending length
    for i in range(b.rows):  # columns ascending within rows
        assert np.all(np.diff(b.col_idx[b.row_start[i]:b.row_start[i + 1]]) > 0)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
@pytest.mark.parametrize("text", [
    "no banner\n1 1 0\n", "", "%%MatrixMarket matrix\n",
    "%%MatrixMarket vector coordinate real general\n1 1 0\n",
    "%%MatrixMarket matrix array real general\n1 1\n1.0\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n",
    "%%MatrixMarket matrix coordinate real general\n",
    "%%MatrixMarket matrix coordinate real general\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n1 a 1\n",
    "%%MatrixMarket matrix coordinate real general\n-1 1 0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n2 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n0 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1 2\n2 2\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n1.5 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n",
    "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 3\n",
])
def test_error_behaviour_matches_reference(text):
    """Same accept/reject decision and the same message as the reference."""
    sys.path.insert(0, REF)
    try:
        import csrdtans as R
    finally:
        sys.path.remove(REF)

    def run(f):
        try:
            coo = f(text)
            return ("ok", coo.rows, coo.cols, coo.row_idx.tolist(), coo.col_idx.tolist(), coo.values.tolist())
        except Exception as e:  # noqa: BLE001 - compare the exception itself
            return ("err", type(e).__name__, str(e))
    assert run(parse_mtx) == run(R.parse_mtx)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
def test_coo_to_csr_matches_reference():
    sys.path.insert(0, REF)
    try:
        import csrdtans as R
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(5)
    for n, k in ((1, 1), (7, 20), (300, 5000), (64, 0)):
        key = rng.choice(n * n, min(k, n * n), replace=False)
        r, c = np.divmod(key, n)
        v = rng.standard_normal(len(r))
        a = coo_to_csr(P.CooMatrix(n, n, r, c, v))
        b = R.coo_to_csr(R.CooMatrix(n, n, r, c, v))
        assert np.array_equal(a.row_start, b.row_start) and np.array_equal(a.col_idx, b.col_idx)
        assert np.array_equal(a.values, b.values)
