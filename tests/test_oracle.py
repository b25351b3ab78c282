"""Pin the oracle (C restatement) against golden vectors produced by the
reference itself.  CPU only."""

import numpy as np
import pytest

import golden_cases as G
from oracle import oracle as O
import paper_2603_01915_b200 as P

WITH_BYTES = [n for n in G.names() if "container" in G.load(n)]


@pytest.mark.parametrize("name", WITH_BYTES)
def test_oracle_decode_matches_reference(name):
    rec = G.load(name)
    c = O.parse(rec["container"].tobytes())
    row_start, cols, vals = O.decode(c)
    prec = int(rec["precision"])
    vdt = np.float64 if prec == 8 else np.float32
    assert np.array_equal(row_start, rec["row_start"])
    assert np.array_equal(cols, rec["col_idx"])
    ui = np.uint64 if prec == 8 else np.uint32
    assert np.array_equal(vals.view(ui), rec["values"].astype(vdt).view(ui))


@pytest.mark.parametrize("name", [n for n in WITH_BYTES if "spmv" in G.load(n)])
@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_spmv_bitwise_reference(name, threads):
    rec = G.load(name)
    c = O.parse(rec["container"].tobytes())
    out = O.spmv(c, rec["x"], rec["y"], threads=threads)
    assert G.same_bits_or_nan(out, rec["spmv"])
    assert G.same_bits_or_nan(out, rec["reference_spmv"])


def test_oracle_rejects_truncated_stream():
    rec = G.load("fig1_f64")
    c = O.parse(rec["container"].tobytes())
    c.stream = c.stream[:-1]
    c.directory = c.directory.copy()
    with pytest.raises(O.OracleError):
        O.decode(c)


def test_oracle_detects_consumption_mismatch():
    rec = G.load("laplacian_g20_f32")
    c = O.parse(rec["container"].tobytes())
    d = c.directory.copy()
    d[1] += 1
    c.directory = d
    with pytest.raises(O.OracleError):
        O.decode(c)


@pytest.mark.parametrize("name", [n for n in G.names() if "reference_spmv" in G.load(n)])
def test_package_reference_spmv_bitwise(name):
    """The package's reference_spmv (sparse.py:330-353 restated; D13) equals
    the reference's own output bit for bit."""
    rec = G.load(name)
    m = G.matrix(rec)
    if G.encode_kwargs(rec).get("value_width") == 4:  # the golden was made on the f32 matrix
        m = P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx, m.values.astype(np.float32))
    out = P.reference_spmv(m, rec["x"], rec["y"])
    assert G.same_bits_or_nan(out, rec["reference_spmv"])
