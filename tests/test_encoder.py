"""Byte identity of the C++ encoder with the reference encoder (CPU only).

Goldens: tests/golden/cases/*.npz, produced by running the reference's
encode_matrix + serialize (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

import golden_cases as G
import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth


@pytest.mark.parametrize("name", G.names())
def test_encode_byte_identical_to_reference(name):
    rec = G.load(name)
    c = P.encode_matrix(G.matrix(rec), **G.encode_kwargs(rec))
    blob = P.serialize(c)
    assert hashlib.sha256(blob).hexdigest() == str(rec["sha256"])
    assert len(c.stream) == int(rec["nwords"])
    assert P.size_bytes(c) == int(rec["size_bytes"])
    m = G.matrix(rec)
    assert [P.format_size_bytes(m, f, c.precision) for f in ("coo", "csr", "sell")] == rec["fmt_sizes"].tolist()


@pytest.mark.parametrize("name", [n for n in G.names() if "container" in G.load(n)])
def test_deserialize_reference_bytes(name):
    rec = G.load(name)
    blob = rec["container"].tobytes()
    c = P.deserialize(blob)
    assert P.serialize(c) == blob
    mine = P.encode_matrix(G.matrix(rec), **G.encode_kwargs(rec))
    assert mine == c


@pytest.mark.parametrize("threads", [1, 2, 5, 0])
def test_encoder_thread_count_invariant(threads):
    m = synth.banded(3000, 9, levels=17, seed=5)
    ref = P.serialize(P.encode_matrix(m, threads=1))
    assert P.serialize(P.encode_matrix(m, threads=threads)) == ref


def test_rejects_descending_columns():
    m = P.CsrMatrix(1, 5, np.array([0, 2]), np.array([3, 1]), np.array([1.0, 2.0]))
    with pytest.raises(P.ParameterError):
        P.encode_matrix(m)


def test_rejects_out_of_range_column():
    m = P.CsrMatrix(1, 3, np.array([0, 1]), np.array([3]), np.array([1.0]))
    with pytest.raises(P.ParameterError):
        P.encode_matrix(m)


def test_rejects_bad_row_start():
    m = P.CsrMatrix(2, 3, np.array([0, 1]), np.array([0]), np.array([1.0]))
    with pytest.raises(P.ParameterError):
        P.encode_matrix(m)


def test_rejects_non_production_geometry():
    with pytest.raises(P.ParameterError):
        P.encode_matrix(synth.fig1(), params=P.DtansParams.toy())


def test_value_width_cast():
    c = P.encode_matrix(synth.fig1(), value_width=4)
    assert c.precision == 4 and c.value_dtype == np.float32


def test_container_fields_fig1():
    c = P.encode_matrix(synth.fig1())
    # Fig.1 stream words with the default seed
    assert [f"{w:08x}" for w in c.stream] == ["1708f217"] * 4 + [
        "08f2c0e2", "08f24082", "08f21708", "08f21708", "cc8f08f2", "cc170b13", "f210c8f2", "f2f2df9d"]
    assert c.directory.tolist() == [0, 12]
    assert c.row_symbols.tolist() == [4, 4, 2, 2]


def test_deserialize_rejects_corruption():
    blob = bytearray(P.serialize(P.encode_matrix(synth.fig1())))
    with pytest.raises(P.ContainerError):
        P.deserialize(bytes(blob[:-5]))
    blob[100] ^= 1
    with pytest.raises(P.ContainerError):
        P.deserialize(bytes(blob))
    with pytest.raises(P.ContainerError):
        P.deserialize(b"XXXX" + bytes(60))


def test_tables_api():
    c = P.encode_matrix(synth.fig1())
    t = c.delta_tables
    assert t.k == 4096
    assert t.has_symbol(1) and t.base_of(1) >= 1
    assert t.pad_symbol() in t.retained_symbols()
    assert sum(1 for s in t.symbols if s is P.ESCAPE) == int(t.escape.sum())


def test_sort_rows_by_length_is_a_row_permutation():
    m = synth.rmat(10, 5000, seed=1)
    for window in (None, 100):
        pm, perm = P.sort_rows_by_length(m, window)
        assert sorted(perm.tolist()) == list(range(m.rows))
        nz = np.diff(m.row_start)
        assert np.array_equal(np.diff(pm.row_start), nz[perm.astype(np.int64)])
        for i in (0, 7, m.rows - 1):
            r = int(perm[i])
            assert np.array_equal(pm.row_cols(i), m.row_cols(r))
            assert np.array_equal(pm.row_values(i), m.row_values(r))
        pm.validate()
