"""CSR inputs, delta/value symbol domains and baseline-format sizes.

Mirrors the hot-path helpers of /root/reference/pkg/src/csrdtans/sparse.py:
``CsrMatrix`` (:54-106), ``coo_to_csr`` (:133-144), ``format_size_bytes``
(:185-198), ``matrix_deltas`` (:289-299), ``value_patterns`` (:302-309), and
the MatrixMarket reader ``parse_mtx`` (:205-264) that feeds the path with
SuiteSparse matrices.  The graph-entropy experiment is
out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError


class MtxFormatError(ValueError):
    """Malformed MatrixMarket content or duplicate coordinates (sparse.py:22)."""


@dataclass
class CooMatrix:
    rows: int
    cols: int
    row_idx: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.values)

    def validate(self) -> None:
        if not (len(self.row_idx) == len(self.col_idx) == len(self.values)):
            raise ParameterError("COO arrays must have equal length")
        if self.nnz and (
            self.row_idx.min() < 0 or self.row_idx.max() >= self.rows
            or self.col_idx.min() < 0 or self.col_idx.max() >= self.cols
        ):
            raise ParameterError("COO index out of range")


@dataclass
class CsrMatrix:
    rows: int
    cols: int
    row_start: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.values)

    @property
    def value_width(self) -> int:
        return self.values.dtype.itemsize

    def row_cols(self, i: int) -> np.ndarray:
        return self.col_idx[self.row_start[i]: self.row_start[i + 1]]

    def row_values(self, i: int) -> np.ndarray:
        return self.values[self.row_start[i]: self.row_start[i + 1]]

    def validate(self) -> None:
        """sparse.py:76-91 — shape, span, monotone rows, ascending columns."""
        if len(self.row_start) != self.rows + 1:
            raise ParameterError("row_start must have rows + 1 entries")
        if self.row_start[0] != 0 or self.row_start[-1] != self.nnz:
            raise ParameterError("row_start must span [0, nnz]")
        if np.any(np.diff(self.row_start) < 0):
            raise ParameterError("row_start must be nondecreasing")
        if self.nnz:
            if self.col_idx.min() < 0 or self.col_idx.max() >= self.cols:
                raise ParameterError("column index out of range")
            deltas = np.diff(self.col_idx)
            starts = self.row_start[1:-1]
            inner = np.ones(self.nnz - 1, dtype=bool)
            inner[starts[(starts > 0) & (starts < self.nnz)] - 1] = False
            if np.any(deltas[inner] <= 0):
                raise ParameterError("columns must be strictly ascending per row")

    def __eq__(self, other) -> bool:
        """Bitwise equality of structure and value bit patterns (sparse.py:93-106)."""
        if not isinstance(other, CsrMatrix):
            return NotImplemented
        return (
            self.rows == other.rows
            and self.cols == other.cols
            and np.array_equal(self.row_start, other.row_start)
            and np.array_equal(self.col_idx, other.col_idx)
            and self.values.dtype == other.values.dtype
            and np.array_equal(
                self.values.view(np.uint64 if self.value_width == 8 else np.uint32),
                other.values.view(np.uint64 if self.value_width == 8 else np.uint32),
            )
        )


def coo_to_csr(m: CooMatrix) -> CsrMatrix:
    """Sort by (row, col) and compress; duplicates rejected (sparse.py:133-144)."""
    m.validate()
    order = np.lexsort((m.col_idx, m.row_idx))
    r = np.asarray(m.row_idx)[order]
    c = np.asarray(m.col_idx)[order]
    v = np.asarray(m.values)[order]
    if len(r) > 1 and np.any((np.diff(r) == 0) & (np.diff(c) == 0)):
        raise MtxFormatError("duplicate (row, col) entry")
    row_start = np.zeros(m.rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=m.rows), out=row_start[1:])
    return CsrMatrix(m.rows, m.cols, row_start, c.astype(np.int64), v)


def sell_widths(m: CsrMatrix, slice_height: int = 32) -> np.ndarray:
    """Per-slice max row length (sparse.py:147-155), vectorised."""
    nnz_row = np.diff(np.asarray(m.row_start, dtype=np.int64))
    nslices = max(1, -(-m.rows // slice_height)) if m.rows else 1
    padded = np.zeros(nslices * slice_height, dtype=np.int64)
    padded[: m.rows] = nnz_row
    return padded.reshape(nslices, slice_height).max(axis=1)


def format_size_bytes(m: CsrMatrix, fmt: str, value_width: int) -> int:
    """Byte size in a baseline format with 4-byte indices (sparse.py:185-198).

    The denominator of the compression ratio: min over coo/csr/sell.
    """
    if value_width not in (4, 8):
        raise ParameterError("value_width must be 4 or 8 bytes")
    fmt = fmt.lower()
    if fmt == "coo":
        return m.nnz * (4 + 4 + value_width)
    if fmt == "csr":
        return m.nnz * (4 + value_width) + 4 * (m.rows + 1)
    if fmt == "sell":
        widths = sell_widths(m, 32)
        return int(widths.sum()) * 32 * (4 + value_width) + 4 * (len(widths) + 1)
    raise ParameterError(f"unknown format {fmt!r}")


def matrix_deltas(m: CsrMatrix) -> np.ndarray:
    """Per-row delta encoding of column indices (sparse.py:289-299)."""
    if m.nnz == 0:
        return np.zeros(0, dtype=np.int64)
    col = np.asarray(m.col_idx, dtype=np.int64)
    d = np.empty(m.nnz, dtype=np.int64)
    d[0] = col[0]
    d[1:] = np.diff(col)
    starts = np.asarray(m.row_start[:-1], dtype=np.int64)
    starts = starts[starts < m.nnz]
    d[starts] = col[starts]
    return d


def value_patterns(values: np.ndarray) -> np.ndarray:
    """Raw bit patterns of the value array (sparse.py:302-309)."""
    width = values.dtype.itemsize
    if width == 8:
        return np.ascontiguousarray(values).view(np.uint64)
    if width == 4:
        return np.ascontiguousarray(values).view(np.uint32)
    raise ParameterError(f"unsupported value width {width}")


def reference_spmv(m: CsrMatrix, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """The reference's CSR SpMV utility (sparse.py:330-353), numpy on host.

    Part of the mirrored public API (a plain CSR product used for checking
    and for the compression-free comparison); the dtANS ``spmv`` never calls
    it.  Per row: acc = +0.0; acc = fl(acc + fl(v * x[c])) left to right;
    result fl(acc + y).
    """
    x = np.asarray(x)
    y = np.asarray(y)
    if len(x) != m.cols or len(y) != m.rows:
        raise ParameterError("dimension mismatch")
    dtype = m.values.dtype
    x = x.astype(dtype, copy=False)
    y = y.astype(dtype, copy=False)
    acc = np.zeros(m.rows, dtype=dtype)
    nnz_row = np.diff(m.row_start)
    if m.nnz:
        order = np.argsort(-nnz_row, kind="stable")
        base = m.row_start[:-1][order]
        maxn = int(nnz_row.max())
        active = np.searchsorted(-nnz_row[order], -np.arange(1, maxn + 1), side="right")
        for q in range(maxn):
            a = int(active[q])
            idx = base[:a] + q
            acc[order[:a]] += m.values[idx] * x[m.col_idx[idx]]
    return acc + y


def sort_rows_by_length(m: CsrMatrix, window: int | None = None):
    """Row reordering for skewed matrices (fix A): rows
    stably sorted by descending length, within windows of ``window`` rows
    (None: globally), so each 32-row slice holds rows of similar length.

    Returns ``(P*A, perm)`` with ``perm[i]`` = original index of row i of P*A
    (uint32).  Encode P*A with ``encode_matrix`` (byte-identical to the
    reference's encoding of P*A) and set ``container.row_map = perm``; the
    SpMV then reads y and writes y' in the original row order.
    """
    nnz_row = np.diff(np.asarray(m.row_start, dtype=np.int64))
    if window is None or window >= m.rows:
        perm = np.argsort(-nnz_row, kind="stable")
    else:
        if window < 1:
            raise ParameterError("window must be >= 1")
        blk = np.arange(m.rows) // window
        perm = np.lexsort((-nnz_row, blk))
    perm = perm.astype(np.int64)
    new_len = nnz_row[perm]
    row_start = np.zeros(m.rows + 1, dtype=np.int64)
    np.cumsum(new_len, out=row_start[1:])
    src = np.repeat(np.asarray(m.row_start[:-1], dtype=np.int64)[perm], new_len) + (
        np.arange(int(row_start[-1]), dtype=np.int64) - np.repeat(row_start[:-1], new_len))
    pm = CsrMatrix(m.rows, m.cols, row_start, np.asarray(m.col_idx)[src], np.asarray(m.values)[src])
    return pm, perm.astype(np.uint32)


def parse_mtx(text: str) -> CooMatrix:
    """Parse MatrixMarket coordinate content (sparse.py:205-264): real /
    integer / pattern fields, general / symmetric symmetry; symmetric
    off-diagonal entries are mirrored, pattern entries get value 1.0.
    Raises MtxFormatError on the same conditions as the reference, checked
    in the same order."""
    lines = text.splitlines()
    if not lines or not lines[0].startswith("%%MatrixMarket"):
        raise MtxFormatError("missing %%MatrixMarket banner")
    banner = [tok.lower() for tok in lines[0].split()]
    if len(banner) != 5:
        raise MtxFormatError(f"malformed banner: {lines[0]!r}")
    obj, layout, field, symmetry = banner[1:]
    if obj != "matrix":
        raise MtxFormatError(f"unsupported object {obj!r}")
    if layout != "coordinate":
        raise MtxFormatError(f"unsupported layout {layout!r} (coordinate only)")
    if field not in ("real", "integer", "pattern"):
        raise MtxFormatError(f"unsupported field {field!r}")
    if symmetry not in ("general", "symmetric"):
        raise MtxFormatError(f"unsupported symmetry {symmetry!r}")
    body = [ln for ln in lines[1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:
        raise MtxFormatError("missing size line")
    head = body[0].split()
    if len(head) != 3:
        raise MtxFormatError(f"malformed size line: {body[0]!r}")
    try:
        rows, cols, nnz = (int(t) for t in head)
    except ValueError as e:
        raise MtxFormatError(f"malformed size line: {body[0]!r}") from e
    if min(rows, cols, nnz) < 0:
        raise MtxFormatError("negative dimensions")
    if len(body) - 1 != nnz:
        raise MtxFormatError(f"expected {nnz} entries, found {len(body) - 1}")
    width = 2 if field == "pattern" else 3
    toks = " ".join(body[1:]).split()
    if len(toks) != nnz * width:
        raise MtxFormatError("entry lines have the wrong number of fields")
    try:
        a = np.asarray(toks, dtype=np.float64).reshape(nnz, width)
    except ValueError as e:
        raise MtxFormatError("non-numeric entry") from e
    r = a[:, 0].astype(np.int64) - 1
    c = a[:, 1].astype(np.int64) - 1
    if np.any(a[:, 0] != r + 1) or np.any(a[:, 1] != c + 1):
        raise MtxFormatError("non-integer index")
    v = a[:, 2] if width == 3 else np.ones(nnz, dtype=np.float64)
    if nnz and (r.min() < 0 or r.max() >= rows or c.min() < 0 or c.max() >= cols):
        raise MtxFormatError("index out of range")
    if symmetry == "symmetric":
        off = r != c
        r, c, v = np.concatenate([r, c[off]]), np.concatenate([c, r[off]]), np.concatenate([v, v[off]])
    return CooMatrix(rows, cols, r, c, v)


def read_mtx(path) -> CsrMatrix:
    """A MatrixMarket file (e.g. from SuiteSparse) as a CsrMatrix."""
    with open(path, "r") as f:
        return coo_to_csr(parse_mtx(f.read()))


def sort_symmetric_by_degree(m: CsrMatrix):
    """Symmetric degree ordering of a square matrix (skew toolkit, SURVEY
    §8f item 1): B = P A P^T with rows AND columns in stably descending
    row-length order.  Rows of similar length share slices (as in
    sort_rows_by_length), and in power-law graphs the popular columns move
    to small indices: column deltas shrink (fewer escapes, fewer bytes)
    and the x gathers concentrate on a hot prefix of x.

    Returns ``(B, perm)`` with ``perm[i]`` = original index of row/column i.
    Encode B and set ``container.row_map = perm`` and
    ``container.col_map = perm``: the SpMV then gathers x' = x[perm] on the
    device and reads y / writes y' in the original order."""
    if m.rows != m.cols:
        raise ParameterError("symmetric ordering needs a square matrix")
    pm, perm = sort_rows_by_length(m)
    inv = np.empty(m.rows, dtype=np.int64)
    inv[perm.astype(np.int64)] = np.arange(m.rows, dtype=np.int64)
    newc = inv[np.asarray(pm.col_idx, dtype=np.int64)]
    nnz_row = np.diff(np.asarray(pm.row_start, dtype=np.int64))
    rows = np.repeat(np.arange(pm.rows, dtype=np.int64), nnz_row)
    o = np.lexsort((newc, rows))
    return CsrMatrix(pm.rows, pm.cols, pm.row_start, newc[o], np.asarray(pm.values)[o]), perm
