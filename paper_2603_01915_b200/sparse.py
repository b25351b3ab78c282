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
    """COO -> CSR with rows in order and columns ascending within a row;
    a repeated (row, col) coordinate raises MtxFormatError (the contract of
    reference sparse.py:133-144).

    One stable argsort of the linearised coordinate row * cols + col
    orders the entries; equal neighbouring keys are duplicates, and the row
    pointers are the searchsorted positions of every row start in the
    sorted rows."""
    m.validate()
    rows_i = np.asarray(m.row_idx, dtype=np.int64)
    cols_i = np.asarray(m.col_idx, dtype=np.int64)
    key = rows_i * np.int64(max(m.cols, 1)) + cols_i
    perm = np.argsort(key, kind="stable")
    skey = key[perm]
    if skey.size > 1 and bool((skey[1:] == skey[:-1]).any()):
        raise MtxFormatError("duplicate (row, col) entry")
    srow = rows_i[perm]
    row_start = np.searchsorted(srow, np.arange(m.rows + 1, dtype=np.int64), side="left").astype(np.int64)
    return CsrMatrix(m.rows, m.cols, row_start, cols_i[perm], np.asarray(m.values)[perm])


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
    """The reference's plain CSR product (contract of sparse.py:330-353):
    y' = A x + y in the matrix precision, each row accumulated strictly left
    to right from +0.0, i.e. acc = fl(acc + fl(v * x[c])), then fl(acc + y).
    x and y are cast to the matrix dtype; a new array is returned.

    Host numpy, a checker and API mirror only (the dtANS ``spmv`` never
    calls it).  The products fl(v * x[c]) do not depend on order, so they
    are formed once for all nonzeros; the sums are then folded by position
    within the row: step q adds the q-th product of every row that has one
    (each row at most once per step, so a fancy-indexed add is exact)."""
    x = np.asarray(x)
    y = np.asarray(y)
    if len(x) != m.cols or len(y) != m.rows:
        raise ParameterError("dimension mismatch")
    dt = m.values.dtype
    xv = x.astype(dt, copy=False)
    yv = y.astype(dt, copy=False)
    acc = np.zeros(m.rows, dtype=dt)
    if m.nnz == 0:
        return acc + yv
    rs = np.asarray(m.row_start, dtype=np.int64)
    lens = np.diff(rs)
    with np.errstate(all="ignore"):
        prod = np.asarray(m.values) * xv[np.asarray(m.col_idx)]
    owner = np.repeat(np.arange(m.rows, dtype=np.int64), lens)
    pos = np.arange(m.nnz, dtype=np.int64) - rs[owner]
    by_pos = np.argsort(pos, kind="stable")
    bounds = np.concatenate([[0], np.cumsum(np.bincount(pos))])
    with np.errstate(all="ignore"):
        for q in range(len(bounds) - 1):
            sel = by_pos[bounds[q]:bounds[q + 1]]
            tgt = owner[sel]
            acc[tgt] = acc[tgt] + prod[sel]
        return acc + yv


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


_MTX_FIELDS = {"real": 3, "integer": 3, "pattern": 2}  # tokens per entry line
_MTX_SYMMETRY = ("general", "symmetric")


def _mtx_header(first: str):
    """Banner line -> (field, symmetry); the reference's checks in order
    (object, layout, field, symmetry)."""
    if not first.startswith("%%MatrixMarket"):
        raise MtxFormatError("missing %%MatrixMarket banner")
    words = first.split()
    if len(words) != 5:
        raise MtxFormatError(f"malformed banner: {first!r}")
    obj, layout, field, symmetry = (w.lower() for w in words[1:])
    checks = ((obj == "matrix", f"unsupported object {obj!r}"),
              (layout == "coordinate", f"unsupported layout {layout!r} (coordinate only)"),
              (field in _MTX_FIELDS, f"unsupported field {field!r}"),
              (symmetry in _MTX_SYMMETRY, f"unsupported symmetry {symmetry!r}"))
    for ok, msg in checks:
        if not ok:
            raise MtxFormatError(msg)
    return field, symmetry


def _mtx_size(line: str):
    parts = line.split()
    try:
        if len(parts) != 3:
            raise ValueError
        dims = tuple(int(p) for p in parts)
    except ValueError as e:
        raise MtxFormatError(f"malformed size line: {line!r}") from e
    if any(d < 0 for d in dims):
        raise MtxFormatError("negative dimensions")
    return dims


def parse_mtx(text: str) -> CooMatrix:
    """MatrixMarket coordinate content -> CooMatrix (0-based), with the
    reference's accepted dialect and MtxFormatError conditions (sparse.py:
    205-264): real / integer / pattern fields (pattern -> 1.0), general /
    symmetric (off-diagonal entries of a symmetric file are mirrored and
    appended after the stored ones); '%' comment and blank lines skipped.
    The entry count is checked per line and the field count over the whole
    token stream, as the reference does."""
    all_lines = text.splitlines()
    field, symmetry = _mtx_header(all_lines[0] if all_lines else "")
    content = [ln for ln in all_lines[1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if not content:
        raise MtxFormatError("missing size line")
    nrows, ncols, count = _mtx_size(content[0])
    entries = content[1:]
    if len(entries) != count:
        raise MtxFormatError(f"expected {count} entries, found {len(entries)}")
    per = _MTX_FIELDS[field]
    flat = [tok for ln in entries for tok in ln.split()]
    if len(flat) != count * per:
        raise MtxFormatError("entry lines have the wrong number of fields")
    try:
        table = np.array(flat, dtype=np.float64).reshape(count, per)
    except ValueError as e:
        raise MtxFormatError("non-numeric entry") from e
    one_based = table[:, :2]
    idx = one_based.astype(np.int64)
    if not np.array_equal(idx.astype(np.float64), one_based):
        raise MtxFormatError("non-integer index")
    idx -= 1
    r, c = idx[:, 0], idx[:, 1]
    v = table[:, 2].copy() if per == 3 else np.ones(count, dtype=np.float64)
    if count and (idx.min() < 0 or r.max() >= nrows or c.max() >= ncols):
        raise MtxFormatError("index out of range")
    if symmetry == "symmetric":
        mirror = np.flatnonzero(r != c)
        r, c, v = (np.concatenate([r, c[mirror]]), np.concatenate([c, r[mirror]]),
                   np.concatenate([v, v[mirror]]))
    return CooMatrix(nrows, ncols, r, c, v)


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
