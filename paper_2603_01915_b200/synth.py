"""Synthetic matrices of the five BASELINE.json configurations.

All generators are seeded and vectorised (numpy), and return a
``CsrMatrix`` with strictly ascending columns per row.  There is no network
in this environment, so these shapes stand in for SuiteSparse inputs.
"""

from __future__ import annotations

import numpy as np

from .sparse import CsrMatrix


def fig1() -> CsrMatrix:
    """The 4x4 running example (reference tests/test_sparse.py:27-39)."""
    row_start = np.array([0, 2, 4, 5, 6], dtype=np.int64)
    cols = np.array([1, 3, 0, 2, 1, 3], dtype=np.int64)
    vals = np.array([7.0, 5.0, 3.0, 2.0, 4.0, 1.0])
    return CsrMatrix(4, 4, row_start, cols, vals)


def _csr_from_sorted_codes(rows: int, cols: int, r: np.ndarray, c: np.ndarray,
                           v: np.ndarray) -> CsrMatrix:
    row_start = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=rows), out=row_start[1:])
    return CsrMatrix(rows, cols, row_start, c.astype(np.int64), v)


def config1_random(n: int = 4096, nnz: int = 2**15, seed: int = 0) -> CsrMatrix:
    """Config 1: uniform random pattern, N(0,1) fp64 values."""
    rng = np.random.default_rng(seed)
    flat = rng.choice(n * n, nnz, replace=False)
    r, c = np.divmod(flat, n)
    v = rng.standard_normal(nnz)
    order = np.lexsort((c, r))
    return _csr_from_sorted_codes(n, n, r[order], c[order], v[order])


def laplacian_2d(g: int, dtype=np.float64) -> CsrMatrix:
    """Config 2: 5-point Laplacian on a g x g grid (diag 4, neighbours -1)."""
    return laplacian_rows(g, 0, g * g, dtype)


def laplacian_row_nnz(g: int) -> np.ndarray:
    """Nonzeros per row of ``laplacian_2d(g)`` (shard planning without the matrix)."""
    a, b = np.divmod(np.arange(g * g, dtype=np.int64), g)
    return 1 + (a > 0) + (b > 0) + (b < g - 1) + (a < g - 1)


def laplacian_rows(g: int, r0: int, r1: int, dtype=np.float64) -> CsrMatrix:
    """Rows [r0, r1) of ``laplacian_2d(g)`` (a row shard; all columns)."""
    n = g * g
    i = np.arange(r0, r1, dtype=np.int64)
    a, b = np.divmod(i, g)
    offs = np.array([-g, -1, 0, 1, g], dtype=np.int64)
    valid = np.stack([a > 0, b > 0, np.ones(len(i), bool), b < g - 1, a < g - 1], axis=1)
    cols = i[:, None] + offs[None, :]
    vals = np.where(offs == 0, 4.0, -1.0).astype(dtype)
    vals = np.broadcast_to(vals, (len(i), 5))
    row_start = np.zeros(len(i) + 1, dtype=np.int64)
    np.cumsum(valid.sum(axis=1), out=row_start[1:])
    return CsrMatrix(len(i), n, row_start, cols[valid], np.ascontiguousarray(vals[valid]))


def banded(rows: int, band: int = 27, levels: int = 256, seed: int = 0,
           positive: bool = False, dtype=np.float64) -> CsrMatrix:
    """Configs 4/5: FEM-like band of ``band`` entries centred on the
    diagonal (clipped at the edges), values i.i.d. from a ``levels``-level
    alphabet (linspace(-1,1) or, for power iteration, (1..levels)/levels)."""
    half = band // 2
    i = np.arange(rows, dtype=np.int64)
    lo = np.maximum(0, i - half)
    hi = np.minimum(rows, i - half + band)
    cnt = hi - lo
    row_start = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(cnt, out=row_start[1:])
    nnz = int(row_start[-1])
    row_of = np.repeat(i, cnt)
    cols = lo[row_of] + (np.arange(nnz, dtype=np.int64) - row_start[row_of])
    if positive:
        alphabet = (np.arange(levels, dtype=np.float64) + 1.0) / levels
    else:
        alphabet = np.linspace(-1.0, 1.0, levels)
    rng = np.random.default_rng(seed)
    vals = alphabet.astype(dtype)[rng.integers(0, levels, nnz)]
    return CsrMatrix(rows, rows, row_start, cols, vals)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = (z + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def banded_row_nnz(rows_total: int, band: int) -> np.ndarray:
    """Nonzeros per row of the banded shape (shard planning without the matrix)."""
    i = np.arange(rows_total, dtype=np.int64)
    half = band // 2
    return np.minimum(rows_total, i - half + band) - np.maximum(0, i - half)


def banded_rows(rows_total: int, r0: int, r1: int, band: int = 32, levels: int = 256, seed: int = 0,
                positive: bool = True, dtype=np.float64) -> CsrMatrix:
    """Rows [r0, r1) of the ``rows_total``-row banded matrix of ``banded``'s
    shape, values from a counter-based hash of (seed, row, column), so every
    row block of the same global matrix is generated independently and
    identically on each rank (power iteration / scaling runs)."""
    half = band // 2
    i = np.arange(r0, r1, dtype=np.int64)
    lo = np.maximum(0, i - half)
    hi = np.minimum(rows_total, i - half + band)
    cnt = hi - lo
    row_start = np.zeros(len(i) + 1, dtype=np.int64)
    np.cumsum(cnt, out=row_start[1:])
    nnz = int(row_start[-1])
    row_of = np.repeat(np.arange(len(i), dtype=np.int64), cnt)
    cols = lo[row_of] + (np.arange(nnz, dtype=np.int64) - row_start[row_of])
    key = (i[row_of].astype(np.uint64) * np.uint64(rows_total) + cols.astype(np.uint64)) ^ np.uint64(seed * 0x5851F42D)
    lvl = (_splitmix64(key) % np.uint64(levels)).astype(np.int64)
    del key, row_of
    if positive:
        alphabet = (np.arange(levels, dtype=np.float64) + 1.0) / levels
    else:
        alphabet = np.linspace(-1.0, 1.0, levels)
    return CsrMatrix(len(i), rows_total, row_start, cols, alphabet.astype(dtype)[lvl])


def rmat(scale: int, nnz: int, seed: int = 0, probs=(0.57, 0.19, 0.19, 0.05),
         dtype=np.float32, batch: int = 1 << 24) -> CsrMatrix:
    """Config 3: R-MAT (a,b,c,d)=(.57,.19,.19,.05) adjacency, values 1.0.

    Edges are drawn in batches (quadrants from 8-bit uniform draws against
    thresholds round(p * 256): a=146/256, a+b=195/256, a+b+c=243/256, within
    0.4% of the target probabilities) until at least ``nnz`` distinct edges exist;
    if there are more, a seeded uniform subset of exactly ``nnz`` is kept.
    No symmetrisation, no self-loop removal."""
    a, b, c, _ = probs
    ta, tab, tabc = (int(round(v * 256)) for v in (a, a + b, a + b + c))
    n = 1 << scale
    rng = np.random.default_rng(seed)
    it = np.uint32 if scale <= 31 else np.int64
    uniq = np.zeros(0, dtype=np.int64)
    while len(uniq) < nnz:
        need = int((nnz - len(uniq)) * 1.3) + 4096
        parts = [uniq]
        while need > 0:
            m = min(batch, need)
            r = np.zeros(m, dtype=it)
            cc = np.zeros(m, dtype=it)
            for _ in range(scale):
                uu = np.frombuffer(rng.bytes(m), dtype=np.uint8)
                r <<= 1
                cc <<= 1
                r |= uu >= tab
                cc |= ((uu >= ta) & (uu < tab)) | (uu >= tabc)
            parts.append((r.astype(np.int64) << scale) | cc)
            need -= m
        allc = np.sort(np.concatenate(parts))  # sort-based unique (np.unique is slow here)
        uniq = allc[np.concatenate([[True], allc[1:] != allc[:-1]])] if len(allc) else allc
    if len(uniq) > nnz:
        keep = rng.choice(len(uniq), nnz, replace=False)
        keep.sort()
        uniq = uniq[keep]
    r, cc = np.divmod(uniq, n)
    return _csr_from_sorted_codes(n, n, r, cc, np.ones(nnz, dtype=dtype))


def vectors(m: CsrMatrix, seed_x: int = 1, seed_y: int = 2, y_zero=False):
    """x ~ N(0,1) (seed 1), y ~ N(0,1) (seed 2) in the matrix precision."""
    dtype = m.values.dtype
    x = np.random.default_rng(seed_x).standard_normal(m.cols).astype(dtype)
    if y_zero:
        y = np.zeros(m.rows, dtype=dtype)
    else:
        y = np.random.default_rng(seed_y).standard_normal(m.rows).astype(dtype)
    return x, y


def config(name: str) -> CsrMatrix:
    """Full-size matrices of BASELINE.json configs by short name."""
    if name == "config1":
        return config1_random()
    if name == "laplacian":
        return laplacian_2d(2591)
    if name == "rmat":
        return rmat(23, 2**27)
    if name == "banded27":
        return banded(-(-2**28 // 27), 27)
    if name == "banded32":
        return banded(2**24, 32, positive=True)
    raise KeyError(name)
