"""Loader for the golden fixtures generated from the reference
(tests/golden/make_golden.py)."""

import glob
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CASE_DIR = os.path.join(HERE, "golden", "cases")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(CASE_DIR, "*.npz")))


def load(name):
    z = np.load(os.path.join(CASE_DIR, name + ".npz"), allow_pickle=False)
    return {k: z[k] for k in z.files}


def matrix(rec):
    from paper_2603_01915_b200.sparse import CsrMatrix
    return CsrMatrix(int(rec["rows"]), int(rec["cols"]), rec["row_start"], rec["col_idx"], rec["values"])


def encode_kwargs(rec):
    kw = {}
    if int(rec["value_width"]) > 0:
        kw["value_width"] = int(rec["value_width"])
    seed = int(rec["permutation_seed"])
    if seed == -1:
        kw["permutation_seed"] = None
    elif seed != 2654435761:
        kw["permutation_seed"] = seed
    return kw


def same_bits_or_nan(a, b):
    """Bitwise equality, treating any NaN as equal to any NaN."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    ui = np.uint64 if a.dtype.itemsize == 8 else np.uint32
    eq = a.view(ui) == b.view(ui)
    both_nan = np.isnan(a) & np.isnan(b)
    return bool(np.all(eq | both_nan))


LONG_SEG = 64  # slices whose longest row has more segments use the task kernel
TASK_SEG = 16  # segments per checkpointed task (DTANS_CHUNK default, api.cu)


def long_slice_rows(row_start, rows):
    """Boolean mask of rows that may be split into several checkpointed
    tasks (their reduction order differs from the reference's): slices
    longer than one task (TASK_SEG segments).  Shorter slices are decoded by
    one warp in lockstep order (main kernel, or a single task) and must match
    bitwise."""
    nnz_row = np.diff(np.asarray(row_start, dtype=np.int64))
    nseg = (2 * nnz_row + 7) // 8
    ns = -(-rows // 32)
    pad = np.zeros(ns * 32, dtype=np.int64)
    pad[:rows] = nseg
    long_slice = pad.reshape(ns, 32).max(axis=1) > TASK_SEG
    return np.repeat(long_slice, 32)[:rows]


def check_spmv(out, ref, m, x, y, c=None):
    """Parity policy (north star / SURVEY 8c): bitwise for rows decoded in
    lockstep order; for rows whose slice was split into several tasks
    |out-ref| <= tol*(sum|a x| + |y|), tol 1e-12 (f64) / 1e-5 (f32);
    NaN == NaN.  With the container ``c`` (rows in the order of ``out``) the
    split rows are the device plan's (dtans_split_slices); otherwise every
    slice longer than one 16-segment task counts as split."""
    out = np.asarray(out)
    ref = np.asarray(ref)
    if out.shape != ref.shape or out.dtype != ref.dtype:
        return False
    if c is not None:
        lr = c.device(0).split_rows(m.rows) | long_slice_rows(m.row_start, m.rows)
    else:
        lr = long_slice_rows(m.row_start, m.rows)
    if not same_bits_or_nan(out[~lr], ref[~lr]):
        return False
    if not lr.any():
        return True
    tol = 1e-12 if out.dtype == np.float64 else 1e-5
    vals = np.abs(np.asarray(m.values, dtype=np.float64))
    ax = vals * np.abs(np.asarray(x, dtype=np.float64))[np.asarray(m.col_idx)]
    rows_of = np.repeat(np.arange(m.rows), np.diff(np.asarray(m.row_start)))
    s = np.bincount(rows_of, weights=ax, minlength=m.rows) + np.abs(np.asarray(y, dtype=np.float64))
    o, r = out[lr].astype(np.float64), ref[lr].astype(np.float64)
    both_nan = np.isnan(o) & np.isnan(r)
    ok = (np.abs(o - r) <= tol * s[lr]) | both_nan | (o == r)
    return bool(np.all(ok))
