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
