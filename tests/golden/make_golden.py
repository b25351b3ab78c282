"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (it needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

For every case of the matrix zoo it records, from the reference package
(/root/reference/pkg/src/csrdtans):

* the input CSR matrix and the encode options,
* ``sha256(serialize(encode_matrix(m, ...)))`` (container.py:126-204,647-664)
  and, for small cases, the container bytes themselves,
* ``size_bytes`` (container.py:723-731), the stream length,
* ``spmv(c, x, y)`` (container.py:554-596) and ``reference_spmv``
  (sparse.py:330-353) on seeded x, y.

It also asserts ``decode_matrix(c) == m`` (container.py:524-531) so the
stored input *is* the reference decode output.  The fixtures are what the
GPU box sees: nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, REPO)
sys.dont_write_bytecode = True

import csrdtans as R  # noqa: E402  (the reference)
from helpers import random_csr, banded_matrix  # noqa: E402  (reference test builders)

from paper_2603_01915_b200 import synth  # noqa: E402

OUT = os.path.join(HERE, "cases")
KEEP_BYTES_MAX = 80_000  # store container bytes when the stream is small


def to_ref(m):
    return R.CsrMatrix(m.rows, m.cols, np.asarray(m.row_start, dtype=np.int64),
                       np.asarray(m.col_idx, dtype=np.int64), m.values)


def custom(rows, cols, row_lists, dtype=np.float64):
    r, c, v = [], [], []
    for i, lst in enumerate(row_lists):
        for col, val in lst:
            r.append(i)
            c.append(col)
            v.append(val)
    coo = R.CooMatrix(rows, cols, np.array(r, dtype=np.int64),
                      np.array(c, dtype=np.int64), np.array(v, dtype=dtype))
    return R.coo_to_csr(coo)


def cases():
    yield "fig1_f64", synth.fig1(), {}
    yield "fig1_f32", synth.fig1(), {"value_width": 4}
    yield "fig1_seed_none", synth.fig1(), {"permutation_seed": None}
    yield "fig1_seed_12345", synth.fig1(), {"permutation_seed": 12345}
    yield "config1", synth.config1_random(), {}
    for seed in range(24):
        for prec in (8, 4):
            m = random_csr(random.Random(seed), max_rows=200, max_nnz=2500,
                           precision=prec)
            yield f"random_csr_s{seed}_p{prec}", m, {}
    yield "laplacian_g48", synth.laplacian_2d(48), {}
    yield "laplacian_g20_f32", synth.laplacian_2d(20, dtype=np.float32), {}
    yield "banded27_1500", synth.banded(1500, 27), {}
    yield "banded32_pos_700", synth.banded(700, 32, positive=True), {}
    yield "banded_ref_helper", banded_matrix(300, 9, value_pool=[0.5, 1.0, 2.0]), {}
    yield "rmat_s11_f32", synth.rmat(11, 12000), {}
    yield "rmat_s9_f64", synth.rmat(9, 3000, seed=3, dtype=np.float64), {}
    # Edge cases: empty, ragged slices, one very long row, specials, sentinels.
    yield "empty_70x40", custom(70, 40, [[] for _ in range(70)]), {}
    yield "zero_rows", custom(0, 5, []), {}
    yield "ragged_33", synth.banded(33, 5), {}
    yield "one_long_row", custom(3, 5000, [[], [(c, float(c % 7) - 3.0) for c in range(0, 5000, 2)], [(1, 1.0)]]), {}
    rng = np.random.default_rng(7)
    long_rows = [[(int(c), float(v)) for c, v in zip(sorted(rng.choice(900, k, replace=False)), rng.standard_normal(k))]
                 for k in rng.integers(0, 400, 64)]
    yield "skewed_64", custom(64, 900, long_rows), {}
    nan = float("nan")
    sent64 = np.array([0xFFFFFFFFFFFFFFFF], dtype=np.uint64).view(np.float64)[0]
    yield "specials_f64", custom(40, 40, [[(i, [0.0, -0.0, np.inf, -np.inf, nan, sent64, 1e-300, 5e-324][i % 8])] + ([(i + 1, 2.0)] if i < 39 else []) for i in range(40)]), {}
    sent32 = np.array([0xFFFFFFFF], dtype=np.uint32).view(np.float32)[0]
    yield "specials_f32", custom(40, 40, [[(i, [0.0, -0.0, np.inf, nan, sent32, 1.5][i % 6])] for i in range(40)], dtype=np.float32), {}
    yield "single_value_f64", custom(100, 100, [[(i, 3.0)] for i in range(100)]), {}
    # cols = 2^32: the delta 0xFFFFFFFF equals the sentinel and must escape.
    yield "wide_cols_sentinel", custom(2, 2**32, [[(0, 1.0), (2**32 - 1, 2.0)], [(5, 1.0)]]), {"spmv": False}


def main():
    os.makedirs(OUT, exist_ok=True)
    index = []
    for i, (name, m, opts) in enumerate(cases()):
        opts = dict(opts)
        do_spmv = opts.pop("spmv", True)
        rm = to_ref(m)
        c = R.encode_matrix(rm, **opts)
        blob = R.serialize(c)
        sha = hashlib.sha256(blob).hexdigest()
        dec = R.decode_matrix(c)
        prec = c.precision
        vdt = np.float64 if prec == 8 else np.float32
        expect = R.CsrMatrix(rm.rows, rm.cols, rm.row_start, rm.col_idx,
                             rm.values.astype(vdt))
        assert dec == expect, name
        rec = dict(
            rows=np.int64(m.rows), cols=np.int64(m.cols),
            row_start=np.asarray(m.row_start, dtype=np.int64),
            col_idx=np.asarray(m.col_idx, dtype=np.int64),
            values=np.asarray(m.values),
            precision=np.int64(prec),
            value_width=np.int64(opts.get("value_width", -1) or -1),
            permutation_seed=np.int64(-1 if ("permutation_seed" in opts and opts["permutation_seed"] is None)
                                      else opts.get("permutation_seed", 2654435761)),
            sha256=np.array(sha),
            nwords=np.int64(len(c.stream)),
            size_bytes=np.int64(R.size_bytes(c)),
            fmt_sizes=np.array([R.format_size_bytes(rm, f, prec) for f in ("coo", "csr", "sell")], dtype=np.int64),
        )
        if len(blob) <= KEEP_BYTES_MAX or name in ("config1",):
            rec["container"] = np.frombuffer(blob, dtype=np.uint8)
        if do_spmv:
            xr = np.random.default_rng(1000 + i)
            x = xr.standard_normal(m.cols).astype(vdt)
            y = xr.standard_normal(m.rows).astype(vdt)
            rec["x"], rec["y"] = x, y
            out = R.spmv(c, x, y)
            ref = R.reference_spmv(dec, x, y)
            assert np.array_equal(out.view(np.uint8), ref.view(np.uint8)) or np.allclose(out, ref, equal_nan=True), name
            rec["spmv"] = out
            rec["reference_spmv"] = ref
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **rec)
        index.append(f"{name} {sha} {len(blob)} {len(c.stream)}")
        print(index[-1], flush=True)
    with open(os.path.join(HERE, "INDEX.txt"), "w") as f:
        f.write("# name sha256(serialize(encode_matrix)) container_bytes stream_words\n")
        f.write("\n".join(index) + "\n")


if __name__ == "__main__":
    main()
