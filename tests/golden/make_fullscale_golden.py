"""Full-scale encoder goldens: the REFERENCE encoder's tables and sampled
slices on the BASELINE-size matrices the benchmark encodes.

Run in the build container only (it needs /root/reference, ~20 GB of RAM and
a few minutes):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fullscale_golden.py [laplacian rmat banded27]

The small-case zoo (make_golden.py) pins byte identity up to ~82k stream
words and ~20k distinct symbols.  The benchmark matrices are far larger:
config 2 has ~6.7M distinct first deltas, which drives quantize
(entropy.py:223-321) into its coarse-to-fine branch with a huge tail, and
config 4 has 2^28 symbols per domain.  Running the whole reference
encode_matrix at that size takes hours (~40-430 us per nonzero), so this
script runs the reference's own steps of encode_matrix
(container.py:126-204) at full size where they are vectorised or cheap and
on a sample where they are per-symbol Python:

* full size: matrix_deltas / value_patterns (sparse.py:289-309), the
  distributions (container.py:112-114), quantize (entropy.py:223-321) for
  both domains, the seeded slot permutations (container.py:162-164) and
  build_tables (entropy.py:404-436) -> the serialized table block
  (container.py:612-625), recorded as its SHA-256;
* sampled: for 64 slices (the first, the last and a seeded uniform sample),
  every row's dtans_encode (codec.py:296-368) against the full-size tables,
  then interleave_warp (container.py:283-317) -> the slice's stream words,
  recorded as SHA-256 + length, with the slice's row_symbols.

The matrices come from paper_2603_01915_b200/synth.py, the generators
bench.py runs (identical seeds).  Output: tests/golden/fullscale.json (small;
no matrix data).  tests/test_fullscale_encoder.py checks the host and GPU
encoders against it on the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.dont_write_bytecode = True

import csrdtans as R  # noqa: E402  (the reference)
import csrdtans.container  # noqa: E402,F401
import csrdtans.entropy  # noqa: E402,F401
import csrdtans.sparse  # noqa: E402,F401

# the package re-exports functions named like its modules (csrdtans.entropy
# is a function there), so take the modules from sys.modules
RC = sys.modules["csrdtans.container"]
RE = sys.modules["csrdtans.entropy"]
RS = sys.modules["csrdtans.sparse"]
from csrdtans.codec import DtansParams, dtans_encode  # noqa: E402

from paper_2603_01915_b200 import synth  # noqa: E402

OUT = os.path.join(HERE, "fullscale.json")
NSAMPLE = 64
SAMPLE_SEED = 20260317


def matrices():
    """The BASELINE-size matrices exactly as bench.py builds them (Spec)."""
    yield "laplacian", lambda: synth.laplacian_rows(2591, 0, 2591 * 2591)
    yield "rmat", lambda: synth.rmat(23, 2**27)
    n27 = -(-2**28 // 27)
    yield "banded27", lambda: synth.banded_rows(n27, 0, n27, 27, positive=False)


def sample_slices(nslices: int) -> list:
    rng = np.random.default_rng(SAMPLE_SEED)
    pick = set(rng.choice(nslices, min(nslices, NSAMPLE - 2), replace=False).tolist())
    pick.update({0, nslices - 1})
    return sorted(pick)


def run(name, gen):
    t0 = time.time()
    m = gen()
    rm = R.CsrMatrix(m.rows, m.cols, np.asarray(m.row_start, dtype=np.int64),
                     np.asarray(m.col_idx, dtype=np.int64), m.values)
    params = DtansParams.production()
    precision = rm.value_width
    values = rm.values.astype(np.float64 if precision == 8 else np.float32, copy=False)
    deltas = RS.matrix_deltas(rm)
    patterns = RS.value_patterns(values)
    ddist = RC._distribution_from_array(deltas)
    vdist = RC._distribution_from_array(patterns)
    t1 = time.time()
    qd = RE.quantize(ddist, params.k, params.m, 32, never_retain=frozenset({RC.DELTA_SENTINEL}))
    qv = RE.quantize(vdist, params.k, params.m, precision * 8,
                     never_retain=frozenset({RC.VALUE_SENTINEL[precision]}))
    rng = np.random.default_rng(RC.DEFAULT_PERMUTATION_SEED)
    perm_d = rng.permutation(params.k).tolist()
    perm_v = rng.permutation(params.k).tolist()
    dt = RE.build_tables(qd, perm_d)
    vt = RE.build_tables(qv, perm_v)
    t2 = time.time()
    # the table block through the reference's own serializer (a container
    # shell carrying only the tables)
    shell = RC.CsrDtansContainer(rows=0, cols=m.cols, nnz=0, precision=precision, params=params,
                                 permutation_seed=RC.DEFAULT_PERMUTATION_SEED, delta_tables=dt,
                                 value_tables=vt, row_symbols=np.zeros(0, np.uint32),
                                 directory=np.zeros(1, np.uint64), stream=np.zeros(0, np.uint32))
    block = RC._tables_block(shell)
    rec = {"rows": int(m.rows), "cols": int(m.cols), "nnz": int(m.nnz), "precision": precision,
           "delta_distinct": len(ddist.symbols), "value_distinct": len(vdist.symbols),
           "delta_retained": sum(1 for x in qd.multiplicities if x), "value_retained": sum(1 for x in qv.multiplicities if x),
           "tables_sha256": hashlib.sha256(block).hexdigest(), "tables_bytes": len(block)}
    nsl = -(-m.rows // RC.SLICE_HEIGHT)
    rs = np.asarray(m.row_start, dtype=np.int64)
    dl = deltas
    pl = patterns
    tables = (dt, vt)
    raw = (32, precision * 8)
    slices = []
    for s in sample_slices(nsl):
        lo, hi = s * RC.SLICE_HEIGHT, min((s + 1) * RC.SLICE_HEIGHT, m.rows)
        streams, traces, nsym = [], [], []
        for i in range(lo, hi):
            a, b = int(rs[i]), int(rs[i + 1])
            u = RC.row_symbol_list(dl[a:b].tolist(), pl[a:b].tolist(), 0, b - a)
            nsym.append(len(u))
            v, tr = dtans_encode(u, tables, params, raw)
            streams.append(v)
            traces.append(tr)
        words, sched = RC.interleave_warp(streams, traces, params)
        sched.check_coalescing()
        w = np.asarray(words, dtype=np.uint32)
        slices.append({"slice": int(s), "words": int(len(w)), "sha256": hashlib.sha256(w.tobytes()).hexdigest(),
                       "row_symbols_sha256": hashlib.sha256(np.asarray(nsym, np.uint32).tobytes()).hexdigest()})
    rec["slices"] = slices
    rec["seconds"] = {"distributions": round(t1 - t0, 1), "quantize_tables": round(t2 - t1, 1),
                      "slices": round(time.time() - t2, 1)}
    return rec


def main():
    want = set(sys.argv[1:])
    out = {}
    if os.path.exists(OUT):
        out = json.load(open(OUT))
    out["_about"] = ("reference encoder at BASELINE size: full-size quantize + build_tables, "
                     f"{NSAMPLE} sampled slices of dtans_encode + interleave_warp "
                     "(tests/golden/make_fullscale_golden.py)")
    for name, gen in matrices():
        if want and name not in want:
            continue
        t = time.time()
        out[name] = run(name, gen)
        print(name, f"{time.time() - t:.0f}s", {k: v for k, v in out[name].items() if k != "slices"}, flush=True)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
