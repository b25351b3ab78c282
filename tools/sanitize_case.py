"""Small SpMV/decode cases for compute-sanitizer (memcheck / racecheck /
synccheck): the main kernel (chunks of several slices), the long-slice task
kernel (streamed windows), the solo and finalize kernels, the scaled power-
iteration step, the host-buffer path, and a rows-sorted R-MAT through the
default long-slice launch chain (empty-slice kernel, PDL).  Each result is checked against
the oracle so a sanitizer run is also a parity run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01915_b200 as P  # noqa: E402
from paper_2603_01915_b200 import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker)

os.environ.setdefault("DTANS_KCHUNK", "4")
cases = [("laplacian", synth.laplacian_2d(120)), ("banded27", synth.banded(4000, 27, seed=1)),
         ("rmat_f32", synth.rmat(11, 30000, seed=3)), ("random_f64", synth.config1_random(3000, 40000, seed=2))]
os.environ["DTANS_LONG_SEG"] = "6"  # force long slices (task + solo + finalize kernels)
for name, m in cases:
    x, y = synth.vectors(m)
    c = P.encode_matrix(m)
    out = P.spmv(c, x, y)
    ref = O.spmv(O.parse(P.serialize(c)), x, y, threads=4)
    tol = 1e-12 if m.values.dtype == np.float64 else 1e-5
    s = np.abs(m.values.astype(np.float64)) * np.abs(x.astype(np.float64))[m.col_idx]
    s = np.bincount(np.repeat(np.arange(m.rows), np.diff(m.row_start)), weights=s, minlength=m.rows) + np.abs(y)
    assert np.all(np.abs(out.astype(np.float64) - ref) <= tol * s), name
    assert P.decode_matrix(c) == P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx, m.values.astype(c.value_dtype))
    dev = c.device(0)
    xt = torch.from_numpy(x).cuda()
    S = torch.tensor([4.0, 0.0, 1.0], dtype=torch.float64, device="cuda")
    o2 = torch.empty(m.rows, dtype=xt.dtype, device="cuda")
    dev.spmv_scaled(xt, o2, S[0:1], S[1:2], S[2:3])
    dev.check()
    oh = np.empty_like(y)
    dev.spmv_host(x, y, oh)
    print(name, "ok", dev.plan())
# rows-sorted R-MAT with the default planner: every non-empty slice is a
# task, all-empty slices go to the empty-slice kernel, and the solo, task and
# finalize launches are chained with programmatic dependent launch; several
# products back to back on one stream (PDL main kernel)
os.environ.pop("DTANS_LONG_SEG")
os.environ.pop("DTANS_KCHUNK")
m = synth.rmat(13, 60000, seed=5)
pm, perm = P.sort_rows_by_length(m)
c = P.encode_matrix(pm)
c.row_map = perm
p64 = perm.astype(np.int64)
x, y = synth.vectors(m)
out = P.spmv(c, x, y)
ref = O.spmv(O.parse(P.serialize(c)), x, y[p64], threads=4)
s = np.abs(pm.values.astype(np.float64)) * np.abs(x.astype(np.float64))[pm.col_idx]
s = np.bincount(np.repeat(np.arange(pm.rows), np.diff(pm.row_start)), weights=s, minlength=pm.rows) + np.abs(y[p64])
assert np.all(np.abs(out[p64].astype(np.float64) - ref) <= 1e-5 * s), "rmat sorted"
dev = c.device(0)
plan = dev.plan()
assert plan["nlong"] > 0 and plan["nempty"] > 0, plan
xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for _ in range(3):
    yt = dev.spmv(xt, yt)
dev.check()
print("rmat_sorted ok", plan)
torch.cuda.synchronize()
print("sanitize cases ok")
