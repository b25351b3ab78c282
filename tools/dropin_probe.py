"""Where the drop-in spmv's time goes (pageable numpy buffers): fresh output
per call vs a reused output vs pinned buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth
m = synth.laplacian_2d(2591)
c = P.encode_matrix(m)
x, y = synth.vectors(m)
dc = c.device(0)
def t(f, n=10):
    f(); f()
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e3
out = np.empty(c.rows)
print("drop-in P.spmv          ms", t(lambda: P.spmv(c, x, y)))
print("np.empty only           ms", t(lambda: np.empty(c.rows).fill(0)))
print("spmv_host reused out    ms", t(lambda: dc.spmv_host(x, y, out)))
xh = torch.from_numpy(x).pin_memory().numpy(); yh = torch.from_numpy(y).pin_memory().numpy()
oh = torch.empty(c.rows, dtype=torch.float64).pin_memory().numpy()
print("spmv_host pinned        ms", t(lambda: dc.spmv_host(xh, yh, oh)))
print("spmv_host pinned in, pageable reused out ms", t(lambda: dc.spmv_host(xh, yh, out)))
