"""Quick CUDA-event timing of the fused kernel on the config-2 Laplacian."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth

g = int(sys.argv[1]) if len(sys.argv) > 1 else 2591
t0 = time.time(); m = synth.laplacian_2d(g); t1 = time.time()
c = P.encode_matrix(m); t2 = time.time()
print(f"gen {t1-t0:.2f}s encode {t2-t1:.2f}s nnz={m.nnz} words={len(c.stream)} size={P.size_bytes(c)} ratio={P.compression_ratio(m, c):.3f}", flush=True)
x, y = synth.vectors(m)
dev = c.device(0)
print(dev.info())
xt = torch.from_numpy(x).cuda(); yt = torch.from_numpy(y).cuda(); out = torch.empty_like(yt)
for _ in range(5): dev.spmv(xt, yt, out)
dev.check()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(20):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); dev.spmv(xt, yt, out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = np.median(ts) * 1e-3
B = P.size_bytes(c) + 8 * m.cols + 16 * m.rows
print(f"median {t*1e6:.1f} us  GFLOP/s {2*m.nnz/t/1e9:.1f}  eff GB/s {B/t/1e9:.1f}  frac {B/t/1e9/6502.5:.3f}")
# cuSPARSE comparator via torch
A = torch.sparse_csr_tensor(torch.from_numpy(m.row_start), torch.from_numpy(m.col_idx), torch.from_numpy(m.values), size=(m.rows, m.cols)).cuda()
for _ in range(3): torch.addmv(yt, A, xt)
ts = []
for _ in range(20):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); torch.addmv(yt, A, xt); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"cusparse (torch.addmv) median {np.median(ts)*1e3:.1f} us")
