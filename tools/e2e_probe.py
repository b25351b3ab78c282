"""e2e probe: the host-buffer path (dtans_spmv_host, pinned x/y/out, copies
inside) for several pipeline depths (DTANS_HOST_STAGES, read per call),
interleaved, against the PCIe floor (tools/pcie_probe.py)."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_01915_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "laplacian"
spec = bench.Spec(cfg, 1.0)
m = spec.block(0, spec.rows)
c = P.encode_matrix(m)
x, y = spec.vectors(0, spec.rows)
dc = c.device(0)
xh = torch.from_numpy(x).pin_memory().numpy()
yh = torch.from_numpy(y).pin_memory().numpy()
oh = torch.empty(m.rows, dtype=torch.from_numpy(x).dtype).pin_memory().numpy()
res = {}
for rnd in range(3):
    for st in [int(v) for v in os.environ.get("PROBE_STAGES", "4 8 16 24 32").split()]:
        os.environ["DTANS_HOST_STAGES"] = str(st)
        for _ in range(2):
            dc.spmv_host(xh, yh, oh)
        t0 = time.perf_counter()
        for _ in range(20):
            dc.spmv_host(xh, yh, oh)
        res.setdefault(st, []).append((time.perf_counter() - t0) / 20 * 1e3)
for st, v in res.items():
    print(cfg, "stages", st, "ms", " ".join(f"{t:.3f}" for t in v))
