"""Lean kernel timing for A/B iterations and ncu captures (not the bench).

    python tools/kbench.py [--config laplacian|banded27|rmat|banded32] [--scale S]
                           [--reorder] [--iters N] [--check] [--launches N]

Builds the bench.py workload (bench.Spec), uploads it and times the fused
SpMV with CUDA events: the median of back-to-back launch groups and of
single cold-L2 launches.  --check compares one result against the oracle
(bitwise).  --launches N just runs N launches (for ncu -s/-c captures).
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_01915_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="laplacian")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reorder", action="store_true")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--launches", type=int, default=0)
    ap.add_argument("--noy", action="store_true", help="y-less product (power-iteration form)")
    ap.add_argument("--cache", default=None, help="directory of encoded containers (CDTA + row map) to reuse")
    ap.add_argument("--env", action="append", default=[], help="KEY=VALUE set before the upload (plan knobs)")
    a = ap.parse_args()
    for kv in a.env:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    spec = bench.Spec(a.config, a.scale)
    t0 = time.time()
    perm = None
    key = f"{a.config}_{a.scale}_{int(a.reorder)}"
    cpath = os.path.join(a.cache, key + ".cdta") if a.cache else None
    if cpath and os.path.exists(cpath):
        c = P.load(cpath)
        if a.reorder:
            perm = np.load(cpath + ".perm.npy")
        m = None
    else:
        m = spec.block(0, spec.rows)
        if a.reorder:
            m, perm = P.sort_rows_by_length(m)
        c = P.encode_matrix(m)
        if cpath:
            os.makedirs(a.cache, exist_ok=True)
            P.save(c, cpath)
            if perm is not None:
                np.save(cpath + ".perm.npy", perm)
    if perm is not None:
        c.row_map = perm
    t_enc = time.time() - t0
    x, y = spec.vectors(0, spec.rows)
    t0 = time.time()
    dc = c.device(0)
    t_up = time.time() - t0
    xt = torch.from_numpy(x).cuda()
    yt = None if a.noy else torch.from_numpy(y).cuda()
    out = torch.empty(c.rows, dtype=xt.dtype, device="cuda")
    if a.launches:
        for _ in range(a.launches):
            dc.spmv(xt, yt, out)
        torch.cuda.synchronize()
        dc.check()
        print(json.dumps({"launches": a.launches, "info": dc.info()}))
        return
    for _ in range(5):
        dc.spmv(xt, yt, out)
    torch.cuda.synchronize()
    dc.check()
    reps = 10
    warm = []
    for _ in range(max(1, a.iters // reps)):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dc.spmv(xt, yt, out)
        e1.record()
        torch.cuda.synchronize()
        warm.append(e0.elapsed_time(e1) / reps)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cold = []
    for _ in range(10):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        dc.spmv(xt, yt, out)
        e1.record()
        torch.cuda.synchronize()
        cold.append(e0.elapsed_time(e1))
    dc.check()
    esz = c.precision
    alg = P.size_bytes(c) + esz * c.cols + (esz if a.noy else 2 * esz) * c.rows
    pk = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    tw = float(np.median(warm))
    tc = float(np.median(cold))
    res = {"config": a.config, "scale": a.scale, "reorder": a.reorder, "nnz": int(c.nnz), "lib": os.environ.get("DTANS_LIB", "in-tree"), "encode_s": round(t_enc, 1), "upload_s": round(t_up, 3),
           "warm_ms": round(tw, 5), "cold_ms": round(tc, 5), "frac_warm": round(alg / (tw * 1e-3) / 1e9 / pk, 4),
           "frac_cold": round(alg / (tc * 1e-3) / 1e9 / pk, 4), "plan": dc.plan()}
    if a.check:
        from oracle import oracle as O
        oc = O.parse(P.serialize(c))
        yy = np.zeros_like(y) if a.noy else y
        xx = x
        if perm is not None:
            p64 = perm.astype(np.int64)
            yy = yy[p64]
        ref = O.spmv(oc, xx, yy, threads=os.cpu_count() or 1)
        o = out.cpu().numpy()
        if perm is not None:
            o = o[perm.astype(np.int64)]
        ui = np.uint64 if esz == 8 else np.uint32
        same = (o.view(ui) == ref.view(ui)) | (np.isnan(o) & np.isnan(ref))
        res["bitwise_rows"] = int(same.sum())
        res["rows"] = int(len(o))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
