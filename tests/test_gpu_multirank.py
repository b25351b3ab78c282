"""Two ranks sharing cuda:0 over gloo run the sharded product and the fused
power iteration with the CUDA kernel (not an injected SpMV), checked against
the oracle and a numpy power iteration.  Only one GPU is available here, so
NCCL (which refuses two ranks on one device) is replaced by gloo; the data
path is the same ShardedSpMV / power_iteration code bench.py runs at N>1.
Reference shard model: /root/reference/pkg/src/csrdtans/container.py:583-595."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, dtype_name):
    import torch.distributed as dist

    import paper_2603_01915_b200 as P
    from paper_2603_01915_b200 import distributed as D
    from paper_2603_01915_b200 import synth
    from oracle import oracle as O
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dtype = np.float64 if dtype_name == "f64" else np.float32
    dev = torch.device("cuda", 0)
    # single SpMV over nnz-balanced shards of a skewed matrix (long slices too)
    m = synth.rmat(13, 70000, seed=4, dtype=dtype)
    x, y = synth.vectors(m)
    c = P.encode_matrix(m)
    op = D.ShardedSpMV(c, rank, world, device=dev)
    r0, r1 = op.rows_of[rank]
    out = op.spmv(torch.from_numpy(x).to(dev), torch.from_numpy(y[r0:r1]).to(dev)).cpu().numpy()
    op._dev.check()
    ref = O.spmv(O.parse(P.serialize(op.local)), x, y[r0:r1], threads=4)
    np.save(os.path.join(outdir, f"spmv_{rank}.npy"), out)
    np.save(os.path.join(outdir, f"spmv_ref_{rank}.npy"), ref)
    # fused power iteration (banded positive: a Perron vector exists)
    mb = synth.banded(20000, 32, positive=True, seed=3)
    if dtype == np.float32:
        mb = P.CsrMatrix(mb.rows, mb.cols, mb.row_start, mb.col_idx, mb.values.astype(np.float32))
    cb = P.encode_matrix(mb)
    opb = D.ShardedSpMV(cb, rank, world, device=dev)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    x0 = torch.full((mb.cols,), 1.0 / np.sqrt(mb.cols), dtype=tdt, device=dev)
    xk, lam = D.power_iteration(opb, x0, 25)
    xu, lu = D.power_iteration(opb, x0, 25, fused=False)
    np.save(os.path.join(outdir, f"pit_{rank}.npy"), np.concatenate([[lam, lu], xk.double().cpu().numpy(),
                                                                     xu.double().cpu().numpy()]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dtype_name", ["f64", "f32"])
def test_two_gloo_ranks_on_one_gpu(tmp_path, dtype_name):
    import torch.multiprocessing as mp

    import golden_cases as G
    import paper_2603_01915_b200 as P
    from paper_2603_01915_b200 import distributed as D
    from paper_2603_01915_b200 import synth
    world = 2
    mp.spawn(_worker, args=(world, _port(), str(tmp_path), dtype_name), nprocs=world, join=True)
    dtype = np.float64 if dtype_name == "f64" else np.float32
    m = synth.rmat(13, 70000, seed=4, dtype=dtype)
    x, y = synth.vectors(m)
    c = P.encode_matrix(m)
    b = D.shard_bounds(c, world)
    for r, (r0, r1) in enumerate(D.shard_rows(c, b)):
        out = np.load(tmp_path / f"spmv_{r}.npy")
        ref = np.load(tmp_path / f"spmv_ref_{r}.npy")
        sub = D.shard(c, int(b[r]), int(b[r + 1]))
        rs = m.row_start[r0:r1 + 1] - m.row_start[r0]
        ms = P.CsrMatrix(r1 - r0, m.cols, rs, m.col_idx[m.row_start[r0]:m.row_start[r1]],
                         m.values[m.row_start[r0]:m.row_start[r1]])
        assert sub.rows == r1 - r0
        assert G.check_spmv(out, ref, ms, x, y[r0:r1], c=sub)
    mb = synth.banded(20000, 32, positive=True, seed=3)
    xr, lr = D.reference_power_iteration(mb, np.full(mb.cols, 1.0 / np.sqrt(mb.cols)), 25)
    tol = 1e-12 if dtype == np.float64 else 1e-5
    for r in range(world):
        v = np.load(tmp_path / f"pit_{r}.npy")
        lam, lu, xk, xu = v[0], v[1], v[2:2 + mb.cols], v[2 + mb.cols:]
        assert abs(lam - lr) <= 10 * tol * lr
        assert abs(lu - lr) <= 10 * tol * lr
        assert np.allclose(xk, xr, rtol=100 * tol, atol=1e-14 if dtype == np.float64 else 1e-7)
        assert np.allclose(xu, xr, rtol=100 * tol, atol=1e-14 if dtype == np.float64 else 1e-7)
