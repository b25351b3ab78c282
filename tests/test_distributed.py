"""Row sharding and the power-iteration driver, multi-process on CPU (gloo,
world_size 2) with the oracle standing in for the per-GPU kernel."""

import os
import socket

import numpy as np
import pytest

import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import distributed as D
from paper_2603_01915_b200 import synth
from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("balance", ["nnz", "words"])
def test_shard_bounds_cover_and_balance(world, balance):
    m = synth.rmat(11, 20000, seed=2)
    c = P.encode_matrix(m)
    b = D.shard_bounds(c, world, balance)
    assert b[0] == 0 and b[-1] == c.nslices and np.all(np.diff(b) >= 0)
    if balance == "nnz":
        nnz_row = np.diff(m.row_start)
        per = [nnz_row[r0:r1].sum() for r0, r1 in D.shard_rows(c, b)]
        slice_max = max(nnz_row[i:i + 32].sum() for i in range(0, m.rows, 32))
        assert max(per) - min(per) <= 2 * slice_max


@pytest.mark.parametrize("world", [2, 3])
def test_shards_decode_to_row_blocks(world):
    m = synth.banded(1000, 9, levels=17, seed=4)
    c = P.encode_matrix(m)
    x, y = synth.vectors(m)
    full = O.spmv(O.parse(P.serialize(c)), x, y)
    b = D.shard_bounds(c, world)
    for i, (r0, r1) in enumerate(D.shard_rows(c, b)):
        sc = D.shard(c, int(b[i]), int(b[i + 1]))
        oc = O.parse(P.serialize(sc))           # a valid container on its own
        rs, cols, vals = O.decode(oc)
        assert np.array_equal(rs, m.row_start[r0:r1 + 1] - m.row_start[r0])
        assert np.array_equal(cols, m.col_idx[m.row_start[r0]:m.row_start[r1]])
        assert np.array_equal(O.spmv(oc, x, y[r0:r1]), full[r0:r1])


def _oracle_spmv_fn(local):
    import torch
    oc = O.parse(P.serialize(local))

    def fn(x, y, out):
        yy = np.zeros(local.rows) if y is None else y.numpy()
        out.copy_(torch.from_numpy(O.spmv(oc, x.numpy(), yy)))
        return out
    return fn


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = synth.banded(3000, 12, levels=16, seed=7, positive=True)
        c = P.encode_matrix(m)
        b = D.shard_bounds(c, world)
        local = D.shard(c, int(b[rank]), int(b[rank + 1]))
        op = D.ShardedSpMV(c, rank, world, spmv_fn=_oracle_spmv_fn(local), bounds=b)
        x0 = torch.full((m.cols,), 1.0 / np.sqrt(m.cols), dtype=torch.float64)
        x, lam = D.power_iteration(op, x0, 25)
        if rank == 0:
            q.put((x.numpy(), lam))
    finally:
        dist.destroy_process_group()


def test_power_iteration_gloo_world2():
    import torch.multiprocessing as mp
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    x, lam = q.get()
    m = synth.banded(3000, 12, levels=16, seed=7, positive=True)
    xr, lr = D.reference_power_iteration(m, np.full(m.cols, 1.0 / np.sqrt(m.cols)), 25)
    assert abs(lam - lr) <= 1e-12 * abs(lr)
    assert np.allclose(x, xr, rtol=1e-12, atol=1e-15)
