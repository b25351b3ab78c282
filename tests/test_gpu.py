"""GPU parity tests: the sm_100a kernels against the reference goldens and
the oracle.  Run on a B200 with `pytest -m gpu`."""

import numpy as np
import pytest

import golden_cases as G
import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

SPMV_CASES = [n for n in G.names() if "spmv" in G.load(n)]


@pytest.mark.parametrize("name", SPMV_CASES)
def test_spmv_bitwise_reference(name):
    rec = G.load(name)
    c = P.encode_matrix(G.matrix(rec), **G.encode_kwargs(rec))
    out = P.spmv(c, rec["x"], rec["y"])
    assert G.check_spmv(out, rec["spmv"], G.matrix(rec), rec["x"], rec["y"], c=c)


@pytest.mark.parametrize("name", G.names())
def test_decode_bit_exact(name):
    rec = G.load(name)
    m = G.matrix(rec)
    c = P.encode_matrix(m, **G.encode_kwargs(rec))
    d = P.decode_matrix(c)
    vdt = np.float64 if c.precision == 8 else np.float32
    assert d == P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx, m.values.astype(vdt))


@pytest.mark.parametrize("name", [n for n in SPMV_CASES if "container" in G.load(n)])
def test_spmv_from_reference_bytes(name):
    rec = G.load(name)
    c = P.deserialize(rec["container"].tobytes())
    out = P.spmv(c, rec["x"], rec["y"])
    assert G.check_spmv(out, rec["spmv"], G.matrix(rec), rec["x"], rec["y"], c=c)


def test_corrupt_directory_raises():
    rec = G.load("laplacian_g48")
    c = P.encode_matrix(G.matrix(rec))
    d = c.directory.copy()
    d[1:-1] += 1  # every slice boundary shifted by one word
    c.directory = d
    with pytest.raises(P.CorruptStream):
        P.spmv(c, rec["x"], rec["y"])


def test_device_tensor_path_and_y_none():
    m = synth.laplacian_2d(300)
    x, y = synth.vectors(m)
    c = P.encode_matrix(m)
    dev = c.device(0)
    xt = torch.from_numpy(x).cuda()
    yt = torch.from_numpy(y).cuda()
    out = dev.spmv(xt, yt)
    dev.check()
    oc = O.parse(P.serialize(c))
    assert G.same_bits_or_nan(out.cpu().numpy(), O.spmv(oc, x, y))
    out0 = dev.spmv(xt, None)
    dev.check()
    assert G.same_bits_or_nan(out0.cpu().numpy(), O.spmv(oc, x, np.zeros_like(y)))


@pytest.mark.parametrize("gen", [
    lambda: synth.laplacian_2d(700),
    lambda: synth.banded(60000, 27),
    lambda: synth.banded(40000, 32, positive=True),
    lambda: synth.rmat(14, 200000),
    lambda: synth.rmat(12, 40000, dtype=np.float64),
    lambda: synth.config1_random(20000, 300000, seed=4),
])
def test_larger_matrices_vs_oracle(gen):
    m = gen()
    x, y = synth.vectors(m)
    c = P.encode_matrix(m)
    assert P.decode_matrix(c) == m
    out = P.spmv(c, x, y)
    ref = O.spmv(O.parse(P.serialize(c)), x, y, threads=8)
    assert G.check_spmv(out, ref, m, x, y, c=c)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_spmv_on_gpu_equals_full(world):
    from paper_2603_01915_b200 import distributed as D
    m = synth.rmat(13, 60000, seed=5)
    x, y = synth.vectors(m)
    c = P.encode_matrix(m)
    full = P.spmv(c, x, y)
    b = D.shard_bounds(c, world)
    xt = torch.from_numpy(x).cuda()
    for i, (r0, r1) in enumerate(D.shard_rows(c, b)):
        sc = D.shard(c, int(b[i]), int(b[i + 1]))
        out = sc.device(0).spmv(xt, torch.from_numpy(y[r0:r1]).cuda()) if sc.rows else None
        if sc.rows:
            sc.device(0).check()
            o = out.cpu().numpy()
            lr = G.long_slice_rows(m.row_start[r0:r1 + 1] - m.row_start[r0], r1 - r0) | \
                sc.device(0).split_rows(r1 - r0) | c.device(0).split_rows(m.rows)[r0:r1]
            assert G.same_bits_or_nan(o[~lr], full[r0:r1][~lr])
            assert np.allclose(o[lr], full[r0:r1][lr], rtol=1e-5, atol=1e-4)


def test_power_iteration_single_gpu():
    from paper_2603_01915_b200 import distributed as D
    m = synth.banded(20000, 32, positive=True, seed=3)
    c = P.encode_matrix(m)
    op = D.ShardedSpMV(c, 0, 1, device=torch.device("cuda", 0))
    x0 = torch.full((m.cols,), 1.0 / np.sqrt(m.cols), dtype=torch.float64, device="cuda")
    x, lam = D.power_iteration(op, x0, 30)
    xr, lr = D.reference_power_iteration(m, np.full(m.cols, 1.0 / np.sqrt(m.cols)), 30)
    assert abs(lam - lr) <= 1e-12 * lr
    assert np.allclose(x.cpu().numpy(), xr, rtol=1e-11, atol=1e-14)


@pytest.mark.parametrize("long_seg", ["4", "64"])
def test_long_slice_tasks_match_oracle(long_seg, monkeypatch):
    """Skewed rows: checkpointed segment-range tasks (checkpoints.cpp) decode
    bit-exactly and sum within tolerance; a small threshold forces almost
    every slice through the task kernel."""
    monkeypatch.setenv("DTANS_LONG_SEG", long_seg)
    monkeypatch.setenv("DTANS_CHUNK", "3")
    for gen in (lambda: synth.rmat(13, 80000, seed=9), lambda: synth.banded(3000, 27, seed=2)):
        m = gen()
        x, y = synth.vectors(m)
        c = P.encode_matrix(m)
        assert P.decode_matrix(c) == m
        out = P.spmv(c, x, y)
        ref = O.spmv(O.parse(P.serialize(c)), x, y, threads=8)
        tol = 1e-12 if m.values.dtype == np.float64 else 1e-5
        s = np.abs(m.values.astype(np.float64)) * np.abs(x.astype(np.float64))[m.col_idx]
        s = np.bincount(np.repeat(np.arange(m.rows), np.diff(m.row_start)), weights=s, minlength=m.rows)
        assert np.all(np.abs(out.astype(np.float64) - ref) <= tol * (s + np.abs(y)))


@pytest.mark.parametrize("window", [None, 4096])
def test_row_reordered_rmat(window):
    """sort_rows_by_length + row_map: results in the original row order."""
    m = synth.rmat(14, 150000, seed=11)
    x, y = synth.vectors(m)
    pm, perm = P.sort_rows_by_length(m, window)
    c = P.encode_matrix(pm)
    c.row_map = perm
    out = P.spmv(c, x, y)
    ref_p = O.spmv(O.parse(P.serialize(c)), x, y[perm.astype(np.int64)], threads=8)
    ref = np.empty_like(ref_p)
    ref[perm.astype(np.int64)] = ref_p
    exp_p = np.empty_like(out)
    exp_p = out[perm.astype(np.int64)]
    assert G.check_spmv(exp_p, ref_p, pm, x, y[perm.astype(np.int64)], c=c)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_power_iteration_fused_matches_unfused(dtype):
    """dtans_spmv_scaled (scale + sum of squares in the SpMV epilogue) gives
    the same iterates as the unfused loop (spmv, dot, divide) within the
    north-star tolerance, and matches numpy."""
    from paper_2603_01915_b200 import distributed as D
    m = synth.banded(30000, 32, positive=True, seed=7)
    if dtype == np.float32:
        m = P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx, m.values.astype(np.float32))
    c = P.encode_matrix(m)
    op = D.ShardedSpMV(c, 0, 1, device=torch.device("cuda", 0))
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    x0 = torch.full((m.cols,), 1.0 / np.sqrt(m.cols), dtype=tdt, device="cuda")
    xf, lf = D.power_iteration(op, x0, 25, fused=True)
    xu, lu = D.power_iteration(op, x0, 25, fused=False)
    op._dev.check()
    tol = 1e-12 if dtype == np.float64 else 1e-5
    assert abs(lf - lu) <= tol * lu
    assert np.allclose(xf.cpu().numpy(), xu.cpu().numpy(), rtol=10 * tol, atol=10 * tol / np.sqrt(m.cols))
    xr, lr = D.reference_power_iteration(m, np.full(m.cols, 1.0 / np.sqrt(m.cols)), 25)
    assert abs(lf - lr) <= 10 * tol * lr


def test_symmetric_reordered_rmat():
    """sort_symmetric_by_degree + row_map + col_map: y = A x in the original
    order (the device gathers x' = x[perm] first)."""
    m = synth.rmat(14, 150000, seed=12)
    x, y = synth.vectors(m)
    pm, perm = P.sort_symmetric_by_degree(m)
    c = P.encode_matrix(pm)
    c.row_map = perm
    c.col_map = perm
    out = P.spmv(c, x, y)
    p64 = perm.astype(np.int64)
    ref_p = O.spmv(O.parse(P.serialize(c)), x[p64], y[p64], threads=8)
    assert G.check_spmv(out[p64], ref_p, pm, x[p64], y[p64], c=c)
    # and through the device-tensor path
    dev = c.device(0)
    o2 = dev.spmv(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    dev.check()
    assert G.same_bits_or_nan(o2.cpu().numpy(), out)


def _host_vs_device(c, x, y, stages=None, monkeypatch=None, pinned=False):
    """dtans_spmv_host with pageable numpy buffers (staged through the
    library's pinned buffers) or pinned ones (the pipelined chunk path)."""
    if stages is not None:
        monkeypatch.setenv("DTANS_HOST_STAGES", str(stages))
    dc = c.device(0)
    V = np.float64 if c.precision == 8 else np.float32

    def host(a):
        a = np.ascontiguousarray(a, V)
        return torch.from_numpy(a).pin_memory().numpy() if pinned else a
    out = host(np.full(c.rows, np.nan, dtype=V))
    dc.spmv_host(host(x), None if y is None else host(y), out)
    xt = torch.from_numpy(np.ascontiguousarray(x, V)).cuda()
    yt = None if y is None else torch.from_numpy(np.ascontiguousarray(y, V)).cuda()
    ref = dc.spmv(xt, yt).cpu().numpy()
    dc.close()
    return out, ref


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("stages", [1, 8, 32])
@pytest.mark.parametrize("gen", ["laplacian", "banded", "random"])
def test_host_buffer_path_matches_device_path(gen, stages, pinned, monkeypatch):
    """dtans_spmv_host (pinned: pipelined H2D / kernel on chunk ranges / D2H;
    pageable: staged copies) equals the device-pointer path bitwise."""
    m = {"laplacian": lambda: synth.laplacian_2d(700),
         "banded": lambda: synth.banded(200000, 27, levels=256, seed=4),
         "random": lambda: synth.config1_random(20000, 300000, seed=3)}[gen]()
    x, y = synth.vectors(m)
    c = P.encode_matrix(m)
    out, ref = _host_vs_device(c, x, y, stages, monkeypatch, pinned)
    assert np.array_equal(out, ref)
    out0, ref0 = _host_vs_device(c, x, None, stages, monkeypatch, pinned)
    assert np.array_equal(out0, ref0)


def test_host_buffer_path_row_reordered():
    """A row map scatters y'/y: the host path must not pipeline row ranges."""
    m = synth.banded(100000, 9, levels=64, seed=2)
    pm, perm = P.sort_rows_by_length(m)
    c = P.encode_matrix(pm)
    c.row_map = perm
    x, y = synth.vectors(m)
    out, ref = _host_vs_device(c, x, y)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_nccl_power_iteration_c_abi(dtype):
    """dtans_mg_power_iteration (NCCL all-reduce + grouped broadcasts in the
    C ABI) on a one-rank communicator matches the torch-driven fused power
    iteration and the numpy reference.  Not bitwise: sum(y^2) is accumulated
    with per-warp f64 atomics, whose order varies from run to run."""
    from paper_2603_01915_b200 import distributed as D
    m = synth.banded(20000, 32, positive=True, seed=3)
    if dtype == np.float32:
        m = P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx, m.values.astype(np.float32))
    c = P.encode_matrix(m)
    op = D.ShardedSpMV(c, 0, 1, device=torch.device("cuda", 0))
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    x0 = torch.full((m.cols,), 1.0 / np.sqrt(m.cols), dtype=tdt, device="cuda")
    x_t, lam_t = D.power_iteration(op, x0, 25)
    comm = D.NcclComm(1, 0, 0, D.NcclComm.unique_id())
    x_c, lam_c = comm.power_iteration(op._dev, [0, m.rows], x0, 25)
    torch.cuda.synchronize()
    tol = 1e-12 if dtype == np.float64 else 1e-5
    assert abs(lam_c - lam_t) <= tol * lam_t
    assert torch.allclose(x_c, x_t, rtol=10 * tol, atol=0)
    xr, lr = D.reference_power_iteration(m, np.full(m.cols, 1.0 / np.sqrt(m.cols)), 25)
    assert abs(lam_c - lr) <= tol * lr
    assert np.allclose(x_c.double().cpu().numpy(), xr, rtol=100 * tol, atol=1e-14 if dtype == np.float64 else 1e-7)
    comm.close()


def test_nccl_power_iteration_rejects_bad_layout():
    from paper_2603_01915_b200 import distributed as D
    m = synth.banded(5000, 8, positive=True, seed=1)
    c = P.encode_matrix(m)
    dev = c.device(0)
    comm = D.NcclComm(1, 0, 0, D.NcclComm.unique_id())
    x0 = torch.ones(m.cols, dtype=torch.float64, device="cuda")
    with pytest.raises(P.ParameterError):
        comm.power_iteration(dev, [0, m.rows - 1], x0, 3)
    comm.close()
