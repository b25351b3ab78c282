"""Parity of the kernel configuration the full-size benchmarks run.

Every config at BASELINE scale packs several consecutive slices into one
staged chunk (api.cu: kcap = nslices / (148 * 32 * 4), clamped to [1, 16]),
so the main kernel's per-warp multi-slice loop runs there (kernels.cuh:
the slice-end offsets, per-slice metadata and row_symbols of a chunk blob).
Small test matrices get kcap = 1 by default; DTANS_KCHUNK forces the
multi-slice chunks here and dtans_plan proves they were used.  Reference
semantics: spmv /root/reference/pkg/src/csrdtans/container.py:554-596,
decode_matrix :524-531."""

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
KCHUNKS = ["2", "5", "16"]

MID = {
    "laplacian700": lambda: synth.laplacian_2d(700),
    "banded27": lambda: synth.banded(60000, 27),
    "banded32pos": lambda: synth.banded(40000, 32, positive=True),
    "rmat14_f32": lambda: synth.rmat(14, 200000),
    "rmat12_f64": lambda: synth.rmat(12, 40000, dtype=np.float64),
    "random20000": lambda: synth.config1_random(20000, 300000, seed=4),
}


def _fresh(c):
    """Drop cached device handles so the next upload sees the environment."""
    for k in [k for k in c._cache if isinstance(k, tuple) and k[0] == "dev"]:
        c._cache.pop(k).close()
    return c


def _pair_fits(c, bufb):
    """Whether two adjacent slices fit one staging buffer (api.cu
    chunk_words: next record + padded header + 2*32 row_symbols + the padded
    stream words)."""
    d = np.asarray(c.directory, dtype=np.int64)
    if len(d) < 3:
        return False
    words = 8 + 64 + ((d[2:] - d[:-2] + 3) & ~3)
    return bool((4 * words <= bufb).any())


def _assert_multichunk(dc, c, kchunk):
    plan = dc.plan()
    # skewed unsorted matrices are scheduled as single-slice chunks, longest
    # first (api.cu, dynamic plan), whatever DTANS_KCHUNK says
    if plan["staged_slices"] >= 2 and int(kchunk) >= 2 and _pair_fits(c, plan["bufb"]) and not plan["dynamic"]:
        assert plan["chunk_slices_max"] >= 2, plan
    return plan


@pytest.mark.parametrize("kchunk", KCHUNKS)
@pytest.mark.parametrize("name", SPMV_CASES)
def test_goldens_multichunk(name, kchunk, monkeypatch):
    """spmv bitwise vs the reference's own spmv output, decode bit-exact,
    with multi-slice chunks."""
    monkeypatch.setenv("DTANS_KCHUNK", kchunk)
    rec = G.load(name)
    m = G.matrix(rec)
    c = _fresh(P.encode_matrix(m, **G.encode_kwargs(rec)))
    out = P.spmv(c, rec["x"], rec["y"])
    _assert_multichunk(c.device(0), c, kchunk)
    assert G.check_spmv(out, rec["spmv"], m, rec["x"], rec["y"], c=c)
    vdt = np.float64 if c.precision == 8 else np.float32
    assert P.decode_matrix(c) == P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx, m.values.astype(vdt))


def _scaled_expect(ref_noy, q, V):
    scale = V(1.0 / np.sqrt(np.float64(q)))
    with np.errstate(all="ignore"):
        return (ref_noy * scale).astype(V)


@pytest.mark.parametrize("kchunk", KCHUNKS)
@pytest.mark.parametrize("gen", list(MID))
def test_mid_matrices_multichunk(gen, kchunk, monkeypatch):
    """SpMV, y-less SpMV, the scaled power-iteration step and decode against
    the oracle, with multi-slice chunks (bitwise except split long rows)."""
    monkeypatch.setenv("DTANS_KCHUNK", kchunk)
    m = MID[gen]()
    x, y = synth.vectors(m)
    c = _fresh(P.encode_matrix(m))
    V = c.value_dtype
    dc = c.device(0)
    _assert_multichunk(dc, c, kchunk)
    oc = O.parse(P.serialize(c))
    ref = O.spmv(oc, x, y, threads=8)
    xt = torch.from_numpy(np.ascontiguousarray(x, V)).cuda()
    yt = torch.from_numpy(np.ascontiguousarray(y, V)).cuda()
    out = dc.spmv(xt, yt).cpu().numpy()
    dc.check()
    assert G.check_spmv(out, ref, m, x, y, c=c)
    ref0 = O.spmv(oc, x, np.zeros_like(y), threads=8)
    out0 = dc.spmv(xt, None).cpu().numpy()
    dc.check()
    assert G.check_spmv(out0, ref0, m, x, np.zeros_like(y), c=c)
    # scaled: out = (A x) * (1 / sqrt(q)), sum(out^2) accumulated
    q = 7.25
    S = torch.tensor([q, 0.0, 3.0], dtype=torch.float64, device="cuda")
    o2 = torch.empty(m.rows, dtype=xt.dtype, device="cuda")
    dc.spmv_scaled(xt, o2, S[0:1], S[1:2], S[2:3])
    dc.check()
    o2 = o2.cpu().numpy()
    exp = _scaled_expect(out0, q, V)
    assert G.same_bits_or_nan(o2, exp)
    tol = 1e-12 if V == np.float64 else 1e-5
    ss = float(np.sum(o2.astype(np.float64) ** 2))
    assert abs(float(S[1]) - ss) <= tol * max(ss, 1e-300) * 10
    assert float(S[2]) == 0.0
    assert P.decode_matrix(c) == P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx, m.values.astype(V))


def test_kchunk_default_is_multislice_at_scale():
    """At 1/4 of the Laplacian benchmark size the default plan already packs
    several slices per chunk (the benchmarked configuration) and matches the
    oracle bitwise."""
    m = synth.laplacian_2d(1296)  # 1.68M rows, 52.5k slices
    x, y = synth.vectors(m)
    c = P.encode_matrix(m)
    dc = c.device(0)
    plan = dc.plan()
    assert plan["chunk_slices_max"] >= 2, plan
    out = dc.spmv(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()).cpu().numpy()
    dc.check()
    ref = O.spmv(O.parse(P.serialize(c)), x, y, threads=8)
    assert G.same_bits_or_nan(out, ref)


def test_clear_row_map_keeps_col_map():
    """dtans_set_row_map(h, NULL) after a symmetric reorder clears only the
    row map: the column gather still runs, and dtans_free frees each buffer
    once."""
    from paper_2603_01915_b200 import _native
    m = synth.rmat(12, 30000, seed=3)
    x, y = synth.vectors(m)
    pm, perm = P.sort_symmetric_by_degree(m)
    c = P.encode_matrix(pm)
    c.row_map = perm
    c.col_map = perm
    dc = c.device(0)
    _native.check(_native.lib().dtans_set_row_map(dc.handle, None))
    p64 = perm.astype(np.int64)
    out = dc.spmv(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()).cpu().numpy()
    dc.check()
    ref = O.spmv(O.parse(P.serialize(c)), x[p64], y, threads=8)
    assert G.check_spmv(out, ref, pm, x[p64], y, c=c)
    dc.close()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_fused_power_iteration_with_long_slices(dtype, monkeypatch):
    """A skewed matrix has long slices (checkpointed tasks): the fused
    power-iteration step scales and sums them in the task / finalize
    kernels, so fused == unfused within the north-star tolerance."""
    from paper_2603_01915_b200 import distributed as D
    monkeypatch.setenv("DTANS_LONG_SEG", "8")
    m = synth.rmat(12, 60000, seed=2, dtype=dtype)
    # symmetrise the pattern (positive values) so a Perron vector exists
    import scipy.sparse as sp
    A = sp.csr_matrix((np.abs(m.values.astype(np.float64)) + 1.0, m.col_idx, m.row_start), shape=(m.rows, m.cols))
    A = (A + A.T).tocsr()
    A.sort_indices()
    m = P.CsrMatrix(A.shape[0], A.shape[1], A.indptr.astype(np.int64), A.indices.astype(np.int64),
                    A.data.astype(dtype))
    c = P.encode_matrix(m)
    op = D.ShardedSpMV(c, 0, 1, device=torch.device("cuda", 0))
    assert op._dev.plan()["nlong"] > 0
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    x0 = torch.full((m.cols,), 1.0 / np.sqrt(m.cols), dtype=tdt, device="cuda")
    xf, lf = D.power_iteration(op, x0, 20, fused=True)
    xu, lu = D.power_iteration(op, x0, 20, fused=False)
    op._dev.check()
    tol = 1e-12 if dtype == np.float64 else 1e-5
    assert abs(lf - lu) <= 10 * tol * lu
    assert np.allclose(xf.cpu().numpy(), xu.cpu().numpy(), rtol=100 * tol, atol=100 * tol / np.sqrt(m.cols))


@pytest.mark.parametrize("gen", ["laplacian700", "rmat14_f32"])
def test_streamed_upload_from_mmapped_file(gen, tmp_path, monkeypatch):
    """dtans_upload streams the chunk blobs (and, with long slices, the raw
    arrays) through pinned staging buffers straight from a mmapped CDTA
    file (container.py:647-720): many small batches (DTANS_UPLOAD_KB=64)
    give the same product as the oracle, bitwise."""
    monkeypatch.setenv("DTANS_UPLOAD_KB", "64")
    m = MID[gen]()
    x, y = synth.vectors(m)
    c0 = P.encode_matrix(m)
    path = tmp_path / "m.cdta"
    P.save(c0, str(path))
    c = P.load(str(path))
    dc = c.device(0)
    plan = dc.plan()
    assert plan["upload_batches"] >= 4, plan
    out = P.spmv(c, x, y)
    ref = O.spmv(O.parse(P.serialize(c0)), x, y, threads=8)
    assert G.check_spmv(out, ref, m, x, y, c=c)
    assert P.decode_matrix(c) == P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx,
                                             m.values.astype(c.value_dtype))


@pytest.mark.parametrize("long_seg,chunk", [("4", "3"), ("8", "5"), ("0", "16")])
def test_gpu_checkpoint_walk_matches_host_walk(long_seg, chunk, monkeypatch):
    """The long-slice index built by the GPU walk (dtans_walk_kernel, the
    default) and by the host walk (DTANS_GPU_WALK=0, checkpoints.cpp) give
    bitwise identical products and decodes, warp and solo tasks included,
    and both match the oracle within the split-row tolerance."""
    monkeypatch.setenv("DTANS_LONG_SEG", long_seg)
    monkeypatch.setenv("DTANS_CHUNK", chunk)
    for gen in (lambda: synth.rmat(13, 80000, seed=9), lambda: synth.rmat(12, 50000, seed=2, dtype=np.float64),
                lambda: P.sort_rows_by_length(synth.rmat(13, 90000, seed=4))[0]):
        m = gen()
        x, y = synth.vectors(m)
        outs, decs = [], []
        for walk in ("1", "0"):
            monkeypatch.setenv("DTANS_GPU_WALK", walk)
            c = _fresh(P.encode_matrix(m))
            assert c.device(0).plan()["nlong"] > 0
            outs.append(P.spmv(c, x, y))
            decs.append(P.decode_matrix(c))
        assert G.same_bits_or_nan(outs[0], outs[1])
        assert decs[0] == decs[1] == P.CsrMatrix(m.rows, m.cols, m.row_start, m.col_idx,
                                                 m.values.astype(c.value_dtype))
        ref = O.spmv(O.parse(P.serialize(c)), x, y, threads=8)
        assert G.check_spmv(outs[0], ref, m, x, y, c=c)
