"""All-empty slices of plans with long slices (api.cu planner ->
kernels.cuh dtans_empty_kernel): a rows-sorted skewed matrix ends in slices
whose 32 rows have no symbols; their y' = +0.0 + y (container.py:534-551 for
an empty row) is written outside the main kernel's chunks.  Checked bitwise
against the oracle and against the same plan with DTANS_EMPTY=0 (the empty
slices staged through the main kernel), including -0.0, NaN and inf in y,
the y-less product, and the fused power-iteration step."""

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


def _fresh(c):
    for k in [k for k in c._cache if isinstance(k, tuple) and k[0] == "dev"]:
        c._cache.pop(k).close()
    return c


def _sorted_rmat(dtype):
    m = synth.rmat(15, 120000, seed=21, dtype=dtype)
    pm, perm = P.sort_rows_by_length(m)
    c = P.encode_matrix(pm)
    c.row_map = perm
    return m, pm, perm, c


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_empty_slices_sorted_rmat(dtype, monkeypatch):
    monkeypatch.setenv("DTANS_LONG_SEG", "4")
    m, pm, perm, c = _sorted_rmat(dtype)
    p64 = perm.astype(np.int64)
    x, y = synth.vectors(m)
    # special y values on rows that are empty (sorted last): +0.0 + (-0.0) = +0.0
    empty_rows = np.flatnonzero(np.diff(np.asarray(m.row_start)) == 0)
    assert len(empty_rows) > 64 * 32
    y[empty_rows[:7]] = np.array([-0.0, 0.0, np.nan, np.inf, -np.inf, -1.5, 2.0 ** -140], dtype=dtype)
    out = P.spmv(c, x, y)
    plan = c.device(0).plan()
    assert plan["nempty"] > 0 and plan["nlong"] > 0
    ref_p = O.spmv(O.parse(P.serialize(c)), x, y[p64], threads=8)
    assert G.check_spmv(out[p64], ref_p, pm, x, y[p64], c=c)
    assert G.same_bits_or_nan(out[empty_rows], np.asarray(0.0, dtype=dtype) + y[empty_rows])
    # the same plan with the empty slices staged through the main kernel
    monkeypatch.setenv("DTANS_EMPTY", "0")
    _fresh(c)
    out0 = P.spmv(c, x, y)
    assert c.device(0).plan()["nempty"] == 0
    assert G.same_bits_or_nan(out, out0)
    # y-less product through the device-tensor path
    monkeypatch.delenv("DTANS_EMPTY")
    _fresh(c)
    dev = c.device(0)
    o = dev.spmv(torch.from_numpy(x).cuda(), None)
    dev.check()
    ref0 = O.spmv(O.parse(P.serialize(c)), x, np.zeros(m.rows, dtype=dtype), threads=8)
    assert G.check_spmv(o.cpu().numpy()[p64], ref0, pm, x, np.zeros(m.rows, dtype=dtype), c=c)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_empty_slices_fused_power_iteration(dtype, monkeypatch):
    """Zero rows spanning whole slices in a matrix with long slices: the
    fused power-iteration step (scale + sum of squares) still equals the
    unfused loop, and the plan used the empty-slice kernel."""
    from paper_2603_01915_b200 import distributed as D
    import scipy.sparse as sp
    monkeypatch.setenv("DTANS_LONG_SEG", "8")
    m = synth.rmat(12, 60000, seed=3, dtype=dtype)
    A = sp.csr_matrix((np.abs(m.values.astype(np.float64)) + 1.0, m.col_idx, m.row_start), shape=(m.rows, m.cols))
    A = (A + A.T).tolil()
    A[1024:1024 + 640, :] = 0  # 20 all-empty slices
    A = A.tocsr()
    A.eliminate_zeros()
    A.sort_indices()
    m = P.CsrMatrix(A.shape[0], A.shape[1], A.indptr.astype(np.int64), A.indices.astype(np.int64),
                    A.data.astype(dtype))
    c = P.encode_matrix(m)
    op = D.ShardedSpMV(c, 0, 1, device=torch.device("cuda", 0))
    plan = op._dev.plan()
    assert plan["nlong"] > 0 and plan["nempty"] >= 20
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    x0 = torch.full((m.cols,), 1.0 / np.sqrt(m.cols), dtype=tdt, device="cuda")
    xf, lf = D.power_iteration(op, x0, 20, fused=True)
    xu, lu = D.power_iteration(op, x0, 20, fused=False)
    op._dev.check()
    tol = 1e-12 if dtype == np.float64 else 1e-5
    assert abs(lf - lu) <= 10 * tol * lu
    xf, xu = xf.cpu().numpy(), xu.cpu().numpy()
    assert np.allclose(xf, xu, rtol=100 * tol, atol=100 * tol / np.sqrt(m.cols))
    assert np.all(xf[1024:1024 + 640] == 0) and not np.signbit(xf[1024:1024 + 640]).any()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_launch_chain_variants_identical(dtype, monkeypatch):
    """The long-slice launch chain (api.cu launch: PDL between the solo,
    task and finalize kernels, solo first with task tickets, the empty-slice
    kernel, 48-segment tasks for sorted rows) changes only the schedule:
    every variant gives the same bits, the decode stays bit-exact, and the
    result matches the oracle under the parity policy."""
    m, pm, perm, c = _sorted_rmat(dtype)
    p64 = perm.astype(np.int64)
    x, y = synth.vectors(m)
    outs = {}
    for env in ({}, {"DTANS_PDL": "0"}, {"DTANS_SOLO_FIRST": "0"}, {"DTANS_EMPTY": "0"},
                {"DTANS_PDL": "1"}, {"DTANS_PDL_MAIN": "0"}):
        for k in ("DTANS_PDL", "DTANS_SOLO_FIRST", "DTANS_EMPTY", "DTANS_PDL_MAIN"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        _fresh(c)
        outs[tuple(env.items())] = P.spmv(c, x, y)
        plan = c.device(0).plan()
        assert plan["nlong"] > 0 and plan["ntasks"] > 0
        assert (plan["nempty"] > 0) == (env.get("DTANS_EMPTY") != "0")
        assert P.decode_matrix(c) == pm
    base = outs[()]
    for k, o in outs.items():
        assert G.same_bits_or_nan(o, base), k
    ref_p = O.spmv(O.parse(P.serialize(c)), x, y[p64], threads=8)
    assert G.check_spmv(base[p64], ref_p, pm, x, y[p64], c=c)


def test_back_to_back_products_on_one_stream():
    """Consecutive products on one stream overlap through PDL (the main
    kernel's table copy runs in the previous product's tail): a chain of
    dependent products (y_{k+1} = A x + y_k) must equal the same chain run
    with a synchronize between products."""
    m = synth.laplacian_2d(300)
    c = P.encode_matrix(m)
    x, y = synth.vectors(m)
    dev = c.device(0)
    xt = torch.from_numpy(x).cuda()
    ys = [torch.from_numpy(y).cuda()]
    for _ in range(6):
        ys.append(dev.spmv(xt, ys[-1]))
    got = ys[-1].cpu().numpy()
    yy = torch.from_numpy(y).cuda()
    for _ in range(6):
        yy = dev.spmv(xt, yy)
        torch.cuda.synchronize()
    dev.check()
    assert G.same_bits_or_nan(got, yy.cpu().numpy())
    ref = y.copy()
    oc = O.parse(P.serialize(c))
    for _ in range(6):
        ref = O.spmv(oc, x, ref, threads=8)
    assert G.same_bits_or_nan(got, ref)


def test_device_path_rejects_bad_vectors():
    """DeviceContainer.spmv validates x, y and out (dtype, length, device,
    contiguity) before any launch: a short `out` would otherwise be written
    past its end (round-1 advice)."""
    m = synth.laplacian_2d(40)
    c = P.encode_matrix(m)
    dev = c.device(0)
    x = torch.zeros(m.cols, dtype=torch.float64, device="cuda")
    y = torch.zeros(m.rows, dtype=torch.float64, device="cuda")
    bad = [
        dict(x=x, y=y, out=torch.empty(m.rows - 1, dtype=torch.float64, device="cuda")),
        dict(x=x, y=y, out=torch.empty(m.rows, dtype=torch.float32, device="cuda")),
        dict(x=x, y=y, out=torch.empty(m.rows, dtype=torch.float64)),
        dict(x=torch.zeros(2 * m.cols, dtype=torch.float64, device="cuda")[::2], y=y, out=None),
        dict(x=x, y=torch.zeros(m.rows + 1, dtype=torch.float64, device="cuda"), out=None),
    ]
    for kw in bad:
        with pytest.raises(P.ParameterError):
            dev.spmv(kw["x"], kw["y"], kw["out"])
    o = dev.spmv(x, y)
    dev.check()
    assert o.shape == (m.rows,)
