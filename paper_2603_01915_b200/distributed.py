"""Row sharding across GPUs and the iterated SpMV (power iteration).

The data-parallel unit is the 32-row slice: a contiguous slice range of a
container, with its directory rebased and the same coding tables, is itself
a valid container whose decode equals the corresponding rows of the whole
(the reference's decode walks slices independently, container.py:370-521,
each from directory[s], :174,190).  So a matrix is row-partitioned into
nnz-balanced slice ranges, one per rank, and each GPU decodes only its shard.

* single SpMV: no collective at all (y stays sharded);
* power iteration (BASELINE configs[4]): per iteration, local y = A_r x,
  all-reduce of sum(y^2) (one double), scale, then an all-gather of the
  y shards into the next x.  torch.distributed (NCCL over NVLink/NVSwitch)
  carries the collectives; shards are padded to a common length so
  all_gather_into_tensor moves them in one call, followed by a compaction.

CPU tests exercise this logic with the gloo backend and an injected SpMV
(the oracle); the product path always calls the CUDA kernel.
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np

from .container import SLICE_HEIGHT, CsrDtansContainer
from .errors import ParameterError


def shard_bounds(c: CsrDtansContainer, nshards: int, balance: str = "nnz") -> np.ndarray:
    """Slice boundaries [0 = b_0 <= b_1 <= ... <= b_n = nslices] splitting the
    container into ``nshards`` contiguous slice ranges with balanced nnz
    (``balance="nnz"``, the north star's rule) or balanced stream words
    (``"words"``, the decode-time driver)."""
    if nshards < 1:
        raise ParameterError("nshards must be >= 1")
    ns = c.nslices
    if balance == "nnz":
        rs = np.zeros(ns * SLICE_HEIGHT, dtype=np.int64)
        rs[: c.rows] = np.asarray(c.row_symbols, dtype=np.int64) // 2
        per = rs.reshape(ns, SLICE_HEIGHT).sum(axis=1) if ns else np.zeros(0, np.int64)
        cum = np.concatenate([[0], np.cumsum(per)])
    elif balance == "words":
        cum = np.asarray(c.directory, dtype=np.int64)
    else:
        raise ParameterError(f"unknown balance {balance!r}")
    total = cum[-1] if len(cum) else 0
    b = np.zeros(nshards + 1, dtype=np.int64)
    for r in range(1, nshards):
        b[r] = int(np.searchsorted(cum, total * r / nshards, side="left"))
    b[nshards] = ns
    b = np.maximum.accumulate(np.clip(b, 0, ns))
    return b


def shard(c: CsrDtansContainer, s_lo: int, s_hi: int) -> CsrDtansContainer:
    """Sub-container of slices [s_lo, s_hi): rows [32 s_lo, min(32 s_hi, rows)),
    same tables and parameters, directory rebased to start at 0."""
    if not (0 <= s_lo <= s_hi <= c.nslices):
        raise ParameterError("bad slice range")
    if c.row_map is not None:
        raise ParameterError("sharding a row-reordered container is not supported")
    r0 = s_lo * SLICE_HEIGHT
    r1 = min(s_hi * SLICE_HEIGHT, c.rows)
    r1 = max(r0, r1)
    d = np.asarray(c.directory, dtype=np.uint64)
    w0, w1 = int(d[s_lo]), int(d[s_hi])
    rs = np.asarray(c.row_symbols[r0:r1], dtype=np.uint32).copy()
    return replace(
        c, rows=r1 - r0, nnz=int(rs.astype(np.int64).sum() // 2), row_symbols=rs,
        directory=(d[s_lo: s_hi + 1] - np.uint64(w0)).astype(np.uint64),
        stream=np.asarray(c.stream[w0:w1], dtype=np.uint32).copy(), _cache={})


def shard_rows(c: CsrDtansContainer, bounds: np.ndarray):
    """Row ranges [(r0, r1)] of the shards given slice bounds."""
    return [(int(bounds[i]) * SLICE_HEIGHT, min(int(bounds[i + 1]) * SLICE_HEIGHT, c.rows))
            for i in range(len(bounds) - 1)]


class ShardedSpMV:
    """One rank's view: its shard on its GPU plus the row layout of all shards.

    ``spmv_fn(x, y_or_None, out)`` computes the local product; by default the
    CUDA kernel of the shard (``DeviceContainer.spmv``)."""

    def __init__(self, c: CsrDtansContainer, rank: int, world: int, device=None, spmv_fn=None,
                 balance: str = "nnz", bounds=None):
        self.bounds = shard_bounds(c, world, balance) if bounds is None else np.asarray(bounds)
        self.rows_of = shard_rows(c, self.bounds)
        self.rank, self.world = rank, world
        self.cols = c.cols
        self.global_rows = c.rows
        self.local = shard(c, int(self.bounds[rank]), int(self.bounds[rank + 1]))
        self.max_rows = max(r1 - r0 for r0, r1 in self.rows_of) if self.rows_of else 0
        self.device = device
        self._dev = None
        if spmv_fn is None:
            dev = self.local.device(device.index if hasattr(device, "index") and device.index is not None else 0)
            self._dev = dev

            def spmv_fn(x, y, out):
                return dev.spmv(x, y, out)
        self.spmv_fn = spmv_fn

    @classmethod
    def from_local(cls, local: CsrDtansContainer, rows_of, rank: int, world: int, device=None,
                   spmv_fn=None):
        """A rank that encoded only its own row block (``local``), given the
        global row layout ``rows_of`` = [(r0, r1)] of all ranks."""
        self = cls.__new__(cls)
        self.rows_of = [(int(a), int(b)) for a, b in rows_of]
        self.bounds = None
        self.rank, self.world = rank, world
        self.cols = local.cols
        self.global_rows = self.rows_of[-1][1]
        self.local = local
        self.max_rows = max(r1 - r0 for r0, r1 in self.rows_of)
        self.device = device
        self._dev = None
        if spmv_fn is None:
            dev = local.device(device.index if device is not None and device.index is not None else 0)
            self._dev = dev

            def spmv_fn(x, y, out):
                return dev.spmv(x, y, out)
        self.spmv_fn = spmv_fn
        return self

    def spmv(self, x, y=None, out=None):
        """Local rows of A x (+ y)."""
        import torch
        if out is None:
            out = torch.empty(self.local.rows, dtype=x.dtype, device=x.device)
        if self.local.rows == 0:
            return out
        return self.spmv_fn(x, y, out)


def power_iteration(op: ShardedSpMV, x0, iters: int, group=None, return_history: bool = False,
                    fused: bool | None = None):
    """x <- A x / ||A x||_2 for ``iters`` iterations over all ranks.

    x0: full-length vector on this rank's device (every rank holds the same
    x).  Returns (x, lambda) where lambda = ||A x_{k-1}|| at the last step
    (the dominant eigenvalue estimate for a Perron matrix).

    With the CUDA kernel (``fused`` default), one iteration is ONE kernel:
    the scaled SpMV computes y_k = (A y_{k-1}) / ||y_{k-1}|| and accumulates
    ||y_k||^2 into a device scalar in its epilogue (dtans_spmv_scaled), so the
    separate dot / copy / divide passes over y disappear; N>1 adds the NCCL
    all-reduce of that scalar and the all-gather of y.  x_k = y_{k-1}/||y_{k-1}||
    is materialised only once, at the end."""
    import torch
    import torch.distributed as dist
    world = op.world
    if len(x0) != op.cols or op.cols != op.global_rows:
        raise ParameterError("power iteration needs a square matrix and a full-length x0")
    if fused is None:
        fused = op._dev is not None and not return_history
        if world > 1:
            # every rank must take the same path (the two exchange different
            # quantities); a rank with an injected spmv_fn cannot fuse
            flag = torch.tensor([1 if fused else 0], dtype=torch.int32,
                                device=x0.device if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            fused = bool(flag.item())
    if fused:
        return _power_iteration_fused(op, x0, iters, group)
    x = x0.clone()
    dtype, device = x.dtype, x.device
    pad = torch.zeros(op.max_rows, dtype=dtype, device=device)
    gathered = torch.empty(world * op.max_rows, dtype=dtype, device=device)
    # compaction index from the padded gather layout to the row order
    idx = torch.cat([torch.arange(r * op.max_rows, r * op.max_rows + (r1 - r0), device=device)
                     for r, (r0, r1) in enumerate(op.rows_of)]) if world > 1 else None
    sq = torch.zeros(1, dtype=torch.float64, device=device)
    hist = []
    lam = float("nan")
    for _ in range(iters):
        y = pad[: op.local.rows]
        op.spmv(x, None, y)
        sq[0] = torch.dot(y.to(torch.float64), y.to(torch.float64))
        if world > 1:
            dist.all_reduce(sq, group=group)
        norm = torch.sqrt(sq)
        lam = norm
        if world > 1:
            dist.all_gather_into_tensor(gathered, pad, group=group)
            x = torch.index_select(gathered, 0, idx)
        else:
            x = y.clone()
        x.div_(norm.to(dtype))
        if return_history:
            hist.append(float(norm.item()))
    lam = float(lam.item()) if torch.is_tensor(lam) else lam
    return (x, lam, hist) if return_history else (x, lam)


def _power_iteration_fused(op: ShardedSpMV, x0, iters: int, group=None):
    import torch
    import torch.distributed as dist
    world = op.world
    dtype, device = x0.dtype, x0.device
    # three rotating f64 scalars: step k reads S[k-1] (its scale), adds into
    # S[k] and zeroes S[k+1]
    S = torch.zeros(3, dtype=torch.float64, device=device)
    ybuf = [torch.empty(op.max_rows, dtype=dtype, device=device) for _ in range(2)]
    if world > 1:
        gathered = torch.empty(world * op.max_rows, dtype=dtype, device=device)
        idx = torch.cat([torch.arange(r * op.max_rows, r * op.max_rows + (r1 - r0), device=device)
                         for r, (r0, r1) in enumerate(op.rows_of)])
    x = x0
    rows = op.local.rows
    k_last = -1
    for k in range(iters):
        y = ybuf[k & 1]
        s_in = S[(k - 1) % 3: (k - 1) % 3 + 1] if k > 0 else None
        if rows:
            op._dev.spmv_scaled(x, y[:rows], s_in, S[k % 3: k % 3 + 1], S[(k + 1) % 3: (k + 1) % 3 + 1])
        else:  # an empty shard adds nothing but still zeroes the next accumulator
            S[(k + 1) % 3].zero_()
        if world > 1:
            dist.all_reduce(S[k % 3: k % 3 + 1], group=group)
            dist.all_gather_into_tensor(gathered, y, group=group)
            x = torch.index_select(gathered, 0, idx)
        else:
            x = y[:rows]
        k_last = k
    if k_last < 0:
        return x0.clone(), float("nan")
    norm = torch.sqrt(S[k_last % 3])
    x = (x / norm.to(dtype)).contiguous()
    return x, float(norm.item())


class NcclComm:
    """An NCCL communicator owned by libdtans (``dtans_mg_init``): one per
    process / GPU.  ``unique_id`` comes from ``NcclComm.unique_id()`` on rank
    0 and is shared with the other ranks by any means (``from_torch`` uses a
    torch.distributed broadcast)."""

    def __init__(self, nranks: int, rank: int, device: int, unique_id: bytes):
        import ctypes
        from . import _native
        if len(unique_id) != 128:
            raise ParameterError("an NCCL unique id has 128 bytes")
        self._L = _native.lib()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        h = ctypes.c_void_p()
        _native.check(self._L.dtans_mg_init(ctypes.addressof(buf), nranks, rank, device, ctypes.byref(h)))
        self.handle, self.nranks, self.rank, self.device = h, nranks, rank, device

    @staticmethod
    def unique_id() -> bytes:
        import ctypes
        from . import _native
        buf = (ctypes.c_uint8 * 128)()
        _native.check(_native.lib().dtans_mg_unique_id(ctypes.addressof(buf)))
        return bytes(buf)

    @classmethod
    def from_torch(cls, device: int, group=None) -> "NcclComm":
        """Rank 0 makes the id; torch.distributed broadcasts it."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(world, rank, device, obj[0])

    def power_iteration(self, dev, row_off, x0, iters: int, stream=None):
        """dtans_mg_power_iteration: ``dev`` is this rank's DeviceContainer
        (rows [row_off[rank], row_off[rank+1]) of a square matrix), ``x0`` a
        full-length CUDA tensor in the container precision, the same on every
        rank.  Returns (x_iters, lambda) like ``power_iteration``."""
        import ctypes
        import torch
        from . import _native
        ro = np.ascontiguousarray(row_off, dtype=np.int64)
        if len(ro) != self.nranks + 1:
            raise ParameterError("row_off needs nranks + 1 entries")
        want = torch.float64 if dev.precision == 8 else torch.float32
        if x0.dtype != want or not x0.is_cuda or x0.numel() != int(ro[-1]):
            raise ParameterError("x0 must be a full-length CUDA tensor in the container precision")
        x = x0.detach().clone().contiguous()
        lam = ctypes.c_double(float("nan"))
        st = torch.cuda.current_stream(x.device).cuda_stream if stream is None else stream
        _native.check(self._L.dtans_mg_power_iteration(self.handle, dev.handle, ro.ctypes.data, x.data_ptr(),
                                                       int(iters), ctypes.byref(lam), st))
        return x, lam.value

    def close(self):
        if getattr(self, "handle", None):
            self._L.dtans_mg_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def reference_power_iteration(A_csr, x0: np.ndarray, iters: int):
    """Plain numpy power iteration on a CSR matrix (test checker)."""
    import scipy.sparse as sp
    A = sp.csr_matrix((A_csr.values, A_csr.col_idx, A_csr.row_start), shape=(A_csr.rows, A_csr.cols))
    x = x0.astype(np.float64).copy()
    lam = math.nan
    for _ in range(iters):
        y = A @ x
        lam = float(np.sqrt(np.dot(y, y)))
        x = y / lam
    return x, lam
