"""The CSR-dtANS container and the drop-in hot path.

Same names, argument order, defaults and return types as the reference
/root/reference/pkg/src/csrdtans/container.py:
  encode_matrix  (:126-204)  -> C++ encoder in libdtans.so (byte-identical)
  spmv           (:554-596)  -> fused sm_100a decode+SpMV kernel
  decode_matrix  (:524-531)  -> sm_100a decode kernel (bit-exact)
  serialize / deserialize / size_bytes (:599-731) -> numpy, same byte format
There is no CPU compute path: without libdtans.so or a CUDA device these
functions raise ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import struct
import weakref
import zlib
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ContainerError, NativeUnavailable, ParameterError
from .params import DtansParams, require_container_params
from .sparse import CsrMatrix
from .tables import CodingTables

MAGIC = b"CDTA"
FORMAT_VERSION = 1
SLICE_HEIGHT = 32
DEFAULT_PERMUTATION_SEED = 2654435761
DELTA_SENTINEL = 0xFFFFFFFF
VALUE_SENTINEL = {4: 0xFFFFFFFF, 8: 0xFFFFFFFFFFFFFFFF}

_HEADER = struct.Struct("<4sHBBQQQ")
_PARAMS = struct.Struct("<BBBBBBQ")
_SLOT_DTYPE = {
    8: np.dtype([("vsym", "<u8"), ("dsym", "<u4"), ("ddig", "u1"), ("dbm1", "u1"),
                 ("vdig", "u1"), ("vbm1", "u1")]),
    4: np.dtype([("vsym", "<u4"), ("dsym", "<u4"), ("ddig", "u1"), ("dbm1", "u1"),
                 ("vdig", "u1"), ("vbm1", "u1")]),
}


def _tables_from_records(rec: np.ndarray, precision: int):
    dsym = rec["dsym"].astype(np.uint64)
    vsym = rec["vsym"].astype(np.uint64)
    desc = rec["dsym"] == DELTA_SENTINEL
    vesc = rec["vsym"] == VALUE_SENTINEL[precision]
    dt = CodingTables(np.where(desc, 0, dsym).astype(np.uint64), desc, rec["ddig"].copy(),
                      rec["dbm1"].astype(np.int32) + 1)
    vt = CodingTables(np.where(vesc, 0, vsym).astype(np.uint64), vesc, rec["vdig"].copy(),
                      rec["vbm1"].astype(np.int32) + 1)
    return dt, vt


def _validate_tables(t: CodingTables) -> None:
    """CodingTables.from_slots checks (entropy.py:351-374): digit < base,
    one base per symbol, every (symbol, digit) of the full-base runs present."""
    if np.any(t.digits.astype(np.int64) >= t.bases):
        raise ContainerError("invalid coding tables: slot digit out of range for its base")
    ret = ~t.escape
    if ret.any():
        s, b, d = t.sym[ret], t.bases[ret], t.digits[ret].astype(np.int64)
        order = np.lexsort((d, s))
        s, b, d = s[order], b[order], d[order]
        starts = np.concatenate([[True], s[1:] != s[:-1]])
        grp = np.cumsum(starts) - 1
        first_base = b[starts][grp]
        if np.any(b != first_base):
            raise ContainerError("invalid coding tables: inconsistent bases")
        counts = np.bincount(grp)
        if np.any(counts != b[starts]):
            raise ContainerError("invalid coding tables: missing slot")
        pos = np.arange(len(s)) - np.flatnonzero(starts)[grp]
        if np.any(d != pos):
            raise ContainerError("invalid coding tables: missing slot")
    if t.escape.any():
        e = t.escape_base
        full = t.escape & (t.bases == e)
        have = np.zeros(e, dtype=bool)
        have[t.digits[full].astype(np.int64)] = True
        if not have.all():
            raise ContainerError("invalid coding tables: missing escape slot")


@dataclass(eq=False)
class CsrDtansContainer:
    rows: int
    cols: int
    nnz: int
    precision: int
    params: DtansParams
    permutation_seed: int
    delta_tables: CodingTables
    value_tables: CodingTables
    row_symbols: np.ndarray  # uint32 [rows]
    directory: np.ndarray    # uint64 [nslices + 1]
    stream: np.ndarray       # uint32 [words]
    table_records: np.ndarray = field(default=None, repr=False)  # K slot records
    # optional extension, not serialized: this container encodes P*A and
    # row_map[i] is the original row of encoded row i (sort_rows_by_length);
    # spmv then reads y / writes y' in the original order
    row_map: np.ndarray = field(default=None, repr=False)
    # optional extension (sort_symmetric_by_degree): this container encodes
    # P*A*P^T; the SpMV gathers x'[j] = x[col_map[j]] on the device first
    col_map: np.ndarray = field(default=None, repr=False)
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def nslices(self) -> int:
        return -(-self.rows // SLICE_HEIGHT)

    @property
    def value_dtype(self):
        return np.float64 if self.precision == 8 else np.float32

    def raw_widths(self) -> tuple:
        return (32, self.precision * 8)

    def tables_pair(self) -> tuple:
        return (self.delta_tables, self.value_tables)

    def __eq__(self, other) -> bool:
        if not isinstance(other, CsrDtansContainer):
            return NotImplemented
        return (self.rows == other.rows and self.cols == other.cols and self.nnz == other.nnz
                and self.precision == other.precision and self.params == other.params
                and self.permutation_seed == other.permutation_seed
                and self.delta_tables == other.delta_tables
                and self.value_tables == other.value_tables
                and np.array_equal(self.row_symbols, other.row_symbols)
                and np.array_equal(self.directory, other.directory)
                and np.array_equal(self.stream, other.stream))

    # -- device side -------------------------------------------------------
    def device(self, device: int = 0) -> "DeviceContainer":
        """Upload once per device (cached), like the reference's ``_cache``."""
        key = ("dev", int(device))
        h = self._cache.get(key)
        if h is None or h.closed:
            h = DeviceContainer(self, device)
            self._cache[key] = h
        return h


# ---------------------------------------------------------------------------
# Encoding


def encode_matrix(m: CsrMatrix, params: DtansParams | None = None,
                  value_width: int | None = None,
                  permutation_seed: int | None = DEFAULT_PERMUTATION_SEED,
                  *, threads: int = 0, device: int | None = None) -> CsrDtansContainer:
    """Compress ``m``; bytes identical to the reference encoder
    (container.py:126-204).  ``threads`` (keyword-only, new) sets the C++
    encoder's thread count (0 = all cores).  ``device`` (keyword-only, new):
    run the per-symbol passes on that CUDA device (dtans_encode_device: the
    distributions, the base pass and the digit pass + warp interleave; the
    same bytes); None = the host encoder."""
    if len(m.row_start) != m.rows + 1:
        raise ParameterError("row_start must have rows + 1 entries")
    params = params or DtansParams.production()
    precision = value_width if value_width is not None else m.value_width
    require_container_params(params, precision)
    if m.cols > 2**32 or m.rows > 2**32:
        raise ParameterError("indices must fit 32 bits")
    vdt = np.float64 if precision == 8 else np.float32
    values = np.ascontiguousarray(np.asarray(m.values).astype(vdt, copy=False))
    row_start = np.ascontiguousarray(m.row_start, dtype=np.int64)
    col_idx = np.ascontiguousarray(m.col_idx, dtype=np.int64)
    if len(values) != len(col_idx):
        raise ParameterError("col_idx and values must have equal length")
    if permutation_seed is None:
        perm_d = perm_v = None
    else:
        # numpy PCG64 + Generator.permutation defines the slot layout
        # (container.py:159-164): the reference's own dependency, called here.
        rng = np.random.default_rng(permutation_seed)
        perm_d = np.ascontiguousarray(rng.permutation(params.k), dtype=np.uint32)
        perm_v = np.ascontiguousarray(rng.permutation(params.k), dtype=np.uint32)
    L = _native.lib()
    nnz = len(values)
    view = _native.CsrView(m.rows, m.cols, nnz, row_start.ctypes.data,
                           col_idx.ctypes.data if nnz else None,
                           values.ctypes.data if nnz else None, precision)
    opts = _native.EncodeOpts(params.k_log2, params.m_log2,
                              perm_d.ctypes.data if perm_d is not None else None,
                              perm_v.ctypes.data if perm_v is not None else None, threads)
    enc = _native.Encoded()
    if device is None:
        _native.check(L.dtans_encode(ctypes.byref(view), ctypes.byref(opts), ctypes.byref(enc)))
    else:
        _native.check(L.dtans_encode_device(ctypes.byref(view), ctypes.byref(opts), int(device), ctypes.byref(enc)))
    try:
        rec_bytes = ctypes.string_at(enc.tables, params.k * enc.rec_size)
        rec = np.frombuffer(rec_bytes, dtype=_SLOT_DTYPE[precision]).copy()
        row_symbols = np.ctypeslib.as_array(
            ctypes.cast(enc.row_symbols, ctypes.POINTER(ctypes.c_uint32)), (max(m.rows, 1),))[: m.rows].copy()
        directory = np.ctypeslib.as_array(
            ctypes.cast(enc.directory, ctypes.POINTER(ctypes.c_uint64)), (enc.nslices + 1,)).copy()
        stream = np.ctypeslib.as_array(
            ctypes.cast(enc.stream, ctypes.POINTER(ctypes.c_uint32)), (max(enc.nwords, 1),))[: enc.nwords].copy()
    finally:
        L.dtans_encoded_free(ctypes.byref(enc))
    dt, vt = _tables_from_records(rec, precision)
    return CsrDtansContainer(
        rows=m.rows, cols=m.cols, nnz=nnz, precision=precision, params=params,
        permutation_seed=0 if permutation_seed is None else permutation_seed,
        delta_tables=dt, value_tables=vt, row_symbols=row_symbols, directory=directory,
        stream=stream, table_records=rec)


# ---------------------------------------------------------------------------
# Device handle


def _torch():
    import torch
    return torch


class DeviceContainer:
    """A container resident in HBM (``dtans_upload``), freed by ``close()``.

    ``spmv(x, y, out)`` takes torch CUDA tensors (zero copy, launched on the
    current torch stream); ``spmv_host`` takes host numpy arrays and copies
    inside the call (the end-to-end C-ABI path).
    """

    def __init__(self, c: CsrDtansContainer, device: int = 0):
        L = _native.lib()
        rec = c.table_records
        if rec is None:
            raise ParameterError("container has no table records")
        self._keep = [np.ascontiguousarray(rec).view(np.uint8),
                      np.ascontiguousarray(c.row_symbols, dtype=np.uint32),
                      np.ascontiguousarray(c.directory, dtype=np.uint64),
                      np.ascontiguousarray(c.stream, dtype=np.uint32)]
        t, rs, di, st = self._keep
        view = _native.ContainerView(
            c.rows, c.cols, c.nnz, c.nslices, len(c.stream), c.precision, t.ctypes.data,
            rs.ctypes.data if len(rs) else None, di.ctypes.data,
            st.ctypes.data if len(st) else None)
        h = ctypes.c_void_p()
        _native.check(L.dtans_upload(ctypes.byref(view), int(device), ctypes.byref(h)))
        self._keep = None
        self.handle = h
        self._fin = weakref.finalize(self, L.dtans_free, h)
        if c.row_map is not None:
            rm = np.ascontiguousarray(c.row_map, dtype=np.uint32)
            if len(rm) != c.rows:
                raise ParameterError("row_map must have one entry per row")
            _native.check(L.dtans_set_row_map(h, rm.ctypes.data))
        if c.col_map is not None:
            cm = np.ascontiguousarray(c.col_map, dtype=np.uint32)
            if len(cm) != c.cols:
                raise ParameterError("col_map must have one entry per column")
            _native.check(L.dtans_set_col_map(h, cm.ctypes.data))
        self.device = int(device)
        self.rows, self.cols, self.nnz, self.precision = c.rows, c.cols, c.nnz, c.precision
        self.row_symbols = c.row_symbols
        self.closed = False

    @property
    def dtype(self):
        return np.float64 if self.precision == 8 else np.float32

    def close(self):
        if not self.closed:
            self._fin()
            self.closed = True

    def info(self) -> dict:
        b = ctypes.c_int64()
        ctas, warps, smem = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _native.check(_native.lib().dtans_info(self.handle, ctypes.addressof(b), ctypes.addressof(ctas),
                                               ctypes.addressof(warps), ctypes.addressof(smem)))
        return {"device_bytes": b.value, "ctas": ctas.value, "warps_per_cta": warps.value,
                "smem_bytes": smem.value}

    def plan(self) -> dict:
        """The work plan of the upload (dtans_plan): chunks, long slices, ..."""
        p = _native.Plan()
        _native.check(_native.lib().dtans_plan(self.handle, ctypes.byref(p)))
        return {k: getattr(p, k) for k, _ in _native.Plan._fields_}

    def split_slices(self) -> np.ndarray:
        """Slices whose rows sum several task partials (dtans_split_slices):
        their y' matches the reference within the north-star tolerance,
        every other row bitwise."""
        lib = _native.lib()
        if not hasattr(lib, "dtans_split_slices"):  # an older A/B build
            return np.zeros(0, dtype=np.uint32)
        n = int(lib.dtans_split_slices(self.handle, None, 0))
        out = np.zeros(max(n, 1), dtype=np.uint32)
        if n:
            lib.dtans_split_slices(self.handle, out.ctypes.data, n)
        return out[:n]

    def split_rows(self, rows: int) -> np.ndarray:
        """Boolean mask of the rows in split slices."""
        m = np.zeros(-(-rows // 32) * 32, dtype=bool)
        s = self.split_slices().astype(np.int64)
        if len(s):
            m[(s[:, None] * 32 + np.arange(32)).ravel()] = True
        return m[:rows]

    def launches(self) -> int:
        return int(_native.lib().dtans_launch_count(self.handle))

    def _check_vec(self, t, n, what, dt):
        if (t.dtype != dt or t.numel() != n or not t.is_cuda or not t.is_contiguous()
                or t.device.index != self.device):
            raise ParameterError(f"{what} must be a contiguous tensor on cuda:{self.device} "
                                 f"of the container dtype with {n} elements")

    def spmv(self, x, y=None, out=None, stream=None):
        """y' = A x (+ y) on torch CUDA tensors; asynchronous."""
        torch = _torch()
        dt = torch.float64 if self.precision == 8 else torch.float32
        self._check_vec(x, self.cols, "x", dt)
        if y is not None:
            self._check_vec(y, self.rows, "y", dt)
        if out is None:
            out = torch.empty(self.rows, dtype=dt, device=x.device)
        else:
            self._check_vec(out, self.rows, "out", dt)
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        fn = _native.lib().dtans_spmv_f64 if self.precision == 8 else _native.lib().dtans_spmv_f32
        _native.check(fn(self.handle, x.data_ptr(), y.data_ptr() if y is not None else None,
                         out.data_ptr(), stream))
        return out

    def spmv_scaled(self, x, out, sumsq_in, sumsq_out, sumsq_zero=None, stream=None):
        """One fused power-iteration step on torch CUDA tensors (asynchronous):
        out = (A x) / sqrt(sumsq_in) (unscaled if sumsq_in is None),
        sumsq_out += sum(out^2), sumsq_zero = 0 (f64 device scalars)."""
        torch = _torch()
        dt = torch.float64 if self.precision == 8 else torch.float32
        self._check_vec(x, self.cols, "x", dt)
        self._check_vec(out, self.rows, "out", dt)
        for s in (sumsq_in, sumsq_out, sumsq_zero):
            if s is not None and (s.dtype != torch.float64 or s.numel() < 1 or not s.is_cuda):
                raise ParameterError("sum-of-squares scalars must be f64 CUDA tensors")
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        ptr = (lambda t: t.data_ptr() if t is not None else None)
        _native.check(_native.lib().dtans_spmv_scaled(self.handle, x.data_ptr(), out.data_ptr(), ptr(sumsq_in),
                                                      ptr(sumsq_out), ptr(sumsq_zero), stream))
        return out

    def check(self, stream=None):
        """Synchronize and raise CorruptStream if a kernel flagged the stream."""
        if stream is None:
            torch = _torch()
            stream = torch.cuda.current_stream(self.device).cuda_stream
        _native.check(_native.lib().dtans_check(self.handle, stream))

    def spmv_host(self, x: np.ndarray, y: np.ndarray | None, out: np.ndarray) -> np.ndarray:
        """Host x, y, out (ideally pinned): H2D, kernel, D2H, check."""
        dt = self.dtype
        for a, n, what in ((x, self.cols, "x"), (y, self.rows, "y"), (out, self.rows, "out")):
            if a is None and what == "y":
                continue
            if (not isinstance(a, np.ndarray) or a.dtype != dt or a.size != max(n, 1 if what == "x" else 0)
                    or not a.flags.c_contiguous or (what == "out" and not a.flags.writeable)):
                raise ParameterError(f"{what} must be a contiguous {np.dtype(dt).name} array of {n} elements")
        _native.check(_native.lib().dtans_spmv_host(
            self.handle, x.ctypes.data, y.ctypes.data if y is not None else None, out.ctypes.data))
        return out

    def decode(self):
        """-> (row_start int64, cols int64, values) decoded on the GPU."""
        torch = _torch()
        nnz_row = np.asarray(self.row_symbols, dtype=np.int64) // 2
        row_start = np.zeros(self.rows + 1, dtype=np.int64)
        np.cumsum(nnz_row, out=row_start[1:])
        nnz = int(row_start[-1])
        dev = torch.device("cuda", self.device)
        rs_t = torch.from_numpy(row_start).to(dev)
        cols_t = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        vb_t = torch.empty(max(nnz, 1), dtype=torch.int64 if self.precision == 8 else torch.int32,
                           device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _native.check(_native.lib().dtans_decode(self.handle, rs_t.data_ptr(), cols_t.data_ptr(),
                                                 vb_t.data_ptr(), stream))
        self.check(stream)
        cols = cols_t[:nnz].cpu().numpy()
        vb = vb_t[:nnz].cpu().numpy()
        vals = vb.view(np.float64) if self.precision == 8 else vb.view(np.float32)
        return row_start, cols, vals


# ---------------------------------------------------------------------------
# Decode and SpMV (the hot path)


def decode_matrix(c: CsrDtansContainer) -> CsrMatrix:
    """Reconstruct the CSR matrix (exact bit patterns) on the GPU
    (container.py:524-531)."""
    row_start, cols, vals = c.device(0).decode()
    if row_start[-1] != c.nnz:
        from .errors import CorruptStream
        raise CorruptStream("row symbol counts disagree with the header nnz")
    return CsrMatrix(c.rows, c.cols, row_start, cols, vals)


def spmv(c: CsrDtansContainer, x: np.ndarray, y: np.ndarray, threads: int = 1,
         *, device: int = 0) -> np.ndarray:
    """y' = A x + y, decoding the container on the fly on the GPU.

    Same contract as the reference (container.py:554-596): x and y are cast
    to the container precision, a new array is returned, y is not mutated.
    ``threads`` is accepted for compatibility and ignored.  Per row the
    products are accumulated left to right in the container precision, so
    the result is bitwise equal to the reference's.
    """
    x = np.asarray(x)
    y = np.asarray(y)
    if len(x) != c.cols or len(y) != c.rows:
        raise ParameterError("dimension mismatch")
    dtype = c.value_dtype
    x = np.ascontiguousarray(x.astype(dtype, copy=False))
    y = np.ascontiguousarray(y.astype(dtype, copy=False))
    if c.rows == 0:
        return np.empty(0, dtype=dtype)
    if c.cols == 0:
        x = np.zeros(1, dtype=dtype)
    dev = c.device(device)
    return dev.spmv_host(x, y, _pinned_empty(c.rows, dtype))


def _pinned_empty(n: int, dtype) -> np.ndarray:
    """A new array in page-locked memory from torch's caching host
    allocator: the D2H lands in it directly, and an array the caller has
    dropped is reused (already faulted in) by the next call, instead of a
    fresh np.empty whose first touch costs page faults (DESIGN 5)."""
    torch = _torch()
    tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
    return torch.empty(n, dtype=tdt, pin_memory=True).numpy()


# ---------------------------------------------------------------------------
# Serialization (container.py:599-731)


def _records(c: CsrDtansContainer) -> np.ndarray:
    if c.table_records is not None:
        return c.table_records
    rec = np.zeros(c.params.k, dtype=_SLOT_DTYPE[c.precision])
    d, v = c.delta_tables, c.value_tables
    rec["dsym"] = np.where(d.escape, DELTA_SENTINEL, d.sym).astype(np.uint32)
    rec["vsym"] = np.where(v.escape, VALUE_SENTINEL[c.precision], v.sym)
    rec["ddig"], rec["dbm1"] = d.digits, d.bases - 1
    rec["vdig"], rec["vbm1"] = v.digits, v.bases - 1
    return rec


def serialize(c: CsrDtansContainer) -> bytes:
    p = c.params
    parts = [
        _HEADER.pack(MAGIC, FORMAT_VERSION, c.precision, 0, c.rows, c.cols, c.nnz),
        _PARAMS.pack(p.w_log2, p.k_log2, p.m_log2, p.l, p.o, p.f, c.permutation_seed),
        _records(c).tobytes(),
        np.asarray(c.row_symbols).astype("<u4").tobytes(),
        np.asarray(c.directory).astype("<u8").tobytes(),
        struct.pack("<Q", len(c.stream)),
        np.asarray(c.stream).astype("<u4").tobytes(),
    ]
    body = b"".join(parts)
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def deserialize(data: bytes) -> CsrDtansContainer:
    """Parse CDTA v1 bytes (container.py:666-720).  Accepts any buffer
    (bytes, bytearray, memoryview, mmap); the arrays are zero-copy views of
    it, so a memory-mapped file is never copied on the host."""
    data = memoryview(data).cast("B")
    if len(data) < _HEADER.size + _PARAMS.size + 4:
        raise ContainerError("container truncated")
    body, crc_bytes = data[:-4], data[-4:]
    if struct.unpack("<I", crc_bytes)[0] != (zlib.crc32(body) & 0xFFFFFFFF):
        raise ContainerError("checksum mismatch")
    magic, version, precision, _, rows, cols, nnz = _HEADER.unpack_from(body, 0)
    if magic != MAGIC:
        raise ContainerError(f"bad magic {magic!r}")
    if version != FORMAT_VERSION:
        raise ContainerError(f"unsupported version {version}")
    if precision not in (4, 8):
        raise ContainerError(f"bad precision {precision}")
    off = _HEADER.size
    wl, kl, ml, l, o, f, seed = _PARAMS.unpack_from(body, off)
    off += _PARAMS.size
    try:
        params = DtansParams(w=2**wl, k=2**kl, m=2**ml, l=l, o=o, f=f)
        params.validate()
    except (ParameterError, OverflowError) as e:
        raise ContainerError(f"invalid parameters: {e}") from e

    def take(nbytes, what):
        nonlocal off
        if off + nbytes > len(body):
            raise ContainerError(f"container truncated in {what}")
        chunk = body[off: off + nbytes]
        off += nbytes
        return chunk

    rec = np.frombuffer(take(params.k * _SLOT_DTYPE[precision].itemsize, "tables"),
                        dtype=_SLOT_DTYPE[precision]).copy()
    dt, vt = _tables_from_records(rec, precision)
    _validate_tables(dt)
    _validate_tables(vt)
    row_symbols = np.frombuffer(take(4 * rows, "row counts"), dtype="<u4")
    nslices = -(-rows // SLICE_HEIGHT)
    directory = np.frombuffer(take(8 * (nslices + 1), "directory"), dtype="<u8")
    (nwords,) = struct.unpack("<Q", take(8, "stream length"))
    stream = np.frombuffer(take(4 * nwords, "stream"), dtype="<u4")
    if off != len(body):
        raise ContainerError("trailing bytes after stream")
    if np.any(np.diff(directory.astype(np.int64)) < 0) or (len(directory) and directory[-1] != nwords):
        raise ContainerError("directory does not span the stream")
    return CsrDtansContainer(
        rows=rows, cols=cols, nnz=nnz, precision=precision, params=params,
        permutation_seed=seed, delta_tables=dt, value_tables=vt,
        row_symbols=row_symbols.astype(np.uint32, copy=False), directory=directory.astype(np.uint64, copy=False),
        stream=stream.astype(np.uint32, copy=False), table_records=rec)


def save(c: CsrDtansContainer, path) -> int:
    """Write the CDTA v1 bytes of ``c`` to ``path`` (streamed, running CRC;
    byte-identical to ``serialize``).  Returns the number of bytes."""
    p = c.params
    parts = [
        _HEADER.pack(MAGIC, FORMAT_VERSION, c.precision, 0, c.rows, c.cols, c.nnz),
        _PARAMS.pack(p.w_log2, p.k_log2, p.m_log2, p.l, p.o, p.f, c.permutation_seed),
        memoryview(np.ascontiguousarray(_records(c))).cast("B"),
        memoryview(np.ascontiguousarray(c.row_symbols, dtype="<u4")).cast("B"),
        memoryview(np.ascontiguousarray(c.directory, dtype="<u8")).cast("B"),
        struct.pack("<Q", len(c.stream)),
        memoryview(np.ascontiguousarray(c.stream, dtype="<u4")).cast("B"),
    ]
    crc, n = 0, 0
    with open(path, "wb") as f:
        for part in parts:
            crc = zlib.crc32(part, crc)
            f.write(part)
            n += len(part)
        f.write(struct.pack("<I", crc & 0xFFFFFFFF))
    return n + 4


def load(path) -> CsrDtansContainer:
    """Memory-map a CDTA file and parse it without copying (the arrays view
    the mapping); upload with ``.device()`` streams it to HBM."""
    import mmap
    with open(path, "rb") as f:
        mm = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ)
    return deserialize(mm)


def size_bytes(c: CsrDtansContainer) -> int:
    """tables + row counts + directory + stream (container.py:723-731)."""
    return (c.params.k * _SLOT_DTYPE[c.precision].itemsize + 4 * c.rows
            + 8 * (c.nslices + 1) + 4 * len(c.stream))


def compression_ratio(m: CsrMatrix, c: CsrDtansContainer) -> float:
    """min(CSR, COO, SELL) bytes / size_bytes (PAPER.md:508 metric)."""
    from .sparse import format_size_bytes
    base = min(format_size_bytes(m, f, c.precision) for f in ("csr", "coo", "sell"))
    return base / size_bytes(c)


__all__ = [
    "CsrDtansContainer", "DeviceContainer", "encode_matrix", "decode_matrix", "spmv",
    "serialize", "deserialize", "size_bytes", "compression_ratio", "NativeUnavailable",
]
