"""ctypes binding of libdtans.so (include/dtans.h).

This is the binding a maintainer of the reference would add:
plain pointers and sizes, status codes mapped onto the reference's exception
classes.  There is no fallback: if the library is missing the product path
raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import CodingError, CorruptStream, NativeUnavailable, ParameterError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DTANS_LIB") or os.path.join(HERE, "libdtans.so")  # DTANS_LIB: experiment builds

DTANS_OK, DTANS_E_PARAM, DTANS_E_CODING, DTANS_E_CORRUPT = 0, 1, 2, 3
DTANS_E_CUDA, DTANS_E_NOMEM, DTANS_E_NODEVICE = 4, 5, 6

# Every symbol include/dtans.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "dtans_last_error", "dtans_abi_version", "dtans_encode", "dtans_encoded_free",
    "dtans_quantize", "dtans_upload", "dtans_free", "dtans_info", "dtans_spmv_f64",
    "dtans_spmv_f32", "dtans_spmv_host", "dtans_decode", "dtans_check",
    "dtans_launch_count", "dtans_set_row_map", "dtans_spmv_scaled", "dtans_set_col_map",
    "dtans_encode_device", "dtans_mg_unique_id", "dtans_mg_init", "dtans_mg_free", "dtans_mg_power_iteration",
    "dtans_plan", "dtans_split_slices",
)


class CsrView(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
        ("row_start", ctypes.c_void_p), ("col_idx", ctypes.c_void_p),
        ("values", ctypes.c_void_p), ("precision", ctypes.c_int32),
    ]


class EncodeOpts(ctypes.Structure):
    _fields_ = [
        ("k_log2", ctypes.c_int32), ("m_log2", ctypes.c_int32),
        ("perm_delta", ctypes.c_void_p), ("perm_value", ctypes.c_void_p),
        ("threads", ctypes.c_int32),
    ]


class Encoded(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
        ("nslices", ctypes.c_int64), ("nwords", ctypes.c_int64),
        ("precision", ctypes.c_int32), ("rec_size", ctypes.c_int32),
        ("tables", ctypes.c_void_p), ("row_symbols", ctypes.c_void_p),
        ("directory", ctypes.c_void_p), ("stream", ctypes.c_void_p),
    ]


class ContainerView(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
        ("nslices", ctypes.c_int64), ("nwords", ctypes.c_int64),
        ("precision", ctypes.c_int32),
        ("tables", ctypes.c_void_p), ("row_symbols", ctypes.c_void_p),
        ("directory", ctypes.c_void_p), ("stream", ctypes.c_void_p),
    ]


class Plan(ctypes.Structure):
    _fields_ = [
        ("nchunks", ctypes.c_int64), ("chunk_slices_max", ctypes.c_int64),
        ("staged_slices", ctypes.c_int64), ("nlong", ctypes.c_int64),
        ("ntasks", ctypes.c_int64), ("nsolo", ctypes.c_int64),
        ("dynamic", ctypes.c_int32), ("dinline", ctypes.c_int32),
        ("bufb", ctypes.c_int32), ("nring", ctypes.c_int32),
        ("upload_bytes", ctypes.c_int64), ("upload_batches", ctypes.c_int64),
        ("pend", ctypes.c_int64), ("nempty", ctypes.c_int64),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (make -C paper_2603_01915_b200/csrc); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.dtans_last_error.restype = ctypes.c_char_p
    L.dtans_abi_version.restype = ctypes.c_int
    L.dtans_encode.argtypes = [ctypes.POINTER(CsrView), ctypes.POINTER(EncodeOpts), ctypes.POINTER(Encoded)]
    L.dtans_encode_device.argtypes = [ctypes.POINTER(CsrView), ctypes.POINTER(EncodeOpts), ctypes.c_int,
                                      ctypes.POINTER(Encoded)]
    L.dtans_mg_unique_id.argtypes = [vp]
    L.dtans_mg_init.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.dtans_mg_free.argtypes = [vp]
    L.dtans_mg_free.restype = None
    L.dtans_mg_power_iteration.argtypes = [vp, vp, vp, vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double), vp]
    L.dtans_encoded_free.argtypes = [ctypes.POINTER(Encoded)]
    L.dtans_encoded_free.restype = None
    L.dtans_quantize.argtypes = [i64, vp, vp, i32, i32, i32, i64, vp, vp, vp, vp]
    L.dtans_upload.argtypes = [ctypes.POINTER(ContainerView), ctypes.c_int, ctypes.POINTER(vp)]
    L.dtans_free.argtypes = [vp]
    L.dtans_free.restype = None
    L.dtans_info.argtypes = [vp, vp, vp, vp, vp]
    L.dtans_spmv_f64.argtypes = [vp, vp, vp, vp, vp]
    L.dtans_spmv_f32.argtypes = [vp, vp, vp, vp, vp]
    L.dtans_spmv_host.argtypes = [vp, vp, vp, vp]
    L.dtans_spmv_scaled.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.dtans_decode.argtypes = [vp, vp, vp, vp, vp]
    L.dtans_check.argtypes = [vp, vp]
    L.dtans_set_row_map.argtypes = [vp, vp]
    L.dtans_set_col_map.argtypes = [vp, vp]
    L.dtans_launch_count.argtypes = [vp]
    L.dtans_launch_count.restype = i64
    L.dtans_plan.argtypes = [vp, ctypes.POINTER(Plan)]
    if hasattr(L, "dtans_split_slices"):  # absent from older builds loaded via DTANS_LIB (A/B runs)
        L.dtans_split_slices.restype = ctypes.c_int64
        L.dtans_split_slices.argtypes = [vp, vp, ctypes.c_int64]
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == DTANS_OK:
        return
    msg = lib().dtans_last_error().decode(errors="replace")
    if rc == DTANS_E_PARAM:
        raise ParameterError(msg)
    if rc == DTANS_E_CODING:
        raise CodingError(msg)
    if rc == DTANS_E_CORRUPT:
        raise CorruptStream(msg)
    if rc == DTANS_E_NODEVICE:
        raise NativeUnavailable(msg)
    if rc == DTANS_E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libdtans: {msg}")
