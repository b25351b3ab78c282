"""B200-native CSR-dtANS: entropy-coded sparse matrices with a fused
decode + SpMV kernel for sm_100a.

Drop-in for the hot path of the reference package ``csrdtans``
(/root/reference/pkg/src/csrdtans/__init__.py:55-66): the container API keeps
its names, signatures and exceptions; ``encode_matrix`` runs a byte-identical
C++ encoder and ``spmv`` / ``decode_matrix`` run hand-written CUDA kernels
(libdtans.so).  There is no CPU fallback on the product path.
"""

from .errors import CodingError, ContainerError, CorruptStream, NativeUnavailable, ParameterError
from .params import DtansParams, validate_params
from .sparse import (CooMatrix, CsrMatrix, MtxFormatError, coo_to_csr, format_size_bytes, matrix_deltas,
                     parse_mtx, read_mtx, reference_spmv, sort_rows_by_length, sort_symmetric_by_degree,
                     value_patterns)
from .tables import ESCAPE, CodingTables, quantize_counts
from .container import (SLICE_HEIGHT, CsrDtansContainer, DeviceContainer, compression_ratio,
                        decode_matrix, deserialize, encode_matrix, load, save, serialize, size_bytes, spmv)

__version__ = "0.1.0"

__all__ = [
    "CodingError", "ContainerError", "CorruptStream", "NativeUnavailable", "ParameterError",
    "DtansParams", "validate_params", "CooMatrix", "CsrMatrix", "MtxFormatError", "coo_to_csr",
    "parse_mtx", "read_mtx", "sort_symmetric_by_degree",
    "format_size_bytes", "matrix_deltas", "reference_spmv", "sort_rows_by_length", "value_patterns", "ESCAPE",
    "CodingTables", "quantize_counts", "SLICE_HEIGHT", "CsrDtansContainer", "DeviceContainer",
    "compression_ratio", "decode_matrix", "deserialize", "encode_matrix", "serialize",
    "size_bytes", "spmv", "load", "save",
]
