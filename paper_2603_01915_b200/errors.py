"""Exception types of the drop-in API.

Mirrors the reference classes so callers catching them keep working:
``ParameterError`` / ``CodingError`` / ``CorruptStream``
(/root/reference/pkg/src/csrdtans/entropy.py:18-27) and ``ContainerError``
(/root/reference/pkg/src/csrdtans/container.py:87-88).
"""


class ParameterError(ValueError):
    """Invalid coder parameters or mismatched dimensions."""


class CodingError(ValueError):
    """Input the coder cannot represent (unknown symbol, oversize payload)."""


class CorruptStream(ValueError):
    """A compressed stream that cannot have been produced by the encoder.

    Raised on the GPU path when the decode kernel's per-slice consumption
    check (cursor == directory[s+1]) or its column bound fails.
    """


class ContainerError(ValueError):
    """Malformed container bytes (magic, version, CRC, truncation)."""


class NativeUnavailable(RuntimeError):
    """The CUDA extension (libdtans.so) or a CUDA device is missing.

    The product path never falls back to a CPU implementation; it raises.
    """
