"""The C-ABI library loads and exports every symbol include/dtans.h declares
(no compute calls that need a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2603_01915_b200 import _native

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "dtans.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dtans_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert sorted(_native.EXPORTS) == declared()


@pytest.mark.parametrize("sym", declared())
def test_symbol_exported(sym):
    lib = ctypes.CDLL(_native.LIB_PATH)
    assert hasattr(lib, sym)


def test_abi_version_and_error_text():
    L = _native.lib()
    assert L.dtans_abi_version() == 1
    assert isinstance(L.dtans_last_error(), bytes)


def test_no_device_is_loud_not_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2603_01915_b200 as P
    from paper_2603_01915_b200 import synth
    c = P.encode_matrix(synth.fig1())
    import numpy as np
    with pytest.raises(P.NativeUnavailable):
        P.spmv(c, np.ones(4), np.zeros(4))
