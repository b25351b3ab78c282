"""Encoder byte identity at BASELINE size.

tests/golden/fullscale.json was made by running the reference's own
encode_matrix steps on the full-size benchmark matrices (configs 2, 3 and
4; tests/golden/make_fullscale_golden.py): quantize + build_tables over the
full distributions (entropy.py:223-436, container.py:126-164) -> the table
block (container.py:612-625), and dtans_encode + interleave_warp
(codec.py:296-368, container.py:283-317) on 64 sampled slices.  Here the
host C++ encoder and the GPU encoder encode the same matrices and must
reproduce the table block and every sampled slice's stream words and
row_symbols byte for byte.

These matrices hold up to 2^28 nonzeros (several GB on the host), so the
test runs on the GPU box (-m gpu), where the GPU encoder is exercised too;
the config-2 host-encoder check also runs in the CPU suite.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth
from paper_2603_01915_b200.container import _records

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "fullscale.json")))

GEN = {
    "laplacian": lambda: synth.laplacian_rows(2591, 0, 2591 * 2591),
    "rmat": lambda: synth.rmat(23, 2**27),
    "banded27": lambda: synth.banded_rows(-(-2**28 // 27), 0, -(-2**28 // 27), 27, positive=False),
}


def _check(c, g):
    assert (c.rows, c.cols, c.nnz, c.precision) == (g["rows"], g["cols"], g["nnz"], g["precision"])
    assert hashlib.sha256(_records(c).tobytes()).hexdigest() == g["tables_sha256"]
    d = np.asarray(c.directory, dtype=np.int64)
    for rec in g["slices"]:
        s = rec["slice"]
        w = np.asarray(c.stream[d[s]:d[s + 1]], dtype=np.uint32)
        assert len(w) == rec["words"], s
        assert hashlib.sha256(w.tobytes()).hexdigest() == rec["sha256"], s
        rs = np.asarray(c.row_symbols[32 * s:min(32 * (s + 1), c.rows)], dtype=np.uint32)
        assert hashlib.sha256(rs.tobytes()).hexdigest() == rec["row_symbols_sha256"], s


def test_fullscale_host_encoder_laplacian():
    """Config 2 (6.7M distinct first deltas) on the host encoder: ~10 s, so
    it also runs in the CPU suite."""
    _check(P.encode_matrix(GEN["laplacian"]()), GOLD["laplacian"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["laplacian", "rmat", "banded27"])
def test_fullscale_encoders_match_reference(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    g = GOLD[name]
    m = GEN[name]()
    c = P.encode_matrix(m)
    _check(c, g)
    cd = P.encode_matrix(m, device=0)
    assert cd == c
