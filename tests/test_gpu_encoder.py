"""GPU encoder (dtans_encode_device): byte identity with the reference
encoder's goldens and with the host encoder on larger matrices.  Run on a
B200 with `pytest -m gpu`."""

import hashlib

import numpy as np
import pytest

import golden_cases as G
import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("name", G.names())
def test_device_encode_byte_identical_to_reference(name):
    rec = G.load(name)
    c = P.encode_matrix(G.matrix(rec), **G.encode_kwargs(rec), device=0)
    assert hashlib.sha256(P.serialize(c)).hexdigest() == str(rec["sha256"])
    assert len(c.stream) == int(rec["nwords"])


def _random_specials(seed, rows, cols, nnz, dtype):
    rng = np.random.default_rng(seed)
    flat = np.sort(rng.choice(rows * cols, nnz, replace=False))
    r, c = np.divmod(flat, cols)
    row_start = np.zeros(rows + 1, dtype=np.int64)
    np.add.at(row_start, r + 1, 1)
    v = rng.standard_normal(nnz).astype(dtype)
    v[rng.random(nnz) < 0.01] = np.inf
    v[rng.random(nnz) < 0.01] = -0.0
    v[rng.random(nnz) < 0.01] = np.nan
    v[rng.random(nnz) < 0.3] = 1.0  # a retained majority next to escapes
    return P.CsrMatrix(rows, cols, np.cumsum(row_start), c.astype(np.int64), v)


LARGE = {
    "laplacian_g700": lambda: synth.laplacian_2d(700),
    "banded27_40k": lambda: synth.banded(40000, 27, levels=256, seed=3),
    "rmat_s14_f32": lambda: synth.rmat(14, 16 << 14),
    "random_specials_f64": lambda: _random_specials(7, 20000, 30000, 300000, np.float64),
    "random_specials_f32": lambda: _random_specials(8, 5000, 70000, 120000, np.float32),
    "one_long_row": lambda: P.CsrMatrix(3, 300000, np.array([0, 1, 150001, 150002]),
                                        np.concatenate([[5], np.arange(0, 300000, 2), [7]]).astype(np.int64),
                                        np.linspace(-1, 1, 150002)),
    "empty_rows": lambda: P.CsrMatrix(100, 10, np.zeros(101, dtype=np.int64), np.zeros(0, dtype=np.int64),
                                      np.zeros(0)),
}


@pytest.mark.parametrize("name", sorted(LARGE))
def test_device_encode_matches_host_encoder(name):
    m = LARGE[name]()
    host = P.serialize(P.encode_matrix(m))
    dev = P.serialize(P.encode_matrix(m, device=0))
    assert dev == host


@pytest.mark.parametrize("seed", [None, 12345])
def test_device_encode_permutation_seed(seed):
    m = synth.banded(5000, 7, levels=40, seed=1)
    assert P.serialize(P.encode_matrix(m, permutation_seed=seed, device=0)) == \
        P.serialize(P.encode_matrix(m, permutation_seed=seed))


def test_device_encode_errors():
    with pytest.raises(P.ParameterError):
        P.encode_matrix(P.CsrMatrix(1, 5, np.array([0, 2]), np.array([3, 1]), np.array([1.0, 2.0])), device=0)
    with pytest.raises(P.ParameterError):
        P.encode_matrix(P.CsrMatrix(1, 3, np.array([0, 1]), np.array([3]), np.array([1.0])), device=0)
    with pytest.raises(P.ParameterError):
        P.encode_matrix(P.CsrMatrix(2, 3, np.array([0, 1]), np.array([0]), np.array([1.0])), device=0)
