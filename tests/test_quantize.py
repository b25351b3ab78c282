"""The C++ quantizer against the reference quantize (golden vectors from
tests/golden/make_quantize_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from paper_2603_01915_b200 import quantize_counts

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "quantize_cases.npz"))
N = int(Z["ncases"])


@pytest.mark.parametrize("i", range(N))
def test_quantize_matches_reference(i):
    k, m, raw = Z[f"c{i}_cfg"].tolist()
    mult, em, es = quantize_counts(Z[f"c{i}_sym"], Z[f"c{i}_cnt"], k, m, raw,
                                   never_retain=Z[f"c{i}_never"].tolist())
    assert np.array_equal(mult, Z[f"c{i}_mult"])
    assert [em, es] == Z[f"c{i}_esc"].tolist()


def test_quantize_paper_example():
    # entropy.py docstring / SPEC: P = {a:1, b:5, c:4}, K=8, M=8 -> (1, 4, 3)
    mult, em, es = quantize_counts([0, 1, 2], [1, 5, 4], 8, 8, 4)
    assert mult.tolist() == [1, 4, 3] and em == 0 and es == 0


def test_quantize_empty_is_escape_only():
    mult, em, es = quantize_counts([], [], 4096, 256, 32)
    assert len(mult) == 0 and em == 256 and es == 4096
