"""StatsReport (paper-style evaluation)."""

import numpy as np
import pytest

import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth
from paper_2603_01915_b200.evaluate import stats_report


def test_stats_report_fields_and_invariants():
    m = synth.laplacian_2d(60)
    r = stats_report(m, 8, "lap60")
    best = min(r["bytes_coo"], r["bytes_csr"], r["bytes_sell"])
    assert r["bytes_dtans"] == P.size_bytes(P.encode_matrix(m))
    assert r["best_baseline_ratio"] == pytest.approx(r["bytes_dtans"] / best)
    assert r["annzpr"] == pytest.approx(m.nnz / m.rows)
    assert r["value_escapes"] == 0 and r["value_entropy_bits"] < 1.0


def test_stats_report_escape_counts_random_values():
    # config 1: every value is distinct, so none fits the 4096-slot table
    m = synth.config1_random()
    r = stats_report(m, 8)
    assert r["value_escapes"] > 0.5 * m.nnz
    assert r["best_baseline_ratio"] > 1.0  # SPEC: random fp64 values never compress


def test_stats_report_f32():
    m = synth.rmat(10, 16 << 10)
    r = stats_report(m, 4)
    assert r["precision"] == 4 and r["bytes_dtans"] > 0


@pytest.mark.gpu
def test_time_spmv_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_01915_b200.evaluate import time_spmv
    m = synth.laplacian_2d(300)
    t = time_spmv(m, runs=3)
    assert t["dtans_ms"] > 0 and t["cusparse_ms"] > 0 and np.isfinite(t["speedup"])
