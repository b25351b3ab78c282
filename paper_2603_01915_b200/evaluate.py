"""Paper-style evaluation (the reference's missing
``cmd_stats`` / ``cmd_spmv`` harness).

``stats_report`` computes the StatsReport fields for one matrix: rows, cols,
nnz, annzpr, bytes per format (COO, CSR, SELL and CSR-dtANS), the
best-baseline ratio dtANS / min(COO, CSR, SELL), the empirical entropies
of the delta and value symbols, and the escape counts.
``time_spmv`` measures the fused kernel and cuSPARSE CSR (torch.addmv) on
one GPU: the median of 7 runs after a warm-up, the paper's protocol
(PAPER.md:469).  Warm runs keep the matrix in L2 when it fits; cold runs
write 2x L2 between runs.
"""

from __future__ import annotations

import statistics

import numpy as np

from .container import encode_matrix, size_bytes
from .sparse import CsrMatrix, format_size_bytes, matrix_deltas, value_patterns


def _entropy_bits(sym: np.ndarray) -> float:
    if len(sym) == 0:
        return 0.0
    _, cnt = np.unique(sym, return_counts=True)
    p = cnt / cnt.sum()
    return max(0.0, float(-(p * np.log2(p)).sum()))


def stats_report(m: CsrMatrix, precision: int = 8, name: str = "", container=None) -> dict:
    """StatsReport of ``m`` encoded at ``precision`` bytes per value (4 | 8)."""
    vdt = np.float64 if precision == 8 else np.float32
    mm = m if np.asarray(m.values).dtype == vdt else CsrMatrix(
        m.rows, m.cols, m.row_start, m.col_idx, np.asarray(m.values, dtype=vdt))
    c = container if container is not None else encode_matrix(mm)
    fmt = {f: format_size_bytes(mm, f, precision) for f in ("coo", "csr", "sell")}
    dt_bytes = size_bytes(c)
    deltas = matrix_deltas(mm)
    vals = value_patterns(np.asarray(mm.values))
    dret = np.asarray(c.delta_tables.retained_symbols(), dtype=np.uint64)
    vret = np.asarray(c.value_tables.retained_symbols(), dtype=np.uint64)
    d_esc = int(len(deltas) - np.isin(deltas.astype(np.uint64), dret).sum())
    v_esc = int(len(vals) - np.isin(vals.astype(np.uint64), vret).sum())
    best = min(fmt.values())
    return {
        "matrix": name, "rows": mm.rows, "cols": mm.cols, "nnz": mm.nnz,
        "annzpr": mm.nnz / mm.rows if mm.rows else 0.0, "precision": precision,
        "bytes_coo": fmt["coo"], "bytes_csr": fmt["csr"], "bytes_sell": fmt["sell"], "bytes_dtans": dt_bytes,
        "best_baseline_ratio": dt_bytes / best if best else float("nan"),
        "compression_vs_best": best / dt_bytes if dt_bytes else float("nan"),
        "delta_entropy_bits": _entropy_bits(deltas), "value_entropy_bits": _entropy_bits(vals),
        "delta_escapes": d_esc, "value_escapes": v_esc,
        "stream_words": int(len(c.stream)),
    }


def time_spmv(m: CsrMatrix, c=None, device: int = 0, runs: int = 7, cold: bool = False) -> dict:
    """Median kernel times (ms) of the fused dtANS SpMV and cuSPARSE CSR on
    the same x, y; GFLOP/s = 2 nnz / t; effective GB/s on the algorithmic
    bytes (container + x + y + y')."""
    import torch

    from .synth import vectors
    c = c if c is not None else encode_matrix(m)
    dev = torch.device("cuda", device)
    V = torch.float64 if c.precision == 8 else torch.float32
    x, y = vectors(m)
    xt = torch.from_numpy(np.asarray(x, dtype=np.float64 if c.precision == 8 else np.float32)).to(dev)
    yt = torch.from_numpy(np.asarray(y, dtype=np.float64 if c.precision == 8 else np.float32)).to(dev)
    out = torch.empty_like(yt)
    dc = c.device(device)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8,
                        device=dev) if cold else None

    def med(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(runs):
            if flush is not None:
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    t_d = med(lambda: dc.spmv(xt, yt, out))
    dc.check()
    A = torch.sparse_csr_tensor(torch.from_numpy(np.asarray(m.row_start)), torch.from_numpy(np.asarray(m.col_idx)),
                                torch.from_numpy(np.asarray(m.values)).to(V), size=(m.rows, m.cols)).to(dev)
    t_c = med(lambda: torch.addmv(yt, A, xt))
    esz = c.precision
    alg = size_bytes(c) + esz * m.cols + 2 * esz * m.rows
    return {"dtans_ms": t_d, "cusparse_ms": t_c, "speedup": t_c / t_d,
            "dtans_gflops": 2 * m.nnz / (t_d * 1e-3) / 1e9, "cusparse_gflops": 2 * m.nnz / (t_c * 1e-3) / 1e9,
            "dtans_eff_gbs": alg / (t_d * 1e-3) / 1e9, "cold": cold}
