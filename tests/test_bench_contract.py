"""bench.py's JSON-line contract on the CPU-runnable legs: the reference arm
(`--impl reference`, the oracle C port timed on the host cores) prints one
line with the keys the driver reads.  The dtANS arm needs a GPU
(tests/test_gpu.py exercises its kernels)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, capture_output=True, text=True,
                         timeout=600, cwd=REPO, env=e)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run(["--impl", "reference", "--config", "config1", "--steps", "2", "--warmup", "1"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["steps"] == 2 and d["warmup"] >= 3  # W >= 3 is enforced
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["config"]["workload"].startswith("random 4096x4096")


def _bench():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(REPO, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_shard_rows_cover_and_balance():
    """N>1: nnz-balanced contiguous slice ranges that cover every row once."""
    import numpy as np
    B = _bench()
    from paper_2603_01915_b200 import synth
    for rn in (synth.laplacian_row_nnz(97), synth.banded_row_nnz(50000, 27),
               np.random.default_rng(0).integers(0, 400, 7777)):
        for world in (1, 2, 3, 8):
            cuts = [B.shard_rows(rn, world, r) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == len(rn)
            for (a, b), (c, d) in zip(cuts, cuts[1:]):
                assert b == c and a % 32 == 0
            per = [int(rn[a:b].sum()) for a, b in cuts]
            assert max(per) - min(per) <= 2 * 32 * int(rn.max()) + 1  # one slice per cut


def test_spec_row_blocks_are_the_global_matrix():
    """Every rank generates only its rows; the blocks concatenate to the
    N=1 matrix (same seeds), so N>1 is strong scaling of one matrix."""
    import numpy as np
    B = _bench()
    for cfg, scale in (("laplacian", 0.02), ("banded27", 1e-4), ("banded32", 1e-3), ("rmat", 2 ** -12)):
        s = B.Spec(cfg, scale)
        full = s.block(0, s.rows)
        assert np.array_equal(np.diff(full.row_start), s.row_nnz())
        cuts = [B.shard_rows(s.row_nnz(), 3, r) for r in range(3)]
        cols = np.concatenate([s.block(a, b).col_idx for a, b in cuts])
        vals = np.concatenate([s.block(a, b).values for a, b in cuts])
        assert np.array_equal(cols, full.col_idx) and np.array_equal(vals, full.values)
        x, y = s.vectors(0, s.rows)
        x2, y2 = s.vectors(*cuts[1])
        assert np.array_equal(x, x2) and np.array_equal(y[cuts[1][0]:cuts[1][1]], y2)
