"""Paper-style report (CSV on stdout): StatsReport per matrix and, with
--gpu, kernel timings vs cuSPARSE (median of 7, warm and cold L2).

    python tools/evaluate.py [--mtx A.mtx ...] [--config laplacian:700 banded:60000 rmat:16 ...]
                             [--precision 8] [--gpu]
"""
import argparse
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_01915_b200 import encode_matrix, read_mtx, synth  # noqa: E402
from paper_2603_01915_b200.evaluate import stats_report, time_spmv  # noqa: E402


def synth_matrix(spec):
    kind, _, arg = spec.partition(":")
    if kind == "laplacian":
        return synth.laplacian_2d(int(arg or 700))
    if kind == "banded":
        return synth.banded(int(arg or 60000), 27)
    if kind == "rmat":
        sc = int(arg or 16)
        return synth.rmat(sc, 16 << sc)
    if kind == "config1":
        return synth.config1_random()
    raise SystemExit(f"unknown synthetic matrix {spec}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mtx", nargs="*", default=[])
    ap.add_argument("--config", nargs="*", default=[])
    ap.add_argument("--precision", type=int, default=8, choices=[4, 8])
    ap.add_argument("--gpu", action="store_true")
    a = ap.parse_args()
    items = [(p, lambda p=p: read_mtx(p)) for p in a.mtx] + [(s, lambda s=s: synth_matrix(s)) for s in a.config]
    w = None
    for name, load in items:
        m = load()
        c = encode_matrix(m, value_width=a.precision)
        row = stats_report(m, a.precision, name, container=c)
        if a.gpu:
            for cold in (False, True):
                t = time_spmv(m, c, cold=cold)
                pre = "cold_" if cold else ""
                row.update({pre + k: v for k, v in t.items() if k != "cold"})
        if w is None:
            w = csv.DictWriter(sys.stdout, fieldnames=list(row))
            w.writeheader()
        w.writerow(row)
        sys.stdout.flush()


if __name__ == "__main__":
    main()
