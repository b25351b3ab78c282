"""Golden vectors for the quantizer, produced by the REFERENCE
(/root/reference/pkg/src/csrdtans/entropy.py:223-321 ``quantize``).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_quantize_golden.py

Each case: ascending integer symbols, counts, (k, m, raw_width_bits,
never_retain) and the reference's multiplicities / escape multiplicity /
escape slots.  Sizes span the exhaustive branch (<= 95 candidates) and the
coarse-to-fine branch (entropy.py:292-306).
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
from csrdtans.entropy import SymbolDistribution, quantize  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(20260317)
    recs = {}
    i = 0
    sizes = [1, 2, 3, 5, 16, 17, 40, 95, 96, 97, 200, 1000, 4095, 4096, 4097, 6000, 20000]
    for n in sizes:
        for shape in ("zipf", "uniform", "flat"):
            for (k, m, raw) in ((4096, 256, 32), (4096, 256, 64), (4096, 16, 32), (1024, 64, 32), (8, 4, 4)):
                if n > 5000 and (k, m) != (4096, 256):
                    continue
                sym = np.sort(rng.choice(2**40, n, replace=False)).astype(np.uint64)
                if shape == "zipf":
                    cnt = np.minimum(rng.zipf(1.3, n), 10**6).astype(np.int64)
                elif shape == "uniform":
                    cnt = rng.integers(1, 50, n).astype(np.int64)
                else:
                    cnt = np.full(n, 7, dtype=np.int64)
                never = []
                if n > 3 and i % 3 == 0:
                    never = [int(sym[j]) for j in rng.choice(n, 2, replace=False)]
                d = SymbolDistribution(tuple(int(s) for s in sym), tuple(int(c) for c in cnt))
                q = quantize(d, k, m, raw, never_retain=frozenset(never))
                recs[f"c{i}_sym"] = sym
                recs[f"c{i}_cnt"] = cnt
                recs[f"c{i}_cfg"] = np.array([k, m, raw], dtype=np.int64)
                recs[f"c{i}_never"] = np.array(never, dtype=np.uint64)
                recs[f"c{i}_mult"] = np.array(q.multiplicities, dtype=np.int32)
                recs[f"c{i}_esc"] = np.array([q.escape_multiplicity, q.escape_slots], dtype=np.int32)
                i += 1
    recs["ncases"] = np.int64(i)
    np.savez_compressed(os.path.join(HERE, "quantize_cases.npz"), **recs)
    print("cases", i)


if __name__ == "__main__":
    main()
