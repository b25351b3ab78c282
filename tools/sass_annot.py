"""Annotated SASS listing from an ncu --page source --print-source sass CSV:
offset, executions, stall samples (and the top reasons), instruction.
Usage: python tools/sass_annot.py X.csv [min_exec] > listing.txt"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 1
stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
base = None
tot_e = tot_s = 0
out = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[ix["Address"]], 16)
    base = a if base is None else base
    e = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot_e += e
    tot_s += s
    st = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:2]
    sd = " ".join(f"{k}:{v}" for v, k in st if v)
    if e >= mn:
        out.append(f"{a - base:05x} {e:>9} {s:>6} {sd:<28} {r[ix['Source']].strip()}")
print(f"# total warp-instructions {tot_e}  stall samples {tot_s}")
print("\n".join(out))
