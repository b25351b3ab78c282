"""Top SASS instructions by warp-stall samples from an ncu source-page CSV
(--page source --csv --print-source sass).  Usage: python tools/sass_stalls.py X.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
ins, base, tot = [], None, 0
for r in rows[2:]:
    try:
        a = int(r[ia], 16); n = int(r[iss] or 0)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    ins.append((a - base, r[isrc].strip(), n)); tot += n
print("total samples", tot)
for off, src, n in sorted(ins, key=lambda t: -t[2])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{off:#07x} {n:>7} ({100*n/tot:4.1f}%) {src}")
