"""Summarise an ncu --page source --print-source sass CSV: basic blocks
(runs of equal execution count) with their instruction counts, sorted by
total executed warp-instructions.  Usage: python tools/sass_hot.py X.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
iw = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
ins = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[iw] or 0) if iw else 0))
    except ValueError:
        pass
base = ins[0][0]
blocks, cur = [], None
for a, s, n, w in ins:
    if cur and cur["n"] == n and n > 0:
        cur["ins"].append(s); cur["wf"] += w
    else:
        cur = {"start": a - base, "n": n, "ins": [s], "wf": w}
        blocks.append(cur)
tot = sum(b["n"] * len(b["ins"]) for b in blocks)
totw = sum(b["wf"] for b in blocks)
print(f"total warp-instr {tot}  shared wavefronts {totw}")
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for b in sorted(blocks, key=lambda b: -b["n"] * len(b["ins"]))[:lim]:
    t = b["n"] * len(b["ins"])
    print(f"{b['start']:#07x} execs {b['n']:>9} len {len(b['ins']):>4} total {t:>10} ({100*t/tot:5.1f}%) wf {b['wf']:>9}  {b['ins'][0][:40]} .. {b['ins'][-1][:40]}")
