"""SASS around the top stall sites with per-reason stall samples and execution
counts, from an ncu source-page CSV.  Usage: python tools/sass_ctx.py X.csv [N] [before]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ir = [hdr.index(h) for h in reasons]
ins = []
for r in rows[2:]:
    try:
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iss] or 0), int(r[iex] or 0),
                    {reasons[k][6:]: int(r[i] or 0) for k, i in enumerate(ir)}))
    except (ValueError, IndexError):
        pass
base = ins[0][0]
tot = sum(t[2] for t in ins)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 6
B = int(sys.argv[3]) if len(sys.argv) > 3 else 6
top = sorted(range(len(ins)), key=lambda i: -ins[i][2])[:N]
for i in sorted(top):
    print("-----")
    for j in range(max(0, i - B), i + 1):
        a, s, n, ex, rs = ins[j]
        why = ", ".join(f"{k}={v}" for k, v in sorted(rs.items(), key=lambda kv: -kv[1]) if v)[:70]
        print(f"{a-base:#07x} ex={ex:>8} st={n:>5} {s[:60]:<60} {why}")
