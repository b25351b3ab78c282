"""Summarise an .ncu-rep: key SOL/scheduler metrics, stall reasons, and
hot SASS blocks (by executed instructions)."""
import csv, subprocess, sys, io, collections

rep = sys.argv[1]
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

rows = page("details")
h = rows[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Active Warps Per SM", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "SM Frequency", "Avg. Active Threads Per Warp"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:<40} {d['Metric Value']:>14} {d['Metric Unit']}")
raw = page("raw")
hdr, units, vals = raw[0], raw[1], raw[2]
rd = dict(zip(hdr, vals))
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "sm__inst_executed.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct"]:
    if k in rd:
        print(f"{k:<60} {rd[k]:>16} {units[hdr.index(k)]}")
stall = [(k, rd[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
stall = sorted(((k, float(v or 0)) for k, v in stall), key=lambda t: -t[1])[:10]
print("top stall reasons (warps per issue-active cycle):")
for k, v in stall:
    print(f"   {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):<28} {v:.3f}")
if len(sys.argv) > 2:
    src = page("source", ["--print-source", "sass"])
    h = src[1]; idx = {k: i for i, k in enumerate(h)}
    data = src[2:]
    tot = sum(int(r[idx["Instructions Executed"]] or 0) for r in data)
    print("total executed warp instructions", tot)
    blocks = []
    cur = None
    for r in data:
        ex = int(r[idx["Instructions Executed"]] or 0)
        st = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        if cur and cur[0] == ex:
            cur[1] += 1; cur[2] += st; cur[3].append(r[idx["Source"]].strip())
        else:
            cur = [ex, 1, st, [r[idx["Source"]].strip()]]; blocks.append(cur)
    for b in blocks:
        if b[0] * b[1] > tot / 200:
            print(f"  exec {b[0]:>9} x {b[1]:>4} = {b[0]*b[1]/1e6:7.2f}M  stalls={b[2]:>6}  {b[3][0][:50]} .. {b[3][-1][:40]}")
