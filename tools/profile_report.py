"""Write a markdown summary of an ncu launch list (CSV) and/or an ncu
--set full report into profiles/.  Usage:
  python tools/profile_report.py OUT.md [--launches L.csv] [--full R.ncu-rep] [--title T]"""
import argparse, csv, io, subprocess, sys
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--launches")
ap.add_argument("--full")
ap.add_argument("--title", default="ncu summary")
ap.add_argument("--cmd", default="")
a = ap.parse_args()
lines = [f"# {a.title}", ""]
if a.cmd:
    lines += ["Command: `" + a.cmd + "`", ""]
if a.launches:
    rows = [r for r in csv.reader(open(a.launches)) if len(r) > 5]
    h = rows[0]; idx = {k: i for i, k in enumerate(h)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        agg[r[idx["Kernel Name"]]][0] += 1
        agg[r[idx["Kernel Name"]]][1] += float(r[idx["Metric Value"]].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines += ["## Launch list (gpu__time_duration.sum, --clock-control none; cold, serialised)", "",
              "| launches | total us | mean us | share | kernel |", "|---:|---:|---:|---:|---|"]
    for k, v in sorted(agg.items(), key=lambda t: -t[1][1]):
        lines.append(f"| {v[0]} | {v[1]/1e3:.1f} | {v[1]/v[0]/1e3:.1f} | {100*v[1]/tot:.1f}% | `{k[:110]}` |")
    lines.append("")
if a.full:
    def page(p, extra=()):
        out = subprocess.run(["ncu", "-i", a.full, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
        return list(csv.reader(io.StringIO(out)))
    raw = page("raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    rd = dict(zip(hdr, vals)); ud = dict(zip(hdr, units))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
    lines += ["## Full capture of the top kernel (ncu --set full)", "", "| metric | value | unit |", "|---|---:|---|"]
    for k in keys:
        if k in rd:
            lines.append(f"| {k} | {rd[k]} | {ud.get(k,'')} |")
    st = [(k, float(rd[k] or 0)) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio")]
    st.sort(key=lambda t: -t[1])
    lines += ["", "Top warp stall reasons (warps per issue-active cycle):", ""]
    for k, v in st[:8]:
        lines.append(f"- {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}: {v:.3f}")
    try:
        rb = float(rd["dram__bytes_read.sum"]); wb = float(rd["dram__bytes_write.sum"])
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tb = rb * mult.get(ud["dram__bytes_read.sum"], 1) + wb * mult.get(ud["dram__bytes_write.sum"], 1)
        lines += ["", f"DRAM traffic per launch: {tb:.0f} bytes"]
        print(f"traffic_bytes {tb:.0f}")
    except Exception:
        pass
open(a.out, "w").write("\n".join(lines) + "\n")
print("wrote", a.out)
