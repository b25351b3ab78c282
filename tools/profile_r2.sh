#!/bin/bash
# Round-2 ncu evidence (one GPU): per config, the launch list of the bench
# command (gpu__time_duration.sum, --clock-control none) and one
# `--set full --import-source on` capture of the dominant kernel(s), each
# summarised into gpurun_out/r2_<cfg>.md (tools/profile_report.py) plus the
# traffic/instruction numbers bench.py reads (gpurun_out/traffic_<config>.json).
#   tools/profile_r2.sh [lap b27 rmat pit]
cd "$(dirname "$0")/.."
CFGS=${@:-lap b27 rmat pit}
full() {  # name kernel-regex skip kbench-or-bench-args...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -f \
      -o gpurun_out/r2_${name} "$@" > gpurun_out/r2_${name}_ncu.log 2>&1
  ncu -i gpurun_out/r2_${name}.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_${name}_src.csv 2>/dev/null
}
traffic() {  # name config
  python - "$1" "$2" <<'PY'
import csv, io, json, subprocess, sys
name, cfg = sys.argv[1:3]
out = subprocess.run(["ncu", "-i", f"gpurun_out/r2_{name}.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v)); un = dict(zip(h, u))
def num(k, scale=1.0):
    x = float(d[k].replace(",", ""))
    unit = un.get(k, "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return x * mult
rec = {"dram_bytes_per_launch": int(num("dram__bytes_read.sum") + num("dram__bytes_write.sum")),
       "warp_inst_per_launch": int(num("smsp__inst_executed.sum")),
       "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
       "duration_us_under_ncu": num("gpu__time_duration.sum") / (1e3 if un.get("gpu__time_duration.sum") == "nsecond" else 1),
       "kernel": d.get("Kernel Name", ""), "source": f"profiles/r2_{name}.md (ncu --set full, one launch)"}
json.dump(rec, open(f"gpurun_out/traffic_{cfg}.json", "w"), indent=1)
print(name, rec)
PY
}
for c in $CFGS; do
  case $c in
  lap)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_lap_launches.csv \
        python bench.py --steps 20 --no-cpu-baseline --no-device-encode > /dev/null 2>&1
    full lap dtans_kernel 5 python tools/kbench.py --config laplacian --launches 7
    python tools/profile_report.py gpurun_out/r2_lap.md --launches gpurun_out/r2_lap_launches.csv --full gpurun_out/r2_lap.ncu-rep \
        --title "Round 2, config 2 (Laplacian 2^25 nnz, f64), 1x B200" --cmd "tools/profile_r2.sh lap"
    traffic lap laplacian ;;
  b27)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2_b27_launches.csv \
        python bench.py --config banded27 --steps 10 --no-cpu-baseline --no-device-encode > /dev/null 2>&1
    full b27 dtans_kernel 5 python tools/kbench.py --config banded27 --launches 7
    python tools/profile_report.py gpurun_out/r2_b27.md --launches gpurun_out/r2_b27_launches.csv --full gpurun_out/r2_b27.ncu-rep \
        --title "Round 2, config 4 (banded-27, 2^28 nnz, f64), 1x B200" --cmd "tools/profile_r2.sh b27"
    traffic b27 banded27 ;;
  rmat)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2_rmat_launches.csv \
        python bench.py --config rmat --reorder --steps 10 --no-cpu-baseline --no-device-encode > /dev/null 2>&1
    full rmat_task dtans_task_kernel 5 python tools/kbench.py --config rmat --reorder --launches 7
    full rmat_main dtans_kernel 5 python tools/kbench.py --config rmat --reorder --launches 7
    python tools/profile_report.py gpurun_out/r2_rmat_task.md --launches gpurun_out/r2_rmat_launches.csv --full gpurun_out/r2_rmat_task.ncu-rep \
        --title "Round 2, config 3 (R-MAT 2^27 nnz, f32, rows sorted): long-slice task kernel, 1x B200" --cmd "tools/profile_r2.sh rmat"
    python tools/profile_report.py gpurun_out/r2_rmat_main.md --full gpurun_out/r2_rmat_main.ncu-rep \
        --title "Round 2, config 3 (R-MAT, rows sorted): main kernel, 1x B200" --cmd "tools/profile_r2.sh rmat" ;;
  pit)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2_pit_launches.csv \
        python bench.py --config powerit --steps 10 --no-device-encode > /dev/null 2>&1
    full pit dtans_kernel 4 python bench.py --config powerit --steps 3 --warmup 3 --no-device-encode
    python tools/profile_report.py gpurun_out/r2_pit.md --launches gpurun_out/r2_pit_launches.csv --full gpurun_out/r2_pit.ncu-rep \
        --title "Round 2, config 5 (power iteration, banded-32 2^29 nnz, f64): scaled y-less kernel, 1x B200" --cmd "tools/profile_r2.sh pit" ;;
  esac
done
# the .ncu-rep files are large (gpurun copies back at most 64 MiB): keep the summaries
rm -f gpurun_out/r2_*.ncu-rep
ls -la gpurun_out | grep r2_
