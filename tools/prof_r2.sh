#!/bin/bash
# Source-level ncu captures (one launch each) of the main kernel (Laplacian,
# banded-27 at 1/4 scale) and of the long-slice task kernel (R-MAT, rows
# sorted), plus plain kbench timings of the same workloads.
# Usage: tools/prof_r2.sh TAG [configs...]
cd "$(dirname "$0")/.."
TAG=${1:-r2}; shift
CFGS=${@:-lap b27 rmat}
for c in $CFGS; do
  case $c in
    lap) A="--config laplacian"; K=dtans_kernel;;
    b27) A="--config banded27 --scale 0.25"; K=dtans_kernel;;
    rmat) A="--config rmat --reorder"; K=dtans_task_kernel;;
    rmatm) A="--config rmat --reorder"; K=dtans_kernel;;
    pit) A="--config banded32 --noy"; K=dtans_kernel;;
  esac
  timeout 600 python tools/kbench.py $A --check > gpurun_out/${TAG}_${c}_time.json 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 -o gpurun_out/${TAG}_${c} -f \
      python tools/kbench.py $A --launches 7 > gpurun_out/${TAG}_${c}_ncu.log 2>&1
  ncu -i gpurun_out/${TAG}_${c}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${c}_src.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${c}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${c}_raw.csv 2>/dev/null
  cat gpurun_out/${TAG}_${c}_time.json | tail -1
done
ls -la gpurun_out | tail -30
