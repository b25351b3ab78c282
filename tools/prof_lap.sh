#!/bin/bash
# Source-level capture of the Laplacian main kernel (one launch).
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/lap_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse "$@" > /dev/null 2>&1
ncu -i gpurun_out/lap_full.ncu-rep --page source --csv --print-source sass > gpurun_out/lap_src.csv 2>/dev/null
ls -la gpurun_out
