#!/bin/bash
# Source-level (SASS) captures of the main kernel: Laplacian and banded-27 (1/4 scale).
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/lap_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse --no-device-encode > /dev/null 2>&1
ncu -i gpurun_out/lap_full.ncu-rep --page source --csv --print-source sass > gpurun_out/lap_src.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/b27_full python bench.py --config banded27 --scale 0.25 --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse --no-device-encode > /dev/null 2>&1
ncu -i gpurun_out/b27_full.ncu-rep --page source --csv --print-source sass > gpurun_out/b27_src.csv 2>/dev/null
