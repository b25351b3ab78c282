#!/bin/bash
# Source-level capture of the R-MAT (1/8 scale, rows sorted) task + main kernels.
ncu --set full --clock-control none --import-source on -k regex:dtans_task_kernel -s 3 -c 1 -o gpurun_out/task_full python bench.py --config rmat --scale 0.125 --reorder --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
ncu -i gpurun_out/task_full.ncu-rep --page source --csv --print-source sass > gpurun_out/task_src.csv 2>/dev/null
ncu -i gpurun_out/task_full.ncu-rep --page raw --csv > gpurun_out/task_raw.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/task_launches.csv python bench.py --config rmat --scale 0.125 --reorder --steps 5 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
