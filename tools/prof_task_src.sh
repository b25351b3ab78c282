#!/bin/bash
# Source-level (SASS) capture of the R-MAT sorted task kernel: stall samples
# per instruction -> gpurun_out/task_src.csv (+ annotated listing).
cd "$(dirname "$0")/.."
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dtans_task_kernel -s 5 -c 1 -f \
    -o gpurun_out/task_src python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --launches 7 > gpurun_out/task_src_ncu.log 2>&1
ncu -i gpurun_out/task_src.ncu-rep --page source --csv --print-source sass > gpurun_out/task_src.csv 2>/dev/null
python tools/sass_annot.py gpurun_out/task_src.csv 1 > gpurun_out/task_src_annot.txt
rm -f gpurun_out/task_src.ncu-rep
head -3 gpurun_out/task_src_annot.txt
