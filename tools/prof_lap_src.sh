#!/bin/bash
# Source-level (SASS) capture of the Laplacian main kernel -> gpurun_out/lap_src_annot.txt
cd "$(dirname "$0")/.."
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -f \
    -o gpurun_out/lap_src python tools/kbench.py --config laplacian --launches 7 > gpurun_out/lap_src_ncu.log 2>&1
ncu -i gpurun_out/lap_src.ncu-rep --page source --csv --print-source sass > gpurun_out/lap_src.csv 2>/dev/null
python tools/sass_annot.py gpurun_out/lap_src.csv 1 > gpurun_out/lap_src_annot.txt
python tools/profile_report.py gpurun_out/lap_src.md --full gpurun_out/lap_src.ncu-rep --title "Laplacian main kernel (source capture)" --cmd "tools/prof_lap_src.sh"
rm -f gpurun_out/lap_src.ncu-rep gpurun_out/lap_src.csv
head -3 gpurun_out/lap_src_annot.txt
