#!/bin/bash
# Round-2 (second pass) ncu evidence for config 3 after the long-slice launch
# chain: launch lists of the rows-sorted and natural-order R-MAT products
# (gpu__time_duration.sum, --clock-control none: cold and serialised, so the
# PDL overlap of the chain is not visible, only each kernel's share) and one
# full capture of the task kernel (sorted).  Summaries: gpurun_out/r2b_*.md
cd "$(dirname "$0")/.."
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2b_rmat_sorted_launches.csv \
    python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --launches 20 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2b_rmat_natural_launches.csv \
    python tools/kbench.py --config rmat --cache /tmp/kcache --launches 20 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dtans_task_kernel -s 5 -c 1 -f \
    -o gpurun_out/r2b_rmat_task python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --launches 7 > gpurun_out/r2b_task_ncu.log 2>&1
python tools/profile_report.py gpurun_out/r2b_rmat_sorted.md --launches gpurun_out/r2b_rmat_sorted_launches.csv --full gpurun_out/r2b_rmat_task.ncu-rep \
    --title "Round 2b, config 3 (R-MAT 2^27 nnz, f32, rows sorted): launch chain + task kernel, 1x B200" --cmd "tools/profile_r2b.sh"
python tools/profile_report.py gpurun_out/r2b_rmat_natural.md --launches gpurun_out/r2b_rmat_natural_launches.csv \
    --title "Round 2b, config 3 (R-MAT 2^27 nnz, f32, natural row order): launch list, 1x B200" --cmd "tools/profile_r2b.sh"
rm -f gpurun_out/r2b_*.ncu-rep
ls -la gpurun_out | grep r2b_
