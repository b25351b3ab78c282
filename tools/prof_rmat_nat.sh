#!/bin/bash
# Launch list of R-MAT natural order (full scale), plus the upload plan.
DTANS_VERBOSE=1 python bench.py --config rmat --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse 2>&1 | grep "\[dtans\]" > gpurun_out/rn_plan.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/rn_launches.csv python bench.py --config rmat --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
