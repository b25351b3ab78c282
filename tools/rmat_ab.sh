#!/bin/bash
# R-MAT (1/8 and full scale) A/B of task staging; parity first.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:12], d["config"].get("row_order","")[:10], "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],3))'
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
DTANS_LONG_SEG=4 python -m pytest tests/test_gpu.py -x -q 2>&1 | tail -1
for v in "DTANS_TASK_STAGE=1" "DTANS_TASK_STAGE=0" "DTANS_TASK_FIT=1" "DTANS_TASK_FIT=1 DTANS_CHUNK=8"; do
  echo "== $v"
  env $v DTANS_VERBOSE=1 python bench.py --config rmat --scale 0.125 --steps 20 --reorder --no-cpu-baseline --no-cusparse 2>gpurun_out/v.err | python -c "$summ"; grep -o "ntasks.*" gpurun_out/v.err | head -1
  env $v python bench.py --config rmat --scale 0.125 --steps 20 --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
done
