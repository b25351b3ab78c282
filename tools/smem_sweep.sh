#!/bin/bash
# Shared-memory cap sweep (L1 left for x gathers), one line per config.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:12], d["config"].get("row_order","")[:10], "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],3))'
for v in "DTANS_SMEM_KB=227" "DTANS_SMEM_KB=196" "DTANS_SMEM_KB=164" "DTANS_SMEM_KB=132"; do
  echo "== $v"
  env $v python bench.py --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
  env $v python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
  env $v python bench.py --config rmat --scale 0.125 --steps 20 --reorder --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
  env $v python bench.py --config rmat --scale 0.125 --steps 20 --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
done
