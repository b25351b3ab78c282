#!/bin/bash
# A/B of experiment builds (DTANS_LIB) on the headline configs, one line each.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:12], "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],3))'
for L in "$@"; do
  echo "== $L"
  DTANS_LIB=$L python -m pytest tests -m gpu -x -q 2>&1 | tail -1
  DTANS_LIB=$L python bench.py --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
  DTANS_LIB=$L python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
  DTANS_LIB=$L python bench.py --config rmat --scale 0.125 --steps 20 --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
  DTANS_LIB=$L python bench.py --config rmat --scale 0.125 --steps 20 --reorder --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
done
