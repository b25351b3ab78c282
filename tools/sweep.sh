#!/bin/bash
# Env-knob sweep on the Laplacian and banded-27 (quarter scale), one line each.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:12], "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],3))'
for v in "$@"; do
  echo "== $v"
  env $v python bench.py --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
  env $v python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "$summ"
done
