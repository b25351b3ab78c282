#!/bin/bash
# DTANS_CTA_STAGES sweep of the CTA-pipelined kernel.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:12], d["config"].get("row_order","")[:8], "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],3))'
for v in "DTANS_CTA=0" "DTANS_CTA=1 DTANS_CTA_STAGES=6" "DTANS_CTA=1 DTANS_CTA_STAGES=8" "DTANS_CTA=1 DTANS_CTA_STAGES=12" "DTANS_CTA=1 DTANS_CTA_STAGES=16"; do
  echo "== $v"
  env $v timeout 300 python bench.py --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  env $v timeout 300 python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  env $v timeout 300 python bench.py --config rmat --scale 0.125 --steps 20 --reorder --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
done
