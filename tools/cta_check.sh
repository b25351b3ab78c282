#!/bin/bash
# CTA-pipelined main kernel (DTANS_CTA=1): parity (bounded by timeouts), then A/B timing.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:12], d["config"].get("row_order","")[:8], "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],3))'
DTANS_CTA=1 DTANS_VERBOSE=1 timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse --no-device-encode 2>&1 | grep -o "cta_stages.*" | head -1; DTANS_CTA=1 DTANS_VERBOSE=1 timeout 120 python bench.py --config banded27 --scale 0.25 --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse --no-device-encode 2>&1 | grep -o "chunks=[0-9]*.*cta_stages.*" | head -1
echo "smoke rc=$?"
DTANS_CTA=1 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "DTANS_CTA=0" "DTANS_CTA=1"; do
  echo "== $v"
  env $v timeout 300 python bench.py --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  env $v timeout 300 python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  env $v timeout 300 python bench.py --config rmat --scale 0.125 --steps 20 --reorder --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  env $v timeout 300 python bench.py --config powerit --scale 0.25 --steps 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("powerit ms/iter", round(d["ms_per_step"],4))'
done
