#!/bin/bash
# CTA kernel with full-stage sizing vs the per-warp ring, all headline configs.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:12], d["config"].get("row_order","")[:8], "ms", round(d["ms_per_step"],4))'
for v in "DTANS_CTA=0" "DTANS_CTA=1"; do
  echo "== $v"
  for rep in 1 2; do env $v timeout 300 python bench.py --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"; done
  env $v DTANS_VERBOSE=1 timeout 300 python bench.py --steps 3 --no-cpu-baseline --no-cusparse --no-device-encode 2>&1 | grep -o "cta_stages=[0-9]* cta_bufb=[0-9]*" | head -1
  env $v timeout 300 python bench.py --config banded27 --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  env $v timeout 300 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  env $v timeout 300 python bench.py --config rmat --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  env $v timeout 600 python bench.py --config powerit --steps 20 --no-device-encode 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("powerit ms/iter", round(d["ms_per_step"],4))'
done
