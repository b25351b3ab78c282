#!/bin/bash
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:12], "ms", round(d["ms_per_step"],4))'
for L in paper_2603_01915_b200/libdtans.so paper_2603_01915_b200/exp/libdtans_fma.so; do
  echo "== $L"
  DTANS_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  DTANS_LIB=$L timeout 300 python bench.py --config banded27 --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  DTANS_LIB=$L timeout 600 python bench.py --config powerit --steps 20 --no-device-encode 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("powerit ms/iter", round(d["ms_per_step"],4))'
done
