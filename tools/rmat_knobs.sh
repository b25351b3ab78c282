#!/bin/bash
# R-MAT (full scale, rows sorted) long-slice knobs: task length and long threshold.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("ms", round(d["ms_per_step"],4))'
for v in "DTANS_CHUNK=16" "DTANS_CHUNK=8" "DTANS_CHUNK=32" "DTANS_CHUNK=64" "DTANS_LONG_SEG=32" "DTANS_LONG_SEG=127" "DTANS_CTA=1" "DTANS_CTA=1 DTANS_CHUNK=32"; do
  echo -n "$v: "; env $v timeout 300 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
done
