#!/bin/bash
# Delta-dictionary replication budget A/B on R-MAT (full scale, sorted and natural).
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("ms", round(d["ms_per_step"],4))'
for kb in 8 16 32 64; do
  DTANS_DDICT_KB=$kb DTANS_VERBOSE=1 timeout 300 python bench.py --config rmat --reorder --steps 3 --no-cpu-baseline --no-cusparse --no-device-encode 2>&1 | grep -o "bufb=[0-9]*.*rep_v=[0-9]*" | head -1
  echo -n "ddict ${kb}KB sorted: "; DTANS_DDICT_KB=$kb timeout 300 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  echo -n "ddict ${kb}KB natural: "; DTANS_DDICT_KB=$kb timeout 300 python bench.py --config rmat --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
done
