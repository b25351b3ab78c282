#!/bin/bash
# Long-slice word-load flavour A/B on R-MAT (full scale, sorted and natural).
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("ms", round(d["ms_per_step"],4))'
for L in paper_2603_01915_b200/libdtans.so paper_2603_01915_b200/exp/libdtans_g1.so paper_2603_01915_b200/exp/libdtans_g2.so; do
  echo "== $L"
  echo -n "sorted: "; DTANS_LIB=$L timeout 300 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
  echo -n "natural: "; DTANS_LIB=$L timeout 300 python bench.py --config rmat --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$summ"
done
DTANS_LIB=paper_2603_01915_b200/exp/libdtans_g2.so DTANS_LONG_SEG=4 timeout 600 python -m pytest tests/test_gpu.py -x -q -k "long_slice or larger or rmat" 2>&1 | tail -1
