#!/bin/bash
# Current build vs HEAD~ build (exp/libdtans_prev.so): Laplacian, banded, power iteration, interleaved runs.
s1='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4))'
for rep in 1 2; do
for L in paper_2603_01915_b200/libdtans.so paper_2603_01915_b200/exp/libdtans_prev.so; do
  echo -n "$L lap "; DTANS_LIB=$L python bench.py --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$s1"
  echo -n "$L b27 "; DTANS_LIB=$L python bench.py --config banded27 --steps 30 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$s1"
  echo -n "$L pit "; DTANS_LIB=$L python bench.py --config powerit --steps 20 --no-device-encode 2>/dev/null | python -c "$s1"
done
done
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
