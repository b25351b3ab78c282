#!/bin/bash
# Host-buffer path: parity tests, then e2e with and without the x windows.
python -m pytest tests/test_gpu.py -x -q -k "host_buffer" 2>&1 | tail -3
e2e='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:14], "e2e", round(d["e2e"]["value"],1), round(d["e2e"]["ms_per_step"],3), "ms", d["e2e"].get("matches_device_result"))'
for v in "DTANS_HOST_WINDOWS=1" "DTANS_HOST_WINDOWS=0" "DTANS_HOST_WINDOWS=1 DTANS_HOST_STAGES=16"; do
  echo "== $v"
  env $v python bench.py --steps 30 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$e2e"
  env $v python bench.py --config banded27 --steps 20 --no-cpu-baseline --no-cusparse --no-device-encode 2>/dev/null | python -c "$e2e"
done
