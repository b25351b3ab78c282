#!/bin/bash
# cuSPARSE format comparator lines.
show='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:14], "dtans ms", round(d["ms_per_step"],4), json.dumps(d.get("cusparse_formats"))[:600])'
timeout 600 python bench.py --scale 0.25 --steps 20 --no-cpu-baseline --no-device-encode 2>&1 | python -c "$show"
timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-device-encode 2>&1 | python -c "$show"
timeout 900 python bench.py --config banded27 --steps 20 --no-cpu-baseline --no-device-encode 2>&1 | python -c "$show"
timeout 900 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline --no-device-encode 2>&1 | python -c "$show"
