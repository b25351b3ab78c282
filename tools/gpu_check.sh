#!/bin/bash
# Quick GPU round: parity tests + the two headline benches, one line each.
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:30], "ms", round(d["ms_per_step"],4), "GF", round(d["value"],1), "frac", round(d["roofline"]["frac"],3), "cus", (d.get("cusparse_csr") or {}).get("ms"))'
python bench.py --no-cpu-baseline --no-cusparse "$@" 2>/dev/null | python -c "$summ"
python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse "$@" 2>/dev/null | python -c "$summ"
python bench.py --config rmat --scale 0.125 --steps 20 --no-cpu-baseline --no-cusparse "$@" 2>/dev/null | python -c "$summ"
python bench.py --config rmat --scale 0.125 --steps 20 --reorder --no-cpu-baseline --no-cusparse "$@" 2>/dev/null | python -c "$summ"
