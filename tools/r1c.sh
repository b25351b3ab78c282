python -m pytest tests -m gpu -x -q 2>&1 | tail -15
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:30], "ms", round(d["ms_per_step"],4), "GF", round(d["value"],1), "frac", round(d["roofline"]["frac"],3), "cus", (d.get("cusparse_csr") or {}).get("ms"), d["config"]["launch"])'
python bench.py --no-cpu-baseline --no-cusparse --steps 100 2>&1 | tail -1 | python -c "$summ"
DTANS_RING=2 python bench.py --no-cpu-baseline --no-cusparse --steps 100 2>&1 | tail -1 | python -c "$summ"
python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse 2>&1 | tail -1 | python -c "$summ"
python bench.py --config rmat --scale 0.125 --reorder --steps 20 --no-cpu-baseline --no-cusparse 2>&1 | tail -1 | python -c "$summ"
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/full_lap3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
