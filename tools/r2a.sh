python -m pytest tests/test_gpu.py -x -q -k "rmat or long" 2>&1 | tail -1
for v in "" "DTANS_RING=1" "DTANS_RING=1 DTANS_CHUNK=8" "DTANS_RING=3"; do
echo "== $v"; env $v DTANS_VERBOSE=1 python bench.py --config rmat --reorder --steps 10 --no-cpu-baseline --no-cusparse 2> gpurun_out/m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>/dev/null; grep "dtans\]" gpurun_out/m.err | tail -1 | cut -c40-250; tail -1 gpurun_out/m.err | cut -c1-200; done
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:30], "ms", round(d["ms_per_step"],4), "GF", round(d["value"],1), "frac", round(d["roofline"]["frac"],3))'
DTANS_RING=1 python bench.py --no-cpu-baseline --no-cusparse --steps 100 2>&1 | tail -1 | python -c "$summ"
DTANS_RING=1 python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse 2>&1 | tail -1 | python -c "$summ"
