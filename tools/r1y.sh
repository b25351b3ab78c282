summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:30], "ms", round(d["ms_per_step"],4), "GF", round(d["value"],1), "frac", round(d["roofline"]["frac"],3))'
for v in "" "DTANS_LIB=paper_2603_01915_b200/exp/libdtans_w28.so" "DTANS_LIB=paper_2603_01915_b200/exp/libdtans_w24.so"; do
echo "== $v"
env $v python bench.py --no-cpu-baseline --no-cusparse --steps 100 2>&1 | tail -1 | python -c "$summ"
env $v python bench.py --config banded27 --scale 0.25 --steps 50 --no-cpu-baseline --no-cusparse 2>&1 | tail -1 | python -c "$summ"
env $v python bench.py --config rmat --reorder --steps 10 --no-cpu-baseline --no-cusparse 2>&1 | tail -1 | python -c "$summ"
done
