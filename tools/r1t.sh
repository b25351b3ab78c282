python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" "DTANS_CHUNK=8" "DTANS_CHUNK=32"; do
echo "== $v"; env $v python bench.py --config rmat --reorder --steps 10 --no-cpu-baseline --no-cusparse 2> gpurun_out/m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>/dev/null; tail -1 gpurun_out/m.err; done
