python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" "DTANS_CHUNK=16" "DTANS_CHUNK=4"; do
echo "== $v"; env $v DTANS_VERBOSE=1 python bench.py --config rmat --reorder --steps 10 --no-cpu-baseline --no-cusparse 2> gpurun_out/m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>/dev/null; grep "dtans\]" gpurun_out/m.err | tail -1 | cut -c1-250; tail -1 gpurun_out/m.err | cut -c1-200; done
echo "== natural"; python bench.py --config rmat --steps 10 --no-cpu-baseline --no-cusparse 2> gpurun_out/m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>/dev/null; tail -1 gpurun_out/m.err | cut -c1-200
