python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" "" "" "DTANS_CHUNK=64" "DTANS_CHUNK=128"; do
echo "== $v"; env $v python bench.py --config rmat --reorder --steps 5 --no-cpu-baseline --no-cusparse 2> gpurun_out/m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>/dev/null; tail -1 gpurun_out/m.err; done
echo "== natural"; python bench.py --config rmat --steps 5 --no-cpu-baseline --no-cusparse 2> gpurun_out/m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>/dev/null; tail -1 gpurun_out/m.err
