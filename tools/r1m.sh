for v in "" "" "DTANS_LIB=paper_2603_01915_b200/exp/libdtans_f.so" "DTANS_LIB=paper_2603_01915_b200/exp/libdtans_wc.so"; do
echo "== $v"; env $v python bench.py --config rmat --reorder --steps 5 --no-cpu-baseline --no-cusparse 2> gpurun_out/m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"; tail -1 gpurun_out/m.err; done
