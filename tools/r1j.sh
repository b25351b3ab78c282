for v in "DTANS_TASK_GMEM=1" "DTANS_CHUNK=8" "DTANS_LONG_SEG=100000" ; do
echo "== $v"; env $v python bench.py --config rmat --reorder --steps 5 --no-cpu-baseline --no-cusparse 2> gpurun_out/j.err | tail -c 200; tail -1 gpurun_out/j.err; done
