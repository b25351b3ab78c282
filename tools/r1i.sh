python bench.py --config rmat --reorder --steps 5 --no-cpu-baseline --no-cusparse > gpurun_out/i_rmat.json 2> gpurun_out/i_rmat.err; tail -5 gpurun_out/i_rmat.err; tail -c 300 gpurun_out/i_rmat.json
ncu --set full --clock-control none --import-source on -k regex:dtans_task_kernel -s 2 -c 1 -o gpurun_out/i_task python bench.py --config rmat --reorder --steps 2 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
ls gpurun_out/
