ncu --set full --clock-control none --import-source on -k regex:"dtans_task_kernel" -s 2 -c 1 -o gpurun_out/z_task python bench.py --config rmat --reorder --steps 2 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
ls gpurun_out | grep z_
