ncu --set full --clock-control none --import-source on -k regex:"dtans_(task|solo)_kernel" -s 2 -c 2 -o gpurun_out/p_task python bench.py --config rmat --reorder --steps 2 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
ls gpurun_out
