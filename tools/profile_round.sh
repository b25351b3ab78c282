# Round profiling pass (one GPU): launch lists + one full capture per headline config.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/pr_launches_lap.csv python bench.py --steps 20 --no-cpu-baseline --no-device-encode > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/pr_full_lap python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse --no-device-encode > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/pr_launches_b27.csv python bench.py --config banded27 --steps 10 --no-cpu-baseline --no-device-encode > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/pr_full_b27 python bench.py --config banded27 --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse --no-device-encode > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/pr_launches_rmat.csv python bench.py --config rmat --reorder --steps 10 --no-cpu-baseline --no-device-encode > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/pr_full_rmat python bench.py --config rmat --reorder --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse --no-device-encode > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/pr_launches_pit.csv python bench.py --config powerit --steps 10 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out
