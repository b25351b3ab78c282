set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_lap.json 2> gpurun_out/bench_lap.err; tail -c 3000 gpurun_out/bench_lap.json
python bench.py --config banded27 --steps 50 --no-cpu-baseline > gpurun_out/bench_b27.json 2>&1; tail -c 1500 gpurun_out/bench_b27.json
python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline > gpurun_out/bench_rmat_r.json 2>&1; tail -c 1500 gpurun_out/bench_rmat_r.json
python bench.py --config rmat --steps 20 --no-cpu-baseline --no-cusparse > gpurun_out/bench_rmat.json 2>&1; tail -c 600 gpurun_out/bench_rmat.json
python bench.py --config powerit --steps 20 > gpurun_out/bench_pit.json 2>&1; tail -c 800 gpurun_out/bench_pit.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_lap.csv python bench.py --steps 20 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/full_lap python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/full_b27 python bench.py --config banded27 --scale 0.25 --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
ls -la gpurun_out
