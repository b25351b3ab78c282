#!/bin/bash
# Round-2 GPU pass: every -m gpu test (no -x), then one bench line per config.
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2a_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2a_tests.txt
tail -3 gpurun_out/r2a_tests.txt
timeout 600 python bench.py --steps 50 > gpurun_out/r2a_lap.json 2> gpurun_out/r2a_lap.err
timeout 600 python bench.py --config banded27 --steps 30 --no-cpu-baseline > gpurun_out/r2a_b27.json 2> gpurun_out/r2a_b27.err
timeout 600 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline > gpurun_out/r2a_rmat_r.json 2> gpurun_out/r2a_rmat_r.err
timeout 600 python bench.py --config rmat --steps 20 --no-cpu-baseline > gpurun_out/r2a_rmat.json 2> gpurun_out/r2a_rmat.err
timeout 600 python bench.py --config powerit --steps 20 > gpurun_out/r2a_pit.json 2> gpurun_out/r2a_pit.err
timeout 300 python bench.py --config config1 --steps 50 > gpurun_out/r2a_c1.json 2> gpurun_out/r2a_c1.err
for f in gpurun_out/r2a_*.json; do echo $f; python tools/summarize_line.py $f; done
