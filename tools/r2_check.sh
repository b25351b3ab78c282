#!/bin/bash
# Round-2 GPU check: all -m gpu tests, then the default bench line.
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?"
tail -3 gpurun_out/r2_tests.txt
