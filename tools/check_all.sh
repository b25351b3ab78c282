#!/bin/bash
# Full -m gpu suite, the default bench line, and kbench checks of the other configs.
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ca_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/ca_tests.txt
tail -3 gpurun_out/ca_tests.txt
timeout 900 python bench.py > gpurun_out/ca_bench.json 2> gpurun_out/ca_bench.err; echo "bench rc=$?"
python tools/summarize_line.py gpurun_out/ca_bench.json
for A in "--config banded27" "--config banded32 --noy" "--config rmat --reorder" "--config rmat"; do
  timeout 900 python tools/kbench.py $A --check 2>&1 | tail -1 | cut -c1-330
done
