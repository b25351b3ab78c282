#!/bin/bash
# End-of-session check on one GPU: the -m gpu suite, smoke(), the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fc_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/fc_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fc_smoke.txt
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo "bench rc=$?"
python tools/summarize_line.py gpurun_out/fc_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fc_ref.json 2> gpurun_out/fc_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/fc_ref.json
