#!/bin/bash
# Round-2 second evidence pass (after the long-slice launch chain): the -m gpu suite, smoke(), and one
# line per BASELINE config (gpurun_out/r2g_*.json), then a summary.
cd "$(dirname "$0")/.."
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2g_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r2g_tests.txt
tail -2 gpurun_out/r2g_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2g_smoke.txt
run() { local tag=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/r2g_$tag.json 2> gpurun_out/r2g_$tag.err; echo "$tag rc=$?"; python tools/summarize_line.py gpurun_out/r2g_$tag.json; }
run lap
run b27 --config banded27 --steps 30
run rmat_sorted --config rmat --reorder --steps 20 --no-cpu-baseline
run rmat --config rmat --steps 20
run powerit --config powerit --steps 20
run config1 --config config1 --steps 50
run ref --impl reference --steps 3 --warmup 1
