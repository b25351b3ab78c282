#!/bin/bash
# Round-end style check on one GPU: smoke, the full -m gpu suite, the default bench line.
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python -m pytest tests -m gpu -q 2>&1 | tail -2
python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; tail -c 2000 gpurun_out/fc_bench.json
python bench.py --impl reference > gpurun_out/fc_ref.json 2> gpurun_out/fc_ref.err; tail -c 600 gpurun_out/fc_ref.json
