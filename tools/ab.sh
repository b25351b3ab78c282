#!/bin/bash
# Quick A/B on one GPU: kbench timings (+ oracle check) of the headline
# configs, then a -m gpu test subset.  Usage: tools/ab.sh TAG [pytest -k expr]
cd "$(dirname "$0")/.."
TAG=${1:-ab}
for A in "--config laplacian" "--config banded27" "--config banded32 --noy" "--config rmat --reorder" "--config rmat"; do
  timeout 600 python tools/kbench.py $A --check 2>&1 | tail -1 | tee -a gpurun_out/${TAG}_kb.txt
done
if [ -n "$2" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$2" 2>&1 | tail -3 | tee gpurun_out/${TAG}_tests.txt
fi
