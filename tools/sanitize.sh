#!/bin/bash
# compute-sanitizer on small shapes (memcheck, racecheck, synccheck); logs in gpurun_out/.
cd "$(dirname "$0")/.."
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --target-processes all --print-limit 20 --num-cuda-barriers 65536 python tools/sanitize_case.py > gpurun_out/san_$T.txt 2>&1
  echo "$T rc=$?"; tail -4 gpurun_out/san_$T.txt
done
