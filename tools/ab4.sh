cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_empty.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
  for C in "--config rmat --reorder" "--config rmat"; do
  bash tools/ab_mix.sh 2 "$C" "e0:-:DTANS_EMPTY=0" "e1:-:DTANS_EMPTY=1" "e1c25:-:DTANS_TASK_CARVE=25" "e1c50:-:DTANS_TASK_CARVE=50" "e1c100:-:DTANS_TASK_CARVE=100"
  done
  timeout 900 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --check 2>&1 | tail -1 | cut -c1-800
  timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
) > gpurun_out/ab4.txt 2>&1
cat gpurun_out/ab4.txt
