cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( bash tools/ab_mix.sh 2 "--config rmat --reorder" "def32:-:" "c16:-:DTANS_CHUNK=16" "c48:-:DTANS_CHUNK=48" "c64:-:DTANS_CHUNK=64"
  timeout 900 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --check 2>&1 | tail -1 | cut -c1-900
  bash tools/prof_task_src.sh
  timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
) > gpurun_out/ab7.txt 2>&1
cat gpurun_out/ab7.txt
