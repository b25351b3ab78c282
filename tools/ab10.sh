cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( bash tools/ab_mix.sh 3 "--config rmat --reorder" "elast:-:" "efirst:efirst:"
  bash tools/ab_mix.sh 2 "--config rmat" "elast:-:" "efirst:efirst:"
  timeout 900 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --check 2>&1 | tail -1 | cut -c1-900
  timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
) > gpurun_out/ab10.txt 2>&1
cat gpurun_out/ab10.txt
