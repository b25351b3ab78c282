cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( for C in "--config rmat --reorder" "--config rmat"; do
  bash tools/ab_mix.sh 3 "$C" "pdl0:-:DTANS_PDL=0" "pdl2:-:DTANS_PDL=2" "solo1:-:DTANS_PDL=2,DTANS_SOLO_FIRST=1" "carve25:-:DTANS_PDL=2,DTANS_TASK_CARVE=25" "carve0:-:DTANS_PDL=2,DTANS_TASK_CARVE=0"
  done
  timeout 900 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --check --env DTANS_PDL=2 --env DTANS_SOLO_FIRST=1 --env DTANS_VERBOSE=1 2>&1 | tail -3 | cut -c1-600
  timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
) > gpurun_out/ab3.txt 2>&1
cat gpurun_out/ab3.txt
