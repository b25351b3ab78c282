cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( bash tools/ab_mix.sh 3 "--config rmat --reorder" "r1:-:" "tka:tka:" "r0:r0:"
  bash tools/ab_mix.sh 2 "--config rmat" "r1:-:" "tka:tka:" "r0:r0:"
  bash tools/ab_mix.sh 2 "--config laplacian" "r1:-:" "r0:r0:"
  bash tools/ab_mix.sh 2 "--config banded27" "r1:-:" "r0:r0:"
  DTANS_LIB=$PWD/variants/tka/libdtans.so timeout 900 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --check 2>&1 | tail -1 | cut -c1-900
  DTANS_LIB=$PWD/variants/tka/libdtans.so timeout 1800 python -m pytest tests/test_gpu.py tests/test_gpu_empty.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
) > gpurun_out/ab9.txt 2>&1
cat gpurun_out/ab9.txt
