cd $GRAFT_REPO_ROOT
bash tools/ab_mix.sh 3 "--config rmat --reorder" "tb1:-:" "tb2:tb2:"
bash tools/ab_mix.sh 2 "--config rmat" "tb1:-:" "tb2:tb2:"
DTANS_LIB=$PWD/variants/tb2/libdtans.so timeout 900 python -m pytest tests/test_gpu_empty.py tests/test_gpu.py -m gpu -q -x -p no:cacheprovider -k "chain or empty or long or reorder" 2>&1 | tail -1
