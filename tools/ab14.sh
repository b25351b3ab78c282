cd $GRAFT_REPO_ROOT
echo "== old"; DTANS_LIB=$PWD/variants/old/libdtans.so python tools/dropin_probe.py 2>&1 | tail -6
echo "== new"; python tools/dropin_probe.py 2>&1 | tail -6
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_parity.py tests/test_gpu_empty.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
