cd $GRAFT_REPO_ROOT
for cfg in laplacian banded27; do
  echo "== old"; DTANS_LIB=$PWD/variants/old/libdtans.so PROBE_STAGES="8" python tools/e2e_probe.py $cfg
  echo "== new"; PROBE_STAGES="6 8 10 12" python tools/e2e_probe.py $cfg
done
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -p no:cacheprovider -k "host" 2>&1 | tail -2
