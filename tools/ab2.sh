cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( for C in "--config rmat --reorder" "--config rmat"; do
  bash tools/ab_mix.sh 3 "$C" "base0:base:DTANS_PDL=0" "base2:base:DTANS_PDL=2" "dyn2:dyn:DTANS_PDL=2" "l2pf2:l2pf:DTANS_PDL=2" "dyn0:dyn:DTANS_PDL=0"
  done
  DTANS_LIB=$PWD/variants/dyn/libdtans.so timeout 600 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --check --env DTANS_PDL=2 | tail -1 | cut -c1-200
  DTANS_LIB=$PWD/variants/dyn/libdtans.so timeout 600 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --check --env DTANS_PDL=2 | python -c "import sys,json; d=json.loads(sys.stdin.read().splitlines()[-1]); print({k:v for k,v in d.items() if 'bit' in k or 'row' in k or 'tol' in k or 'ok' in k})"
) > gpurun_out/ab2.txt 2>&1
cat gpurun_out/ab2.txt
