cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( for C in "--config laplacian" "--config banded27" "--config banded32 --noy" "--config rmat" "--config laplacian --scale 0.125"; do
    bash tools/ab_mix.sh 3 "$C" "pm0:-:DTANS_PDL_MAIN=0" "pm1:-:DTANS_PDL_MAIN=1"
  done
  bash tools/ab_mix.sh 2 "--config rmat --reorder" "c16:-:" "c8:-:DTANS_CHUNK=8" "c12:-:DTANS_CHUNK=12" "c24:-:DTANS_CHUNK=24" "c32:-:DTANS_CHUNK=32"
  bash tools/ab_mix.sh 2 "--config rmat" "c16:-:" "c32:-:DTANS_CHUNK=32" "ls32:-:DTANS_LONG_SEG=32" "ls96:-:DTANS_LONG_SEG=96"
  timeout 1200 python -m pytest tests/test_gpu.py -m gpu -q -x -p no:cacheprovider -k "power or long or reorder" 2>&1 | tail -2
) > gpurun_out/ab6.txt 2>&1
cat gpurun_out/ab6.txt
