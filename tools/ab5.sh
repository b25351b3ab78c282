cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( bash tools/ab_mix.sh 2 "--config rmat --reorder" "c16:-:" "c8:-:DTANS_CHUNK=8" "c12:-:DTANS_CHUNK=12" "c24:-:DTANS_CHUNK=24" "c32:-:DTANS_CHUNK=32"
  bash tools/ab_mix.sh 2 "--config rmat" "c16:-:" "c32:-:DTANS_CHUNK=32" "ls32:-:DTANS_LONG_SEG=32" "ls96:-:DTANS_LONG_SEG=96" "ls127:-:DTANS_LONG_SEG=127"
) > gpurun_out/ab5.txt 2>&1
cat gpurun_out/ab5.txt
