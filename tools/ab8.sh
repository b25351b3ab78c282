cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( for C in "--config rmat --reorder" "--config rmat"; do
    bash tools/ab_mix.sh 2 "$C" "base:base:" "xdep1:xdep1:" "xdep2:xdep2:" "ror:ror:" "rx1:rx1:"
  done
  for C in "--config laplacian" "--config banded27"; do
    bash tools/ab_mix.sh 2 "$C" "base:base:" "xdep2:xdep2:" "ror:ror:"
  done
) > gpurun_out/ab8.txt 2>&1
cat gpurun_out/ab8.txt
