cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( bash tools/ab_env.sh DTANS_PDL=0 DTANS_PDL=1 3 -- --config rmat --reorder
  bash tools/ab_env.sh DTANS_PDL=0 DTANS_PDL=1 2 -- --config rmat
  bash tools/ab_env.sh DTANS_PDL=0 DTANS_PDL=1 2 -- --config laplacian
  timeout 600 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --check | tail -1 | cut -c1-300
) > gpurun_out/ab1.txt 2>&1
cat gpurun_out/ab1.txt
