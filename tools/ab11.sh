cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( timeout 600 python tools/sanitize_case.py 2>&1 | tail -3 | cut -c1-300
  bash tools/ab_mix.sh 2 "--config rmat" "dyn_auto:-:" "dyn0:-:DTANS_DYNAMIC=0" "dyn0k4:-:DTANS_DYNAMIC=0,DTANS_KCHUNK=4"
) > gpurun_out/ab11.txt 2>&1
cat gpurun_out/ab11.txt
