cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/final_r2b.sh > gpurun_out/r2g_summary.txt 2>&1
bash tools/profile_r2.sh lap > gpurun_out/r2g_prof_lap.log 2>&1
bash tools/profile_r2b.sh > gpurun_out/r2g_prof_rmat.log 2>&1
cat gpurun_out/r2g_summary.txt
