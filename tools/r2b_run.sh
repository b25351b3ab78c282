cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/profile_r2b.sh > gpurun_out/r2b_prof.log 2>&1
timeout 1200 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline > gpurun_out/r2b_rmat_sorted.json 2> gpurun_out/r2b_rmat_sorted.err; echo "rc=$?"
python tools/summarize_line.py gpurun_out/r2b_rmat_sorted.json
timeout 1200 python bench.py --config rmat --steps 20 > gpurun_out/r2b_rmat.json 2> gpurun_out/r2b_rmat.err; echo "rc=$?"
python tools/summarize_line.py gpurun_out/r2b_rmat.json
