cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline > gpurun_out/r2h_rmat_sorted.json 2> gpurun_out/r2h_rmat_sorted.err; echo "rc=$?"
python tools/summarize_line.py gpurun_out/r2h_rmat_sorted.json
tail -3 gpurun_out/r2h_rmat_sorted.err
