cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/ab_mix.sh 3 "--config rmat --reorder" "nobatch:old:" "pair:-:"
bash tools/ab_mix.sh 2 "--config rmat" "nobatch:old:" "pair:-:"
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 1200 python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline > gpurun_out/r2i_rmat_sorted.json 2> gpurun_out/r2i_rmat_sorted.err; echo "rc=$?"
python tools/summarize_line.py gpurun_out/r2i_rmat_sorted.json
