cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
timeout 1200 python bench.py --config rmat --steps 20 > gpurun_out/r2j_rmat.json 2> gpurun_out/r2j_rmat.err; echo "rc=$?"
python tools/summarize_line.py gpurun_out/r2j_rmat.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
