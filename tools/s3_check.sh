cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/s3_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/s3_tests.txt
tail -3 gpurun_out/s3_tests.txt
timeout 600 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo "bench rc=$?"
python tools/summarize_line.py gpurun_out/s3_bench.json
for A in "--config rmat --reorder" ; do
  timeout 900 python tools/kbench.py $A --cache /tmp/kcache 2>&1 | tail -1 | cut -c1-400
done
