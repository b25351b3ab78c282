cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r24_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r24_tests.txt
grep -E "FAILED|passed|failed" gpurun_out/r24_tests.txt | tail -8
for E in "DTANS_GPU_WALK=1" "DTANS_GPU_WALK=0"; do
  for A in "--config rmat --reorder" "--config rmat"; do
    echo "$E $A $(env $E timeout 900 python tools/kbench.py $A --check 2>&1 | tail -1 | cut -c90-330)"
  done
done
timeout 300 python bench.py --config config1 --steps 50 --no-cpu-baseline > gpurun_out/r24_c1.json 2>&1; python tools/summarize_line.py gpurun_out/r24_c1.json
