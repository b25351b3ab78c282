cd /root/repo
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "long or rmat or task or reorder or power or upload" > gpurun_out/r10_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r10_tests.txt
tail -3 gpurun_out/r10_tests.txt
for E in "DTANS_TASK_WIN=0" "DTANS_TASK_WIN=1" "DTANS_TASK_WIN=1 DTANS_CHUNK=32" "DTANS_TASK_WIN=0 DTANS_CHUNK=32" "DTANS_STAGED=1"; do
  for A in "--config rmat --reorder" "--config rmat"; do
    echo "$E $A"; env $E timeout 900 python tools/kbench.py $A --cache /tmp/kbc 2>&1 | tail -1 | cut -c1-300
  done
done
