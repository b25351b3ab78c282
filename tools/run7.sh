cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r7_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r7_tests.txt
tail -15 gpurun_out/r7_tests.txt
for A in "--config rmat --reorder" "--config rmat" "--config laplacian" "--config banded27"; do
  timeout 900 python tools/kbench.py $A --cache /tmp/kbc --check 2>&1 | tail -1
  DTANS_STAGED=0 timeout 900 python tools/kbench.py $A --cache /tmp/kbc 2>&1 | tail -1
done
