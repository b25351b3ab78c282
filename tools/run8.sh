cd /root/repo
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "long or rmat or task or reorder or multichunk or power or shard" > gpurun_out/r8_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r8_tests.txt
tail -5 gpurun_out/r8_tests.txt
for E in "" "DTANS_CHUNK=32" "DTANS_CHUNK=64" "DTANS_STAGED=1 DTANS_DYNAMIC=0"; do
  for A in "--config rmat --reorder" "--config rmat"; do
    echo "$E $A"; env $E timeout 900 python tools/kbench.py $A --cache /tmp/kbc 2>&1 | tail -1 | cut -c1-420
  done
done
