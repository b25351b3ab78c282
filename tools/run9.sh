cd /root/repo
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "long or rmat or task or reorder or multichunk or power or shard or upload" > gpurun_out/r9_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r9_tests.txt
tail -5 gpurun_out/r9_tests.txt
bash tools/abv.sh ab9 "r1s base pa1 pa2" "--config laplacian;--config banded27;--config rmat --reorder;--config rmat" 2
