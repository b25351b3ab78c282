cd /root/repo
bash tools/abv.sh ab31 "pre2 rs8" "--config laplacian;--config banded27;--config rmat --reorder;--config laplacian --scale 0.3536" 2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r31_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r31_tests.txt
grep -E "FAILED|passed|failed" gpurun_out/r31_tests.txt | tail -6
