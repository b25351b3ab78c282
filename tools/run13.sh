cd /root/repo
bash tools/abv.sh ab13 "cur emb" "--config laplacian;--config banded27;--config banded32 --noy;--config rmat --reorder" 2
timeout 900 compute-sanitizer --tool synccheck --target-processes all --print-limit 20 --num-cuda-barriers 65536 python tools/sanitize_case.py > gpurun_out/san_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san_synccheck.txt
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "parity or host_buffer or golden or larger" > gpurun_out/r13_tests.txt 2>&1; tail -2 gpurun_out/r13_tests.txt
