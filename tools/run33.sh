cd /root/repo
bash tools/abv.sh ab33 "med0 med1" "--config rmat --reorder;--config rmat;--config laplacian;--config banded27" 2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r33_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r33_tests.txt
grep -E "FAILED|passed|failed" gpurun_out/r33_tests.txt | tail -6
timeout 1500 python bench.py --config rmat --steps 20 > gpurun_out/r2f_rmat.json 2> gpurun_out/r2f_rmat.err; echo "rmat rc=$?"
python tools/summarize_line.py gpurun_out/r2f_rmat.json
python -c "
import json; d=json.loads(open('gpurun_out/r2f_rmat.json').read().strip().splitlines()[-1]); print(json.dumps(d.get('reference_python'))[:600]); print(json.dumps(d.get('cpu_baseline')))"
