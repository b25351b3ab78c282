cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r26_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r26_tests.txt
grep -E "FAILED|passed|failed" gpurun_out/r26_tests.txt | tail -8
timeout 900 python bench.py > gpurun_out/r26_bench.json 2> gpurun_out/r26_bench.err; echo "bench rc=$?"
python tools/summarize_line.py gpurun_out/r26_bench.json
python -c "
import json; d=json.loads(open('gpurun_out/r26_bench.json').read().strip().splitlines()[-1]); print(json.dumps(d['e2e'])); print(d['details'].get('upload_s'), d['details'].get('encode_device_s'))"
