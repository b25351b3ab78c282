cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r23_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r23_tests.txt
tail -4 gpurun_out/r23_tests.txt
timeout 600 python bench.py --config config1 --steps 50 > gpurun_out/r23_c1.json 2> gpurun_out/r23_c1.err; python tools/summarize_line.py gpurun_out/r23_c1.json
python -c "
import json; d=json.loads(open('gpurun_out/r23_c1.json').read().strip().splitlines()[-1]); print(d['details']['plan'], d['details']['launch']); print(json.dumps(d['cusparse_formats'])[:400])"
bash tools/multirank_check.sh 2>&1 | tail -8
