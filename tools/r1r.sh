python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --config powerit --steps 20 > gpurun_out/pit.json 2> gpurun_out/pit.err; tail -2 gpurun_out/pit.err; python -c "import json; d=json.load(open('gpurun_out/pit.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['lambda'])"
