python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "--reorder sym" "--reorder"; do
echo "== $v"; python bench.py --config rmat $v --steps 20 --no-cpu-baseline 2> gpurun_out/m.err > gpurun_out/m.json; python -c "import json; d=json.load(open('gpurun_out/m.json')); print(d['ms_per_step'], d['value'], d['config']['container_bytes'], d['config']['compression_vs_min_csr_coo_sell'], d['cusparse_csr']['ms'], d['e2e']['value'])"; tail -1 gpurun_out/m.err | cut -c1-200; done
