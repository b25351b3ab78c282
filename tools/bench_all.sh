# All bench lines of DESIGN.md section 5 (one GPU).
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/ba_tests.txt
python bench.py > gpurun_out/ba_lap.json 2> gpurun_out/ba_lap.err
python bench.py --config banded27 --steps 50 > gpurun_out/ba_b27.json 2> gpurun_out/ba_b27.err
python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline > gpurun_out/ba_rmat_r.json 2> gpurun_out/ba_rmat_r.err
python bench.py --config rmat --steps 20 > gpurun_out/ba_rmat.json 2> gpurun_out/ba_rmat.err
python bench.py --config rmat --reorder sym --steps 20 --no-cpu-baseline > gpurun_out/ba_rmat_sym.json 2> gpurun_out/ba_rmat_sym.err
python bench.py --config powerit --steps 20 > gpurun_out/ba_pit.json 2> gpurun_out/ba_pit.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ba_ref.json 2> gpurun_out/ba_ref.err
python bench.py --config config1 --steps 50 > gpurun_out/ba_c1.json 2> gpurun_out/ba_c1.err
for f in gpurun_out/ba_*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
cus=(d.get('cusparse_csr') or {})
cpu=(d.get('cpu_baseline') or {})
print(' ms', round(d['ms_per_step'],4), 'GF', round(d['value'],1), 'frac', round((d.get('roofline') or {}).get('frac',0),3), 'cus_ms', cus.get('ms'), 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', cpu.get('value'), cpu.get('cores'), 'comp', d.get('config',{}).get('compression_vs_min_csr_coo_sell'))
"; done
