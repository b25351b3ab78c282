python -m pytest tests -m gpu -x -q 2>&1 | tail -3
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["workload"][:30], d["config"]["row_order"][:8], "ms", round(d["ms_per_step"],4), "GF", round(d["value"],1), "frac", round(d["roofline"]["frac"],3), "cus", (d.get("cusparse_csr") or {}).get("ms"), d["gpu_launches"])'
python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline --no-cusparse 2>&1 | tail -1 | python -c "$summ"
python bench.py --config rmat --steps 20 --no-cpu-baseline --no-cusparse 2>&1 | tail -1 | python -c "$summ"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_rmat2.csv python bench.py --config rmat --reorder --steps 5 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
python - <<'PY'
import csv, collections
for f in ["gpurun_out/launches_rmat2.csv"]:
    rows=[r for r in csv.reader(open(f)) if len(r)>5]
    h=rows[0]; i=h.index("Kernel Name"); v=h.index("Metric Value")
    agg=collections.defaultdict(lambda:[0,0.0])
    for r in rows[1:]:
        agg[r[i][:70]][0]+=1; agg[r[i][:70]][1]+=float(r[v].replace(",",""))
    for k,(n,t) in sorted(agg.items(), key=lambda t:-t[1][1])[:6]: print(f"  {n:4d} {t/n/1e3:9.1f} us  {k}")
PY
