ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_rmat.csv python bench.py --config rmat --reorder --steps 10 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_rmat_nat.csv python bench.py --config rmat --steps 10 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
python - <<'PY'
import csv, collections
for f in ["gpurun_out/launches_rmat.csv", "gpurun_out/launches_rmat_nat.csv"]:
    rows=[r for r in csv.reader(open(f)) if len(r)>5]
    h=rows[0]; i=h.index("Kernel Name"); v=h.index("Metric Value")
    agg=collections.defaultdict(lambda:[0,0.0])
    for r in rows[1:]:
        agg[r[i][:70]][0]+=1; agg[r[i][:70]][1]+=float(r[v].replace(",",""))
    print(f)
    for k,(n,t) in sorted(agg.items(), key=lambda t:-t[1][1])[:8]: print(f"  {n:4d} {t/n/1e3:9.1f} us  {k}")
PY
