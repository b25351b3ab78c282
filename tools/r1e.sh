python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "--config rmat --scale 0.125 --reorder" "--config banded27 --scale 0.25" ""; do
  n=$(echo "$c" | tr -d ' -' | cut -c1-20)
  ncu --set full --clock-control none --import-source on -k regex:dtans_kernel -s 5 -c 1 -o gpurun_out/e_$n python bench.py $c --steps 3 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2>&1
done
python bench.py --config rmat --reorder --steps 20 --no-cpu-baseline > gpurun_out/e_rmat_full.json 2>&1
tail -c 1200 gpurun_out/e_rmat_full.json
ls gpurun_out
