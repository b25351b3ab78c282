#!/bin/bash
# Interleaved A/B of libdtans.so variants (tools/variant.sh) on one GPU.
#   tools/abv.sh TAG "v1 v2 ..." "cfg1;cfg2;..." [rounds]
# cfg = kbench.py arguments, e.g. "--config laplacian;--config banded27".
# The first round also checks every variant against the oracle (bitwise rows).
cd "$(dirname "$0")/.."
TAG=$1; VARS=$2; CFGS=$3; R=${4:-3}
IFS=';' read -ra CL <<< "$CFGS"
OUT=gpurun_out/${TAG}_abv.txt
: > $OUT
for r in $(seq 1 $R); do
  for c in "${CL[@]}"; do
    for v in $VARS; do
      CHK=""; [ $r = 1 ] && CHK=--check
      L=$(DTANS_LIB=$PWD/variants/$v/libdtans.so timeout 900 python tools/kbench.py $c --cache /tmp/kbc $CHK --iters 100 2>&1 | tail -1)
      python - "$v" "$c" "$L" >> $OUT <<'PY'
import json, sys
v, c, l = sys.argv[1:4]
try:
    d = json.loads(l)
    b = f" bitwise {d['bitwise_rows']}/{d['rows']}" if "bitwise_rows" in d else ""
    print(f"{v:10s} {c:32s} warm {d['warm_ms']:.5f} cold {d['cold_ms']:.5f} frac {d['frac_warm']:.4f}{b}")
except Exception:
    print(f"{v:10s} {c:32s} FAILED {l[:300]}")
PY
    done
  done
done
cat $OUT
