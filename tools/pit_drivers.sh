#!/bin/bash
# Power iteration (config 5 shape, 1 GPU): torch-driven loop vs the C-ABI NCCL driver.
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["config"]["driver"], "ms/iter", round(d["ms_per_step"],4), "GF", round(d["value"],1), "lambda", d["lambda"])'
for drv in torch capi; do
  python bench.py --config powerit --steps 50 --driver $drv 2>/dev/null | python -c "$summ"
done
