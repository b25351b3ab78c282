#!/bin/bash
# Interleaved A/B of a plan knob: tools/ab_env.sh "KNOB=a" "KNOB=b" [rounds] -- kbench args...
# prints warm/cold ms per round for each setting
cd "$(dirname "$0")/.."
A=$1; B=$2; R=${3:-3}; shift 3; [ "$1" = "--" ] && shift
for i in $(seq 1 $R); do
  for E in "$A" "$B"; do
    timeout 900 python tools/kbench.py "$@" --cache /tmp/kcache --env "$E" 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$E', d['config'], d['reorder'], d['warm_ms'], d['cold_ms'])" || echo "$E failed"
  done
done
