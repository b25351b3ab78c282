#!/bin/bash
# Interleaved A/B over (variant, env) arms: tools/ab_mix.sh ROUNDS "kbench args" "label:variant:K=V,K=V" ...
# variant "-" = the in-tree libdtans.so; prints warm/cold ms per arm and round.
cd "$(dirname "$0")/.."
R=$1; ARGS=$2; shift 2
for i in $(seq 1 $R); do
  for arm in "$@"; do
    IFS=: read -r lab var envs <<< "$arm"
    E=(); [ -n "$envs" ] && for kv in ${envs//,/ }; do E+=(--env "$kv"); done
    L=""; [ "$var" != "-" ] && L="DTANS_LIB=$PWD/variants/$var/libdtans.so"
    env $L timeout 900 python tools/kbench.py $ARGS --cache /tmp/kcache "${E[@]}" 2>&1 | tail -1 | python -c "import sys,json
try:
  d=json.loads(sys.stdin.read()); print('%-12s %-28s warm %.5f cold %.5f' % ('$lab', '$ARGS', d['warm_ms'], d['cold_ms']))
except Exception as e: print('$lab failed', e)"
  done
done
