cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( bash tools/ab_mix.sh 2 "--config rmat --reorder" "default:-:" "ls64c48:-:DTANS_LONG_SEG=64,DTANS_CHUNK=48" "ls32c48:-:DTANS_LONG_SEG=32,DTANS_CHUNK=48" "ls16c48:-:DTANS_LONG_SEG=16,DTANS_CHUNK=48" "ls8c48:-:DTANS_LONG_SEG=8,DTANS_CHUNK=48" "ls64c16:-:DTANS_LONG_SEG=64"
  for E in DTANS_LONG_SEG=64 DTANS_LONG_SEG=16; do timeout 600 python tools/kbench.py --config rmat --reorder --cache /tmp/kcache --env $E --env DTANS_CHUNK=48 --iters 10 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$E', d['plan'])"; done
) > gpurun_out/ab12.txt 2>&1
cat gpurun_out/ab12.txt
