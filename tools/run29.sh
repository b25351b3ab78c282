cd /root/repo
for S in 0.3536 0.5; do
for E in "" "--env DTANS_KCHUNK=2" "--env DTANS_KCHUNK=3" "--env DTANS_KCHUNK=5" "--env DTANS_WARPS=16" "--env DTANS_WARPS=16 --env DTANS_KCHUNK=4" "--env DTANS_WARPS=24"; do
  echo "S=$S $E $(timeout 600 python tools/kbench.py --config laplacian --scale $S $E --cache /tmp/kbc 2>&1 | tail -1 | cut -c1-260)"
done
done
