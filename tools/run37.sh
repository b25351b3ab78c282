cd /root/repo
for r in 1 2; do
for E in "" "--env DTANS_CHUNK=8" "--env DTANS_CHUNK=12" "--env DTANS_CHUNK=24"; do
  echo "$E $(timeout 900 python tools/kbench.py --config rmat --reorder --cache /tmp/kbc $E 2>&1 | tail -1 | cut -c90-260)"
done; done
