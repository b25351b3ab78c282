cd /root/repo
for S in 0.05 0.1 0.2 0.3536; do
  echo "S=$S $(timeout 600 python tools/kbench.py --config laplacian --scale $S 2>&1 | tail -1 | cut -c1-200)"
done
for S in 0.05 0.2; do
  echo "S=$S W8 $(timeout 600 python tools/kbench.py --config laplacian --scale $S --env DTANS_WARPS=8 2>&1 | tail -1 | cut -c1-200)"
done
