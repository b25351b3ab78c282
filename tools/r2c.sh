for v in "DTANS_HOST_STAGES=8" "DTANS_HOST_STAGES=16" "DTANS_HOST_STAGES=32"; do
echo "== $v"; env $v python bench.py --steps 50 --no-cpu-baseline --no-cusparse 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e'])"; done
