cd /root/repo
for r in 1 2; do for v in sc1 sc0; do
  echo "$v $(DTANS_LIB=$PWD/variants/$v/libdtans.so timeout 900 python bench.py --config powerit --steps 30 --no-device-encode 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["parity"]["ok"], d["lambda"])')"
done; done
