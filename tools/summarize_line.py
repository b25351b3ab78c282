"""One-line summary of a bench.py JSON line (for gpurun tails)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    cf = d.get("cusparse_formats") or {}
    print(" ms %.4f GF %.1f frac %.3f parity %s best_cus %s %s e2e %s clocks %s" % (
        d.get("ms_per_step", 0), d.get("value", 0), (d.get("roofline") or {}).get("frac", 0),
        (d.get("parity") or {}).get("ok"), cf.get("best_format"), cf.get("best_ms"),
        (d.get("e2e") or {}).get("value"), d.get("clocks")))
