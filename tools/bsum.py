"""One-line summaries of bench JSON files: tools/bsum.py f1.json f2.json ..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", e); continue
    r = d.get("roofline", {}).get("kernels", {})
    ks = {k: round(v["kernel_ms"], 4) if isinstance(v, dict) else round(v, 4) for k, v in r.items()}
    print(f, round(d["ms_per_step"], 4), "%.1fM/s" % (d["value"] / 1e6), ks, d.get("clocks", {}).get("sm_mhz"))
