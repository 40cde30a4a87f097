"""One-line summary of bench.py JSON lines: python tools/bl.py file.jsonl ..."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if "ms_per_step" not in d:
            continue
        r = d.get("roofline") or {}
        k = {n: round(v["ms_per_step"], 4) for n, v in (d.get("kernels") or {}).items()}
        print(f, d["n_gpus"], round(d["ms_per_step"], 4), round(d["value"]), r.get("kernel"),
              round(r.get("frac", 0), 3), (d.get("clocks") or {}).get("sm_mhz"), k)
