#!/usr/bin/env python
"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of our kernels
from one `ncu --set full` capture, averaged over the captured launches of each kernel,
merged into profiles/<round>/ncu_traffic.json under the workload key; bench.py reports
it as roofline.traffic for the dominant kernel of the same workload.

    python tools/ncu_traffic.py gpurun_out/m1/full.ncu-rep --workload gpt-125m \
        --out profiles/r1/ncu_traffic.json
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

# ncu kernel name -> bench.py / fp8lm_prof name
NAMES = [
    (r"^void k_amax<", "amax"),
    (r"^void k_quantize<", "quantize"),
    (r"^void k_adam<1,", "adam_pass1"),
    (r"^void k_adam<2,", "adam_pass2"),
    (r"^void k_adam<3,", "quantize+adam_pass1"),
    (r"^void k_adam<4,", "adam_delayed"),
    (r"^void k_adam<5,", "quantize+adam_delayed"),
    (r"^void k_reduce_p2p_a1<", "reduce_p2p"),
    (r"^void k_reduce_p2p<", "reduce_p2p"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    acc = collections.defaultdict(list)
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = next((n for pat, n in NAMES if re.match(pat, d.get("Kernel Name", ""))), None)
        if name is None:
            continue
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[k].replace(",", "")) * SCALE.get(u[k], 1)
        acc[name].append(b)
    data = json.load(open(args.out)) if os.path.exists(args.out) else {}
    wl = data.setdefault(args.workload, {})
    for name, v in acc.items():
        wl[name] = {"dram_bytes_per_launch": sum(v) / len(v), "launches_captured": len(v),
                    "source": os.path.basename(args.rep)}
    json.dump(data, open(args.out, "w"), indent=1, sort_keys=True)
    print(json.dumps(wl, indent=1))


if __name__ == "__main__":
    main()
