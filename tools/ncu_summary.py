#!/usr/bin/env python
"""Summarise ncu output for profiles/: a `--set full` report (.ncu-rep) and/or a launch
list (`--metrics gpu__time_duration.sum --csv`).  Usage:

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu pipe %"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occ lim regs"),
    ("launch__occupancy_limit_shared_mem", "occ lim smem"),
]


def rep_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append(f"### {d.get('Kernel Name', '?')}")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k, name in KEYS:
            if k in d:
                out.append(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        st = {k.split("stalled_")[1]: float(d[k]) for k in hdr
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
              and d.get(k) not in ("", "n/a", None)}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        out.append(f"| top stall reasons (pc sampling) | {', '.join(f'{k} {v / tot:.0%}' for k, v in top)} |")
        out.append("")
    return "\n".join(out)


def launches_summary(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        ns = float(r["Metric Value"])
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for k, v in agg.items() if "fp8lm" in k or k.startswith("k_")) or 1.0
    out = ["| kernel | launches | total us | avg us | share of our kernels |", "|---|---|---|---|---|"]
    for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        ours = "fp8lm" in k or k.startswith("k_")
        out.append(f"| {k} | {n} | {ns / 1e3:.1f} | {ns / n / 1e3:.1f} | {ns / tot:.1%} |" if ours
                   else f"| {k} (not ours) | {n} | {ns / 1e3:.1f} | {ns / n / 1e3:.1f} | - |")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.launches:
        print("## Launch list (ncu gpu__time_duration, cold-cache, serialised)\n")
        print(launches_summary(a.launches))
        print()
    if a.rep:
        print("## ncu --set full\n")
        print(rep_summary(a.rep))
