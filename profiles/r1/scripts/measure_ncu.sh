#!/bin/bash
# ncu evidence for profiles/r1: launch list of our kernels (k_*) and --set full captures
# (JIT and delayed), each after the same command exited 0 without ncu.
set -u
O=gpurun_out/m2
mkdir -p $O
python bench.py --quick --steps 2 --warmup 3 > $O/quick.jsonl 2>&1; echo "quick rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file $O/launches.csv \
    python bench.py --quick --steps 2 --warmup 3 > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
python bench.py --quick --steps 2 --warmup 3 --state-scaling delayed > $O/quick_d.jsonl 2>&1; echo "quick_d rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file $O/launches_delayed.csv \
    python bench.py --quick --steps 2 --warmup 3 --state-scaling delayed > $O/ncu_launches_d.log 2>&1; echo "launches_d rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_adam|k_amax" -c 6 -o $O/full_delayed \
    python bench.py --quick --steps 2 --warmup 3 --state-scaling delayed > $O/ncu_full_d.log 2>&1; echo "full_d rc=$?"
