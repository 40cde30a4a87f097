#!/bin/bash
# Single-GPU measurement set of profiles/r1 (run from the repo root on a B200 box).
set -u
O=gpurun_out/m1
mkdir -p $O
python paper_2310_18313_b200/build.py > /dev/null
python bench.py > $O/bench_n1.jsonl 2> $O/bench_n1.err; echo "bench_n1 rc=$?"
python bench.py --state-scaling delayed > $O/bench_n1_delayed.jsonl 2> $O/bench_n1_delayed.err; echo "delayed rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_n1_reference.jsonl 2> $O/ref.err; echo "ref rc=$?"
python bench.py --config gpt-7b --steps 10 --no-cpu-baseline > $O/bench_7b_n1.jsonl 2> $O/b7.err; echo "7b rc=$?"
python bench.py --config gpt-7b --steps 10 --no-cpu-baseline --state-scaling delayed > $O/bench_7b_n1_delayed.jsonl 2> $O/b7d.err; echo "7bd rc=$?"
# launch list of the same command (quick: no soak / e2e / cpu leg), then one --set full capture
python bench.py --quick --steps 2 --warmup 3 > $O/quick.jsonl 2>&1; echo "quick rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file $O/launches.csv \
    python bench.py --quick --steps 2 --warmup 3 > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_adam|k_amax" -c 8 -o $O/full \
    python bench.py --quick --steps 2 --warmup 3 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python bench.py --quick --steps 2 --warmup 3 --state-scaling delayed > $O/quick_d.jsonl 2>&1; echo "quick_d rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file $O/launches_delayed.csv \
    python bench.py --quick --steps 2 --warmup 3 --state-scaling delayed > $O/ncu_launches_d.log 2>&1; echo "ncu launches_d rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_adam|k_amax" -c 6 -o $O/full_delayed \
    python bench.py --quick --steps 2 --warmup 3 --state-scaling delayed > $O/ncu_full_d.log 2>&1; echo "ncu full_d rc=$?"
