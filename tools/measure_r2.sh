#!/bin/bash
# Round-2 N = 1 set on one B200: the default line (GPT-7B, C3 at N = 1) exactly as the
# driver runs it, C1, C2, one GPT-175B layer, delayed, worst case, the reference arm;
# then the ncu launch list of the default command and --set full of its kernels (each
# ncu pass only after the same command exited 0 without ncu).
set -u
O=${O:-gpurun_out/r2}
mkdir -p $O
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/$name.jsonl 2> $O/$name.err; echo "$name rc=$?"; python tools/bl.py $O/$name.jsonl; }
run bench_7b_n1 --gpus 1 --steps 20 --warmup 5
run bench_c1 --config c1 --steps 200 --warmup 5
run bench_125m --config gpt-125m --steps 100 --warmup 5
run bench_175b_layer --config gpt-175b-layer --steps 20 --warmup 5
run bench_7b_n1_delayed --steps 20 --warmup 5 --state-scaling delayed --no-e2e --no-cpu-baseline
run bench_7b_n1_worst --steps 20 --warmup 5 --worst-case --no-e2e --no-cpu-baseline
run bench_7b_n1_bf16 --steps 20 --warmup 5 --dtype bf16 --no-e2e --no-cpu-baseline
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_7b.jsonl 2> $O/reference_7b.err; echo "reference rc=$?"
if [ "${NCU:-1}" = 1 ]; then
  python bench.py --quick --steps 2 --warmup 3 > $O/quick_7b.jsonl 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file $O/launches_7b.csv \
      python bench.py --quick --steps 2 --warmup 3 > $O/ncu_launches_7b.log 2>&1; echo "launches rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:"k_adam|k_amax" --launch-skip 6 -c 3 -o $O/full_7b -f \
      python bench.py --quick --steps 1 --warmup 2 > $O/ncu_full_7b.log 2>&1; echo "full_7b rc=$?"
  python bench.py --quick --config gpt-125m --steps 2 --warmup 3 > $O/quick_125m.jsonl 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_adam|k_amax" --launch-skip 9 -c 3 -o $O/full_125m -f \
      python bench.py --quick --config gpt-125m --steps 1 --warmup 3 > $O/ncu_full_125m.log 2>&1; echo "full_125m rc=$?"
  python bench.py --quick --config c1 --steps 2 --warmup 3 > $O/quick_c1.jsonl 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_adam|k_amax" --launch-skip 9 -c 3 -o $O/full_c1 -f \
      python bench.py --quick --config c1 --steps 1 --warmup 3 > $O/ncu_full_c1.log 2>&1; echo "full_c1 rc=$?"
fi
