#!/bin/bash
# A/B on one box: the current library (new) against libfp8lm_old.so.bin (the previous
# head), interleaved, plus the GPU parity tests on the new one.
set -u
O=gpurun_out/ab2; mkdir -p $O
L=paper_2310_18313_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_strategies.py tests/test_gpu_fastmath.py -x -q > $O/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -1 $O/pytest_parity.log
for i in 1 2; do
  for v in new old; do
    cp $L/libfp8lm_$v.so.bin $L/libfp8lm.so
    timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/b_${v}_$i.jsonl 2>>$O/err_$v
  done
done
for v in new old; do
  cp $L/libfp8lm_$v.so.bin $L/libfp8lm.so
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --state-scaling delayed > $O/bd_$v.jsonl 2>>$O/err_$v
  timeout 300 python bench.py --config gpt-7b --steps 10 --no-e2e --no-cpu-baseline > $O/b7_$v.jsonl 2>>$O/err_$v
  timeout 300 python bench.py --config gpt-7b --steps 10 --no-e2e --no-cpu-baseline --state-scaling delayed > $O/b7d_$v.jsonl 2>>$O/err_$v
done
cp $L/libfp8lm_new.so.bin $L/libfp8lm.so
timeout 300 python bench.py --quick --steps 2 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_adam" -c 4 -o $O/full \
    python bench.py --quick --steps 2 --warmup 3 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
echo done
