#!/bin/bash
# Multi-GPU measurement set (N GPUs of one B200 box) + the multi-GPU parity tests.
set -u
O=${O:-gpurun_out/mn}
mkdir -p $O
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_sp.py -q -x > $O/pytest_multi.log 2>&1
  echo "pytest multi rc=$?"; tail -2 $O/pytest_multi.log
fi
run() { local n=$1; shift; local tag=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) "$@" > $O/$tag.jsonl 2> $O/$tag.err; echo "$tag rc=$?"; python tools/bl.py $O/$tag.jsonl 2>/dev/null; }
run 2 bench_7b_n2 bench.py --gpus 2 --steps 20 --warmup 5
run 4 bench_7b_n4 bench.py --gpus 4 --steps 20 --warmup 5
run 4 bench_7b_n4_unsplit bench.py --gpus 4 --steps 20 --warmup 5 --buckets 1 --no-e2e
run 4 bench_7b_n4_delayed bench.py --gpus 4 --steps 20 --warmup 5 --state-scaling delayed --no-e2e
run 4 bench_7b_n4_nccl bench.py --gpus 4 --steps 10 --warmup 3 --exchange nccl --no-e2e
run 4 bench_13b_n4_zero bench.py --gpus 4 --config gpt-13b --exchange zero --steps 10 --warmup 3 --buckets 4 --no-e2e
run 4 bench_13b_n4_zero_unsplit bench.py --gpus 4 --config gpt-13b --exchange zero --steps 10 --warmup 3 --buckets 1 --no-e2e
run 2 bench_125m_n2 bench.py --gpus 2 --config gpt-125m --no-e2e
run 4 bench_125m_n4 bench.py --gpus 4 --config gpt-125m --no-e2e
run 2 c5_n2 bench_c5.py --min-log2 10 --max-log2 30 --stride 2
run 4 c5_n4 bench_c5.py --min-log2 10 --max-log2 30 --stride 2
run 2 c5_n2_bf16src bench_c5.py --min-log2 10 --max-log2 30 --stride 4 --src-dtype bf16
NCCL_ALGO=Ring run 4 c5_n4_ring bench_c5.py --min-log2 10 --max-log2 30 --stride 4
NCCL_ALGO=NVLS run 4 c5_n4_nvls bench_c5.py --min-log2 10 --max-log2 30 --stride 4
run 2 sp_n2 bench_sp.py
run 4 sp_n4 bench_sp.py
