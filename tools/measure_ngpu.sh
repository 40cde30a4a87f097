#!/bin/bash
# Multi-GPU measurement set of profiles/r1 (4 GPUs of one B200 box) + the multi-GPU parity tests.
set -u
O=gpurun_out/mn
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_sp.py -q > $O/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -2 $O/pytest_multi.log
run() { local n=$1; shift; local tag=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) "$@" > $O/$tag.jsonl 2> $O/$tag.err; echo "$tag rc=$?"; }
run 2 bench_n2_p2p bench.py --gpus 2
run 4 bench_n4_p2p bench.py --gpus 4
run 2 bench_n2_nccl bench.py --gpus 2 --exchange nccl --no-e2e
run 2 bench_n2_p2p_delayed bench.py --gpus 2 --state-scaling delayed --no-e2e
run 4 bench_n4_p2p_delayed bench.py --gpus 4 --state-scaling delayed --no-e2e
run 2 bench_n2_zero bench.py --gpus 2 --exchange zero --no-e2e
run 4 bench_7b_n4_p2p bench.py --gpus 4 --config gpt-7b --steps 10 --no-e2e
run 4 bench_7b_n4_p2p_delayed bench.py --gpus 4 --config gpt-7b --steps 10 --state-scaling delayed --no-e2e
run 4 bench_13b_n4_zero bench.py --gpus 4 --config gpt-13b --exchange zero --steps 10 --no-e2e
