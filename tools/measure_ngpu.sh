#!/bin/bash
# Multi-GPU measurement set (N GPUs of one B200 box) + the multi-GPU parity tests.
set -u
O=${O:-gpurun_out/mn}
mkdir -p $O
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_sp.py tests/test_gpu_parity.py -q -x \
      -k "multi or nccl or sp or simulated_fused" > $O/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -2 $O/pytest_multi.log
fi
run() { local n=$1; shift; local tag=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > $O/$tag.jsonl 2> $O/$tag.err; echo "$tag rc=$?"; python tools/bl.py $O/$tag.jsonl; }
run 2 bench_125m_n2_p2p --config gpt-125m --no-e2e
run 4 bench_125m_n4_p2p --config gpt-125m --no-e2e
run 2 bench_125m_n2_zero --config gpt-125m --exchange zero --no-e2e
run 4 bench_7b_n4_p2p --steps 10 --no-e2e
run 2 bench_7b_n2_p2p --steps 10 --no-e2e
run 4 bench_7b_n4_p2p_delayed --steps 10 --state-scaling delayed --no-e2e
run 4 bench_13b_n4_zero --config gpt-13b --exchange zero --steps 10 --no-e2e
run 4 bench_7b_n4_nccl --steps 10 --exchange nccl --no-e2e
