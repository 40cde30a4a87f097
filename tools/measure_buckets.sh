#!/bin/bash
# bucketed split step (fp8lm_dp_step_split) at N GPUs: 7B P2P and 13B ZeRO, buckets 1..8
set -u
O=${O:-gpurun_out/bk}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q > $O/loopback.log 2>&1; echo "loopback rc=$?"; tail -2 $O/loopback.log
run() { local n=$1; shift; local tag=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > $O/$tag.jsonl 2> $O/$tag.err; echo "$tag rc=$?"; python tools/bl.py $O/$tag.jsonl; tail -3 $O/$tag.err; }
for b in 1 2 4 8; do run 4 b7b_n4_k$b --steps 10 --no-e2e --buckets $b; done
for b in 1 4; do run 4 b125_n4_k$b --config gpt-125m --no-e2e --buckets $b; done
for b in 1 4; do run 4 b13b_n4_zero_k$b --config gpt-13b --exchange zero --steps 10 --no-e2e --buckets $b; done
run 2 b7b_n2_k4 --steps 10 --no-e2e --buckets 4
