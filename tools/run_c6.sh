set -u
O=gpurun_out/c6; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nccl.py -x -q -k p2p > $O/pytest_nccl.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_nccl.log
run() { local n=$1; shift; local tag=$1; shift
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) "$@" > $O/$tag.jsonl 2> $O/$tag.err; echo "$tag rc=$?"; }
run 2 bench_n2_p2p_delayed bench.py --gpus 2 --state-scaling delayed --no-e2e --no-cpu-baseline
run 4 bench_n4_p2p_delayed bench.py --gpus 4 --state-scaling delayed --no-e2e --no-cpu-baseline
run 4 bench_7b_n4_p2p_delayed bench.py --gpus 4 --config gpt-7b --steps 10 --state-scaling delayed --no-e2e --no-cpu-baseline
