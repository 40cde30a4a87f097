set -u
O=gpurun_out/c10; mkdir -p $O
run() { local n=$1; shift; local tag=$1; shift
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) "$@" > $O/$tag.jsonl 2> $O/$tag.err; echo "$tag rc=$?"; }
FP8LM_P2P_QX=2 run 4 bench_n4_qx2 bench.py --gpus 4 --no-e2e --no-cpu-baseline
FP8LM_P2P_QX=4 run 4 bench_n4_qx4 bench.py --gpus 4 --no-e2e --no-cpu-baseline
FP8LM_P2P_TMA=1 FP8LM_P2P_QX=4 run 4 bench_n4_tma_qx4 bench.py --gpus 4 --no-e2e --no-cpu-baseline
FP8LM_P2P_QX=4 run 4 bench_7b_n4_qx4 bench.py --gpus 4 --config gpt-7b --steps 10 --no-e2e --no-cpu-baseline
FP8LM_P2P_TMA=1 FP8LM_P2P_QX=4 run 4 bench_7b_n4_tma_qx4 bench.py --gpus 4 --config gpt-7b --steps 10 --no-e2e --no-cpu-baseline
FP8LM_P2P_TMA=1 FP8LM_P2P_QX=8 run 4 bench_7b_n4_tma_qx8 bench.py --gpus 4 --config gpt-7b --steps 10 --no-e2e --no-cpu-baseline
run 4 bench_7b_n4_base bench.py --gpus 4 --config gpt-7b --steps 10 --no-e2e --no-cpu-baseline
FP8LM_P2P_QX=2 run 2 bench_n2_qx2 bench.py --gpus 2 --no-e2e --no-cpu-baseline
