set -u
O=gpurun_out/sp; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sp.py -q > $O/pytest_sp.log 2>&1; echo "pytest sp rc=$?"; tail -2 $O/pytest_sp.log
run() { local n=$1; shift; local tag=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) "$@" > $O/$tag.jsonl 2> $O/$tag.err; echo "$tag rc=$?"; }
run 2 sp_converter_n2 bench_sp.py
run 4 sp_converter_n4 bench_sp.py
