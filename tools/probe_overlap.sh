set -u
O=gpurun_out/probe; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/overlap_probe.py"
for cfg in "--config gpt-125m" "--config gpt-7b --layers 8"; do
  for k in "" 1 2; do
    FP8LM_P2P_PER_SM=$k timeout 300 $R $cfg >> $O/probe.jsonl 2>> $O/probe.err; echo "$cfg k=$k rc=$?"
  done
done
