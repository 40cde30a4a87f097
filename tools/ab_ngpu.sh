#!/bin/bash
# multi-GPU A/B of experiment builds: ITEMS="lib.so:bench-args ..." N=4 bash tools/ab_ngpu.sh
O=${O:-gpurun_out/abn}
N=${N:-4}
mkdir -p $O
for rep in 1 2; do
  for item in ${ITEMS}; do
    lib=${item%%:*}; args=${item#*:}; args=${args//,/ }
    tag=$(basename $lib .so)_$(echo $args | tr -d ' -')_$rep
    FP8LM_LIB=$(realpath $lib) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --no-e2e $args \
      > $O/$tag.jsonl 2> $O/$tag.err
    echo "$tag rc=$?"; python tools/bl.py $O/$tag.jsonl
  done
done
