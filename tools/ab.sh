#!/bin/bash
# A/B timing of experiment builds on one box, interleaved to cancel clock drift:
#   LIBS="a.so b.so" [CFGS="gpt-7b gpt-125m"] [ARGS="..."] bash tools/ab.sh
O=${O:-gpurun_out/ab}
mkdir -p $O
for rep in 1 2 3; do
  for lib in ${LIBS}; do
    tag=$(basename $lib .so)
    for cfg in ${CFGS:-gpt-7b gpt-125m}; do
      steps=20; [ $cfg = gpt-125m ] && steps=100
      FP8LM_LIB=$(realpath $lib) python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps $steps $ARGS > $O/${tag}_${cfg}_$rep.jsonl 2>&1
      python tools/bl.py $O/${tag}_${cfg}_$rep.jsonl
    done
  done
done
