#!/bin/bash
# ZeRO (C4) split-step A/B on 4 GPUs: experiment builds x bucket counts, interleaved
O=${O:-gpurun_out/abz}
A="--config,gpt-13b,--exchange,zero,--steps,10,--warmup,3"
ITEMS=${ITEMS:-"build_ab/lib_push.so:$A,--buckets,4 build_ab/lib_zp2new.so:$A,--buckets,4 build_ab/lib_push.so:$A,--buckets,1 build_ab/lib_push.so:$A,--buckets,6"} \
  O=$O N=4 bash tools/ab_ngpu.sh
