#!/bin/bash
# ZeRO (C4) split-step A/B on 4 GPUs: experiment builds x bucket counts, interleaved
O=${O:-gpurun_out/abz}
A="--config,gpt-13b,--exchange,zero,--steps,10,--warmup,3"
ITEMS="build_ab/lib_zp2new.so:$A,--buckets,4 build_ab/lib_zp2old.so:$A,--buckets,4 build_ab/lib_zp2new.so:$A,--buckets,6 build_ab/lib_x296.so:$A,--buckets,4 build_ab/lib_h2.so:$A,--buckets,4" \
  O=$O N=4 bash tools/ab_ngpu.sh
