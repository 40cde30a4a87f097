"""paper_2310_18313_b200 — the FP8-LM (arXiv 2310.18313) data-parallel hot path on B200.

FP8 gradient all-reduce with automatic scaling and a shared minimum scale (§2.1,
Eq. 3-6) feeding the precision-decoupled FP8 AdamW (§2.2, Eq. 8), as hand-written
sm_100a CUDA behind the C ABI in include/fp8lm.h.  This package is the thin Python
binding (argument marshalling only); see DESIGN.md.
"""
from ._binding import (  # noqa: F401
    ALIGN_ELEMS, BF16, E4M3, E5M2, F16, F32, MODE_LOCAL, MODE_NCCL, MODE_P2P, MODE_SIMULATED, MODE_ZERO,
    CompactLayout,
    AdamHP, Comm, FP8DataParallel, FP8LMError, OptimizerState, Plan, STensorSet, adam_hp,
    allreduce_jit, amax_scale_sync, fp8_adam_step, fp8_adam_step_delayed, fp8_dequantize, fp8_grad_allreduce, fp8_quantize,
    has_nccl, lib, LIB_PATH, prof_enable, prof_read, state_init, version, zero_plan,
    STRATEGIES, allreduce_strategy, commstats_buffer, commstats_metrics, commstats_read, SPConverter,
    peer_setup_loopback, peer_timeout_report, set_peer_timeout, BucketedDP, bucket_split,
)
