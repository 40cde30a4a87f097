"""Oracle of the FP8 sequence/tensor-parallel activation converter g (§2.3,
P:193-200, Fig. 5; Table 7): "We add an FP8 datatype conversion prior to g,
such that the all-gather (or reduce-scatter) operation uses FP8 low-bit activation to
save communication cost across GPUs".  SURVEY §8(f) row f4.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings (R31-R32):

R31  Forward g = all-gather of the N sequence partitions x_r (m elements each).  The
     converter makes ONE scaling tensor of the gathered activation: the shared scale of
     Eq. 4 (s = min_r s_r, s_r = fl(448 / amax_r), the pipeline's zero / overflow rules,
     no mu: nothing is summed, so nothing can overflow), codes E4M3(fl(x_r * s)) in rank
     order, scale s, scale_inv fl(1/s); the consumer's view is fl(dec(c) * scale_inv).
R32  Backward g = reduce-scatter of the N ranks' full activation gradients dy_r (N m
     elements each): the same shared-scale quantization of every dy_r (Eq. 4-5), then
     rank k receives the k-th chunk of every rank's codes and sums them in rank order in
     binary32 (R12); its output is fl(S * fl(1/s)) — the sum is consumed in higher
     precision by the sequence-parallel region, so it is not requantized (no second
     rounding, no overflow, hence no mu).
"""
from __future__ import annotations

from typing import Dict, List

import numpy as np

from . import pipeline as P
from .codec import E4M3, decode_f32, encode

F32 = np.float32


def shared_scale(parts: List[np.ndarray]) -> np.float32:
    """Eq. 4 with mu = 1: min_r fl(448 / amax_r) (+inf for all-zero ranks; all-inf -> 1)."""
    s_r = [P.local_scale(*P.amax(x), F32(1.0)) for x in parts]
    s, _ = P.global_scale(s_r)
    return s


def allgather_fp8(parts: List[np.ndarray]) -> Dict:
    """R31: parts[r] = rank r's partition (binary32 values; bf16 inputs widened exactly).
    Returns dict(codes [N m], scale, scale_inv, out [N m] = dequantized gathered view)."""
    xs = [np.asarray(x, dtype=np.float32) for x in parts]
    s = shared_scale(xs)
    codes = np.concatenate([encode(x * s, E4M3) for x in xs]) if xs else np.zeros(0, np.uint8)
    with np.errstate(divide="ignore"):
        sinv = F32(F32(1.0) / s)
    return dict(codes=codes, scale=s, scale_inv=sinv, out=decode_f32(codes, E4M3) * sinv)


def reduce_scatter_fp8(full: List[np.ndarray]) -> Dict:
    """R32: full[r] = rank r's activation gradient of N m elements.  Returns dict(scale,
    scale_inv, codes_by_rank [N][N m], out_by_rank [N][m] = fl(S_k * fl(1/s)))."""
    N = len(full)
    ys = [np.asarray(y, dtype=np.float32) for y in full]
    s = shared_scale(ys)
    codes = [encode(y * s, E4M3) for y in ys]
    with np.errstate(divide="ignore"):
        sinv = F32(F32(1.0) / s)
    m = ys[0].size // N
    sums = [P.rank_order_sum([c[k * m:(k + 1) * m] for c in codes]) for k in range(N)]
    return dict(scale=s, scale_inv=sinv, codes_by_rank=codes, sums=sums, m=m,
                out_by_rank=[S * sinv for S in sums])


def bf16_round(x: np.ndarray) -> np.ndarray:
    """binary32 -> bfloat16 (round to nearest even), returned as binary32 values: the
    optional bf16 outputs of the converter."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    r = np.where(nan, (b | 0x400000) >> 16 << 16, r)
    return r.astype(np.uint32).view(np.float32)
