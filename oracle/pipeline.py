"""Oracle of the FP8 gradient pipeline: amax, auto-scaling factor mu, shared minimum
scale, E4M3 quantization, FP32 rank-order reduction, requantization, saturation
count, dequantization.  PAPER.md §2.1 "FP8 Gradient and All-Reduce Communication",
P:98-142.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Per tensor (nothing couples two tensors), for step t, ranks r = 0..N-1:

  1. amax_r = max_i |g_r[i]|                                  (App. B JIT scaling)
  2. mu update from the previous step's saturation count       (readings R1-R6)
  3. s_r = fl(fl(448 / amax_r) * mu)                           (Eq. 3 g' = mu*g, P:116-121;
                                                                scale reading R7)
  4. s_g = min_r s_r                                           (Eq. 4)
  5. c_r[i] = E4M3(fl(g_r[i] * s_g))                           (Eq. 5; R9)
  6. S[i] = ((dec(c_0[i]) + dec(c_1[i])) + ...) + dec(c_{N-1}[i])  in binary32   (Eq. 6; R12)
  7. c[i] = E4M3(S[i]),  s = fl(N * s_g)                       (Eq. 6; R13)
  8. sat = #{i : |dec(c[i])| == 448}                           ("attains the maximum"; R4)
  9. g_hat[i] = fl(dec(c[i]) * fl(1/s))                        ("actual gradient is g'/s'")

All binary32 arithmetic is spelled with explicit np.float32 operations, one
rounding each.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .codec import E4M3, decode_f32, encode

F32 = np.float32
E4M3_MAX = F32(448.0)
E4M3_MAX_CODE = 0x7E
# mu growth factor: fl(2^(1/1000)) = 0x3F8016B9, so that mu reaches 2 after 1000
# consecutive clean steps from mu = 1 ("exponentially increase mu to 2 over the span
# of 1,000 training steps"; reading R2).
MU_GROWTH = F32(2.0 ** (1.0 / 1000.0))
MU_MAX = F32(2.0)
# "If the ratio of the maximum value exceeds a specified threshold, i.e., 0.001%"
# (P:122): ratio = sat / n > 1e-5  <=>  sat * 100000 > n, compared exactly (R3).
SAT_THRESHOLD_DEN = 100000


def amax(g: np.ndarray) -> Tuple[np.float32, bool]:
    """max |g| over binary32 values (exact: max involves no rounding) and a non-finite flag.

    Reading R14: any NaN makes amax NaN, else any inf makes it inf (the device kernel
    reports the same).  The flag is True iff amax is not finite."""
    g = np.asarray(g, dtype=np.float32)
    if g.size == 0:
        return F32(0.0), False
    a = np.abs(g)
    if np.isnan(a).any():
        return F32(np.nan), True
    m = F32(a.max())
    return m, bool(np.isinf(m))


def mu_update(mu: np.float32, sat: int, n: int, skipped: bool) -> np.float32:
    """Auto-scaling factor update, applied once per step after the reduction.

    R1: "mu is set to 1/2" read as HALVING (assignment cannot recover when mu = 1/2
        still overflows).  R2: otherwise smooth per-step growth by fl(2^(1/1000)),
        capped at 2.  R3: strict '>' on the exact ratio sat/n vs 1e-5.  R14: a
        skipped (non-finite) step halves mu for every tensor.
    """
    mu = F32(mu)
    if skipped or sat * SAT_THRESHOLD_DEN > n:
        return F32(mu * F32(0.5))
    return min(MU_MAX, F32(mu * MU_GROWTH))


def local_scale(amax_r: np.float32, nonfinite: bool, mu: np.float32) -> np.float32:
    """s_r = fl(fl(448 / amax_r) * mu)  (JIT, margin 0, not power-of-two; R7).

    Non-finite gradient -> 0 (forces a global skip via the MIN, R14).  amax == 0, or
    448/amax overflowing, -> +inf (ignored by the MIN; R14)."""
    if nonfinite:
        return F32(0.0)
    if amax_r == 0:
        return F32(np.inf)
    r = F32(E4M3_MAX / F32(amax_r))
    if np.isinf(r):
        return F32(np.inf)
    return F32(r * F32(mu))


def global_scale(local_scales: Sequence[np.float32]) -> Tuple[np.float32, bool]:
    """Eq. 4: s'_g = min(s'_1, ..., s'_N).  Returns (s_g, skip).

    s_g == 0  -> skip the optimizer step (some rank saw a non-finite gradient).
    s_g == inf (every rank all-zero / tiny) -> s_g = 1 (SPEC S:151's zero-tensor scale)."""
    s = F32(np.min(np.asarray(local_scales, dtype=np.float32)))
    if s == 0:
        return F32(0.0), True
    if np.isinf(s):
        return F32(1.0), False
    return s, False


def quantize(g: np.ndarray, s_g: np.float32) -> np.ndarray:
    """Eq. 5 with FP32 input (R9): g''_r = FP8(s'_g * g_r), one rounding to E4M3."""
    scaled = np.asarray(g, dtype=np.float32) * F32(s_g)      # fl(g * s_g)
    return encode(scaled, E4M3)


def rank_order_sum(codes_by_rank: Sequence[np.ndarray]) -> np.ndarray:
    """Eq. 6 'g = g''_1 + ... + g''_N' accumulated in binary32 in rank order (R12)."""
    S = decode_f32(codes_by_rank[0], E4M3)
    for c in codes_by_rank[1:]:
        S = S + decode_f32(c, E4M3)                            # fl(S + dec(c_r))
    return S


def requantize(S: np.ndarray) -> np.ndarray:
    """Stored form of the aggregate: the E4M3 code of the SUM (R13)."""
    return encode(S, E4M3)


def sat_count(codes: np.ndarray) -> int:
    """Number of codes that attain the E4M3 maximum magnitude 448 (R4)."""
    c = np.asarray(codes, dtype=np.uint8)
    return int(np.count_nonzero((c & 0x7F) == E4M3_MAX_CODE))


def aggregated_scale(n_ranks: int, s_g: np.float32) -> Tuple[np.float32, np.float32]:
    """Eq. 6: s = N * s'_g; returns (s, fl(1/s))."""
    s = F32(F32(n_ranks) * F32(s_g))
    with np.errstate(divide="ignore"):
        return s, F32(F32(1.0) / s)


def dequantize(codes: np.ndarray, scale_inv: np.float32) -> np.ndarray:
    """'The actual weight gradient is g'/s'': fl(dec(c) * fl(1/s)) (R8)."""
    return decode_f32(codes, E4M3) * F32(scale_inv)


# ------------------------------------------------------------------ one tensor, N ranks
def allreduce_tensor(grads_by_rank: List[np.ndarray], mu: np.float32):
    """Steps 1-8 for one tensor held by N simulated ranks.

    Returns dict(amax=[N], s_r=[N], s_g, skip, codes_by_rank=[N], codes, sat, scale,
    scale_inv, mu_next)."""
    N = len(grads_by_rank)
    n = int(np.asarray(grads_by_rank[0]).size)
    amaxes, flags = zip(*(amax(g) for g in grads_by_rank))
    s_r = [local_scale(a, f, mu) for a, f in zip(amaxes, flags)]
    s_g, skip = global_scale(s_r)
    codes_by_rank = [quantize(g, s_g) for g in grads_by_rank]
    S = rank_order_sum(codes_by_rank)
    codes = requantize(S)
    sat = sat_count(codes)
    scale, scale_inv = aggregated_scale(N, s_g)
    return dict(amax=list(amaxes), nonfinite=list(flags), s_r=s_r, s_g=s_g, skip=skip,
                codes_by_rank=codes_by_rank, sum=S, codes=codes, sat=sat,
                scale=scale, scale_inv=scale_inv, n=n)
