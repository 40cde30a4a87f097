"""Oracle of the FP8 gradient all-reduce STRATEGIES compared in PAPER.md §2.1 and Fig. 6:
pre-scaling (Eq. 1), post-scaling (Eq. 2) and automatic scaling (Eq. 3-6, the method),
with the Fig. 6 statistics: SNR, underflow rate and overflow rate (
SPEC S:181-241 "CommStats").  SURVEY §8(f) row f3.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings (R28-R30):

R28  All three strategies quantize every rank's binary32 gradient with ONE shared
     per-tensor scale (Eq. 4: s = min_r s_r = s(max_r amax_r)); they differ only in
     where 1/N and mu enter:
       pre   c_r = E4M3(fl(fl(g_r * s) / N)),  s = fl(448 / A)          result scale s
       post  c_r = E4M3(fl(g_r * s)),          s = fl(448 / A)          result scale fl(N s)
       auto  c_r = E4M3(fl(g_r * s)),          s = fl(fl(448 / A) mu)   result scale fl(N s)
     then S = rank-order binary32 sum of dec(c_r) (R12) and c = E4M3(S) (R13) for all
     three.  auto is exactly pipeline.allreduce_tensor; post is auto at mu = 1.
R29  Quantization events: the N*n rank encodes plus the n encodes of the sum.  An event
     UNDERFLOWS when its input is nonzero and its code is zero; it OVERFLOWS when its
     input magnitude exceeds the format maximum 448 (the encoder clamps or rounds it
     down to 448).  underflow_rate / overflow_rate = counts / events.
R30  snr_db = 10 log10(sum m^2 / sum (g_hat - m)^2), m = the float64 mean
     of the ranks' binary32 gradients, g_hat = fl(dec(c) * fl(1/scale)) (the dequantized
     result, A6); +inf when the error is 0, nan when both sums are 0.

mu follows pipeline.mu_update (R1-R3) from the saturation count of c (codes that attain
448) for auto; pre and post keep mu = 1.
"""
from __future__ import annotations

from typing import Dict, List

import numpy as np

from . import pipeline as P
from .codec import E4M3, decode, decode_f32, encode

F32 = np.float32
PRE, POST, AUTO = 0, 1, 2
NAMES = {PRE: "pre", POST: "post", AUTO: "auto"}


def _events(x: np.ndarray, codes: np.ndarray):
    """(underflow, overflow) counts of one batch of encodes x -> codes (R29)."""
    x = np.asarray(x, dtype=np.float32)
    dec = decode(codes, E4M3)
    under = int(np.count_nonzero((x != 0) & (dec == 0)))
    over = int(np.count_nonzero(np.abs(x.astype(np.float64)) > 448.0))
    return under, over


def shared_scale(grads_by_rank: List[np.ndarray], mu: np.float32) -> np.float32:
    """Eq. 4 via the pipeline's rules (local scales, MIN, zero / non-finite handling)."""
    s_r = [P.local_scale(*P.amax(g), mu) for g in grads_by_rank]
    s, _skip = P.global_scale(s_r)
    return s


def allreduce_strategy(grads_by_rank: List[np.ndarray], strategy: int,
                       mu: np.float32 = F32(1.0)) -> Dict:
    """One strategy on one tensor held by N ranks.  Returns dict(codes, scale, scale_inv,
    g_hat, sat, mu_next, underflow, overflow, events, sig2, err2, snr_db)."""
    N = len(grads_by_rank)
    gs = [np.asarray(g, dtype=np.float32) for g in grads_by_rank]
    n = int(gs[0].size)
    mu_used = F32(mu) if strategy == AUTO else F32(1.0)
    s = shared_scale(gs, mu_used)
    under = over = 0
    codes_by_rank = []
    for g in gs:
        x = g * s                                                  # fl(g * s)
        if strategy == PRE:
            x = x / F32(N)                                         # fl(fl(g * s) / N)
        c = encode(x, E4M3)
        u, o = _events(x, c)
        under += u
        over += o
        codes_by_rank.append(c)
    S = P.rank_order_sum(codes_by_rank)
    codes = P.requantize(S)
    u, o = _events(S, codes)
    under += u
    over += o
    if strategy == PRE:
        scale = s
        with np.errstate(divide="ignore"):
            scale_inv = F32(F32(1.0) / scale)
    else:
        scale, scale_inv = P.aggregated_scale(N, s)
    g_hat = decode_f32(codes, E4M3) * scale_inv                   # fl(dec(c) * fl(1/s))
    m = np.zeros(n, np.float64)
    for g in gs:
        m += g.astype(np.float64)
    m /= N
    err = g_hat.astype(np.float64) - m
    sig2 = float(np.dot(m, m))
    err2 = float(np.dot(err, err))
    sat = P.sat_count(codes)
    mu_next = P.mu_update(mu_used, sat, n, False) if strategy == AUTO else F32(1.0)
    return dict(codes=codes, scale=scale, scale_inv=scale_inv, g_hat=g_hat, sat=sat,
                mu_next=mu_next, underflow=under, overflow=over, events=(N + 1) * n,
                sig2=sig2, err2=err2, snr_db=snr_db(sig2, err2), s=s)


def snr_db(sig2: float, err2: float) -> float:
    """R30: 10 log10(signal / error); +inf for zero error, nan for 0/0."""
    if err2 == 0.0:
        return float("nan") if sig2 == 0.0 else float("inf")
    if sig2 == 0.0:
        return float("-inf")
    return 10.0 * float(np.log10(sig2 / err2))
