"""Pins of oracle/sp.py: the FP8 activation converter g of sequence / tensor parallelism
(§2.3, Fig. 5; readings R31-R32).  Expected values come from the
mathematics of the construction (integer sums, half-ulp bounds, the degenerate N = 1),
and bf16 rounding from torch."""
import numpy as np
import torch

from oracle import pipeline as P
from oracle import sp as SP
from oracle.codec import E4M3, decode, encode

F32 = np.float32


def _parts(rng, N, m, spread=True):
    return [(rng.standard_t(3, size=m) * (10.0 ** rng.uniform(-2, 1) if spread else 1.0)).astype(np.float32)
            for _ in range(N)]


def test_allgather_single_rank_is_jit_quantize():
    rng = np.random.default_rng(1)
    x = _parts(rng, 1, 5000)[0]
    r = SP.allgather_fp8([x])
    a, _ = P.amax(x)
    s = F32(F32(448.0) / a)
    assert r["scale"] == s and np.array_equal(r["codes"], encode(x * s, E4M3))
    assert np.max(np.abs(decode(r["codes"], E4M3))) == 448.0


def test_allgather_order_scale_and_half_ulp():
    """Rank order of the gathered codes; the rank holding the global amax attains 448;
    every dequantized value is within half an E4M3 ulp (relative 2^-4 in the normal
    range, 2^-10 / s absolute below it) of the input."""
    rng = np.random.default_rng(2)
    parts = _parts(rng, 4, 3001)
    r = SP.allgather_fp8(parts)
    s = r["scale"]
    big = int(np.argmax([np.abs(x).max() for x in parts]))
    assert s == F32(F32(448.0) / F32(np.abs(parts[big]).max()))
    for k, x in enumerate(parts):
        c = r["codes"][k * 3001:(k + 1) * 3001]
        assert np.array_equal(c, encode(x * s, E4M3))
    assert np.max(np.abs(decode(r["codes"][big * 3001:(big + 1) * 3001], E4M3))) == 448.0
    x = np.concatenate(parts).astype(np.float64)
    out = r["out"].astype(np.float64)
    bound = np.maximum(np.abs(x) * 2.0 ** -4, 2.0 ** -10 / float(s)) * (1 + 1e-6)
    assert np.all(np.abs(out - x) <= bound)


def test_reduce_scatter_sum_is_exact_integer_arithmetic():
    """Every E4M3 value is k 2^-9 (|k| <= 229376): the rank-order binary32 sum equals the
    integer sum of the k's (N <= 73), and the output is fl(S * fl(1/s))."""
    rng = np.random.default_rng(3)
    for N in (2, 3, 8):
        m = 777
        full = [(rng.standard_t(3, size=N * m) * 1e-3).astype(np.float32) for _ in range(N)]
        r = SP.reduce_scatter_fp8(full)
        for k in range(N):
            ks = sum((decode(c[k * m:(k + 1) * m], E4M3) * 512).astype(np.int64) for c in r["codes_by_rank"])
            assert np.array_equal(r["sums"][k].astype(np.float64), ks.astype(np.float64) / 512)
            assert np.array_equal(r["out_by_rank"][k], r["sums"][k] * r["scale_inv"])


def test_reduce_scatter_accuracy_bound():
    """out_k differs from the exact chunk sum by at most the N quantization errors (half
    an ulp each) plus the final binary32 multiply."""
    rng = np.random.default_rng(4)
    N, m = 4, 2000
    full = [(rng.standard_t(3, size=N * m) * 1e-2).astype(np.float32) for _ in range(N)]
    r = SP.reduce_scatter_fp8(full)
    s = float(r["scale"])
    for k in range(N):
        chunk = [f[k * m:(k + 1) * m].astype(np.float64) for f in full]
        exact = sum(chunk)
        err_q = sum(np.maximum(np.abs(c) * 2.0 ** -4, 2.0 ** -10 / s) for c in chunk)
        out = r["out_by_rank"][k].astype(np.float64)
        assert np.all(np.abs(out - exact) <= err_q * (1 + 1e-6) + np.abs(out) * 2.0 ** -23)


def test_scale_rules_zero_ranks():
    """all-zero ranks do not constrain the scale (+inf ignored by the MIN); all zero -> 1"""
    x = np.array([0.5, -2.0, 1.0], np.float32)
    z = np.zeros(3, np.float32)
    assert SP.allgather_fp8([z, x])["scale"] == F32(224.0)          # 448 / 2
    r = SP.allgather_fp8([z, z])
    assert r["scale"] == 1.0 and np.all(r["out"] == 0)


def test_bf16_round_matches_torch():
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(100000) * 10.0 ** rng.uniform(-30, 30, 100000)).astype(np.float32)
    x[:4] = [0.0, -0.0, np.inf, -np.inf]
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(SP.bf16_round(x).view(np.uint32), ref.view(np.uint32))
