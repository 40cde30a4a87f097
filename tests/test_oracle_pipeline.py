"""Pins of oracle/pipeline.py (§2.1) against closed forms,
invariants, exact integer arithmetic and the worked example (task rule ③)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import pipeline as P
from oracle import step as S
from oracle import adam as A
from oracle.codec import E4M3, decode

F32 = np.float32
GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------- mu controller
def test_mu_reaches_two_after_exactly_1000_clean_steps():
    """'exponentially increase mu to 2 over the span of 1,000 training steps'."""
    mu = F32(1.0)
    for k in range(1, 1001):
        mu = P.mu_update(mu, 0, 10 ** 6, False)
        if k == 999:
            assert mu < 2.0
            assert abs(float(mu) - 2 ** (999 / 1000)) < 3e-4     # geometric growth (fl(G) = G(1+5e-8))
    assert mu == F32(2.0)
    assert P.mu_update(mu, 0, 10 ** 6, False) == F32(2.0)        # cap


def test_mu_halves_on_overflow_ratio():
    """'If the ratio ... exceeds ... 0.001%, mu is set to 1/2', read as halving (R1)."""
    assert P.mu_update(F32(1.0), 10, 10 ** 5, False) == F32(0.5)      # 1e-4 > 1e-5
    assert P.mu_update(F32(0.5), 10, 10 ** 5, False) == F32(0.25)     # repeated overflow
    # exact threshold: ratio == 1e-5 does NOT exceed; one more count does (R3)
    assert P.mu_update(F32(1.0), 1, 100000, False) > 1.0
    assert P.mu_update(F32(1.0), 2, 100000, False) == F32(0.5)
    assert P.mu_update(F32(1.0), 0, 7, True) == F32(0.5)              # skipped step (R14)


# ------------------------------------------------------------- scales (Eq. 3, Eq. 4)
def test_local_scale_examples():
    assert P.local_scale(F32(2.0), False, F32(1.0)) == F32(224.0)     # 448/2
    assert P.local_scale(F32(2.0), False, F32(0.5)) == F32(112.0)     # Eq. 3 g' = mu g
    assert P.local_scale(F32(0.0), False, F32(1.0)) == np.inf
    assert P.local_scale(F32(np.inf), True, F32(1.0)) == 0.0
    s, skip = P.global_scale([F32(0.5), F32(1.0), F32(2.0)])           # S:223, Eq. 4
    assert s == F32(0.5) and not skip
    assert P.global_scale([F32(np.inf), F32(np.inf)]) == (F32(1.0), False)
    assert P.global_scale([F32(3.0), F32(0.0)])[1] is True


def test_min_of_scales_is_scale_of_max_amax():
    """RN is monotone, so MIN over rank scales == scale of the MAX amax."""
    rng = np.random.default_rng(3)
    for _ in range(2000):
        N = int(rng.integers(1, 9))
        a = (10.0 ** rng.uniform(-8, 3, size=N)).astype(np.float32)
        mu = F32(2.0 ** rng.integers(-4, 2))
        s = [P.local_scale(x, False, mu) for x in a]
        sg, _ = P.global_scale(s)
        assert sg == P.local_scale(F32(a.max()), False, mu)


# ------------------------------------------------------------- reduce (Eq. 6)
def test_rank_order_sum_is_exact_integer_arithmetic():
    """Every E4M3 value is k * 2^-9 with |k| <= 229376, and binary32 holds every
    multiple of 2^-9 below 2^15, so the FP32 sum of N <= 73 codes is exact (R12)."""
    rng = np.random.default_rng(5)
    for N in (1, 2, 3, 8, 73):
        codes = rng.integers(0, 256, size=(N, 4096)).astype(np.uint8)
        codes[(codes & 0x7F) == 0x7F] = 0x7E                # no NaN
        codes[:, :4] = np.array([0x7E, 0xFE, 0x01, 0x81], np.uint8)   # extremes
        Ssum = P.rank_order_sum(list(codes))
        k = np.rint(decode(codes, E4M3) * 512).astype(np.int64)        # exact integers
        assert np.array_equal(Ssum.astype(np.float64), k.sum(axis=0) / 512.0)
        # order independence (a consequence of exactness)
        perm = rng.permutation(N)
        assert np.array_equal(P.rank_order_sum(list(codes[perm])), Ssum)


def test_requantize_single_rounding_bound():
    rng = np.random.default_rng(6)
    Ssum = (rng.uniform(-448, 448, size=100000)).astype(np.float32)
    c = P.requantize(Ssum)
    d = decode(c, E4M3)
    e = np.floor(np.log2(np.maximum(np.abs(Ssum.astype(np.float64)), 2.0 ** -6)))
    half_ulp = 2.0 ** (e - 3) / 2
    assert np.all(np.abs(d - Ssum) <= half_ulp)


def test_eq6_scale_times_n():
    for N in (1, 2, 4, 8):
        s_g = F32(149333.328125)
        s, sinv = P.aggregated_scale(N, s_g)
        assert Fraction(float(s)) == N * Fraction(float(s_g))          # exact for 2^k
    assert P.sat_count(np.array([0x7E, 0xFE, 0x7D, 0x7F, 0x00], np.uint8)) == 2


def test_allreduce_is_the_mean_within_quantization_error():
    """dequant(all-reduce) approximates mean_r(g_r): each of the N+1 roundings is at most
    half an E4M3 ulp of its operand (P:127 'actual gradient is g'/s'')."""
    rng = np.random.default_rng(7)
    for N in (1, 2, 4, 8):
        g = [(rng.standard_normal(20000) * 1e-3).astype(np.float32) for _ in range(N)]
        # mu = 1/N keeps every sum in range (what the mu controller converges to)
        r = P.allreduce_tensor(g, F32(1.0 / N))
        ghat = P.dequantize(r["codes"], r["scale_inv"]).astype(np.float64)
        mean = np.mean(np.stack([x.astype(np.float64) for x in g]), axis=0)
        sg = float(r["s_g"])

        def half_ulp(v):
            e = np.floor(np.log2(np.maximum(np.abs(v), 2.0 ** -6)))
            return 2.0 ** (e - 3) / 2

        bound = sum(half_ulp(np.asarray(x, np.float64) * sg) for x in g) + half_ulp(r["sum"].astype(np.float64))
        bound = bound / (N * sg) + 1e-6 * np.abs(mean) + 1e-30
        ok = np.abs(r["sum"]) <= 448                             # non-saturated elements
        assert np.all(np.abs(ghat - mean)[ok] <= bound[ok])
        assert ok.all()


def test_n1_reduce_is_identity():
    g = (np.random.default_rng(8).standard_normal(5000) * 3e-4).astype(np.float32)
    r = P.allreduce_tensor([g], F32(1.0))
    assert np.array_equal(r["codes"], r["codes_by_rank"][0])
    assert r["scale"] == r["s_g"]


def test_worked_example_golden():
    w = json.load(open(os.path.join(GOLD, "worked_example.json")))
    g0 = np.array(w["g0"], np.float32)
    g1 = np.array(w["g1"], np.float32)
    r = P.allreduce_tensor([g0, g1], F32(1.0))
    hx = lambda v: "0x%08X" % np.float32(v).view(np.uint32)
    assert [hx(s) for s in r["s_r"]] == w["s_r_hex"]
    assert hx(r["s_g"]) == w["s_g_hex"]
    assert r["codes_by_rank"][0].tolist() == w["c0"]
    assert r["codes_by_rank"][1].tolist() == w["c1"]
    assert r["sum"].tolist() == w["sum"]
    assert r["codes"].tolist() == w["codes"]
    assert r["sat"] == w["sat"]
    assert float(r["scale"]) == w["scale"]
    assert P.mu_update(F32(1.0), r["sat"], 4, False) == F32(w["mu_next"])


def test_nonfinite_skips_step_and_halves_mu():
    g_ok = np.ones(16, np.float32) * 1e-3
    g_bad = g_ok.copy()
    g_bad[3] = np.inf
    w0 = np.linspace(-0.1, 0.1, 16).astype(np.float32)
    st = A.init_state(w0)
    r = S.train_step([[g_ok, g_ok], [g_bad, g_ok]], [F32(1.0), F32(1.0)], [st, st],
                     A.hyper_params(1e-3, 1))
    assert r["skip"]
    assert r["per_tensor"][0]["s_g"] == 0.0
    assert r["mu_next"] == [F32(0.5), F32(0.5)]
    for t in range(2):
        assert np.array_equal(r["states"][t].master.codes, st.master.codes)
        assert np.array_equal(r["states"][t].m1.codes, st.m1.codes)


def test_nan_amax_reported():
    a, f = P.amax(np.array([1.0, np.nan, np.inf], np.float32))
    assert np.isnan(a) and f
    a, f = P.amax(np.array([-3.0, np.inf], np.float32))
    assert np.isinf(a) and f
    assert P.amax(np.zeros(0, np.float32)) == (0.0, False)


def test_worked_example_adam_half_through_train_step():
    """SURVEY §8(c) worked example, Adam half, through oracle.step.train_step's non-skip
    path (dequantize -> adam_step hand-off): u, w', s_m = 2986666.25, m1 codes
    [0x7E, 0xE9, 0x7A, 0x38] and the v / master / w8 codes and scales, each derived by
    hand in tests/golden/worked_example.json _derivation_adam (P:172-178 state layout,
    P:301 hyper-parameters).  Passing scale instead of scale_inv, dequantizing the
    per-rank codes, or skipping Adam changes every one of them."""
    w = json.load(open(os.path.join(GOLD, "worked_example.json")))
    a = w["adam"]
    g0 = np.array(w["g0"], np.float32)
    g1 = np.array(w["g1"], np.float32)
    st0 = A.init_state(np.array(a["w0"], np.float32))
    assert st0.master.codes.tolist() == a["master0_codes"]
    r = S.train_step([[g0], [g1]], [F32(1.0)], [st0], A.hyper_params(a["lr"], a["step"]))
    assert not r["skip"]
    ad = r["per_tensor"][0]["adam"]
    assert ad["m"].tolist() == [float(F32(x)) for x in a["m_new"]]
    assert ad["v"].tolist() == [float(F32(x)) for x in a["v_new"]]
    assert ad["w"].tolist() == [float(F32(x)) for x in a["w_new"]]
    ns = r["states"][0]
    hx = lambda v: "0x%08X" % np.float32(v).view(np.uint32)
    assert ns.m1.scale == F32(a["s_m"])
    assert hx(ns.v.scale) == a["s_v_hex"]
    assert hx(ns.master.scale) == a["s_w_hex"]
    assert hx(ns.w8.scale) == a["s_8_hex"]
    assert ns.m1.codes.tolist() == a["m1_codes"]
    assert ns.v.codes.tolist() == a["v_codes"]
    assert ns.master.codes.tolist() == a["master_codes"]
    assert ns.w8.codes.tolist() == a["w8_codes"]
    # u follows from w' and the master's decoded w: fl(w*decay) - fl(step*u) = w' exactly
    hp = A.hyper_params(a["lr"], a["step"])
    u = np.array(a["u"], np.float32)
    wd = st0.master.value() * hp.decay
    assert ((wd - hp.step_size * u).astype(np.float32) == ad["w"]).all()
