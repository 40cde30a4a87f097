"""Pins of oracle/strategies.py: pre-, post- and auto-scaling FP8 all-reduce and the
Fig. 6 statistics (§2.1 Eq. 1-6; Fig. 6).
Every expected value below is a closed form of the construction, not a re-run."""
import math

import numpy as np

from oracle import pipeline as P
from oracle import strategies as ST
from oracle.codec import E4M3, decode, encode

F32 = np.float32


def _rand(rng, N, n, scale=1e-3):
    return [(rng.standard_t(3, size=n) * scale).astype(np.float32) for _ in range(N)]


def test_auto_is_the_method_and_post_is_auto_at_mu_1():
    rng = np.random.default_rng(1)
    gs = _rand(rng, 3, 5000)
    for mu in (F32(0.5), F32(1.0), F32(2.0)):
        a = ST.allreduce_strategy(gs, ST.AUTO, mu)
        ref = P.allreduce_tensor(gs, mu)
        assert np.array_equal(a["codes"], ref["codes"])
        assert a["scale"] == ref["scale"] and a["sat"] == ref["sat"]
        assert a["mu_next"] == P.mu_update(mu, ref["sat"], 5000, False)
    p = ST.allreduce_strategy(gs, ST.POST)
    a1 = ST.allreduce_strategy(gs, ST.AUTO, F32(1.0))
    assert np.array_equal(p["codes"], a1["codes"]) and p["scale"] == a1["scale"]


def test_single_rank_degenerate():
    """N = 1: pre == post, both equal one quantization."""
    rng = np.random.default_rng(2)
    gs = _rand(rng, 1, 3000)
    pre, post = ST.allreduce_strategy(gs, ST.PRE), ST.allreduce_strategy(gs, ST.POST)
    assert np.array_equal(pre["codes"], post["codes"]) and pre["scale"] == post["scale"]
    q = encode(gs[0] * pre["s"], E4M3)
    assert np.array_equal(pre["codes"], q)
    assert (pre["underflow"], pre["overflow"]) == (post["underflow"], post["overflow"])
    # N + 1 = 2 encodes per element; the second re-encodes exact E4M3 values: no events
    u = int(np.count_nonzero((gs[0] != 0) & (decode(q, E4M3) == 0)))
    assert pre["underflow"] == u and pre["events"] == 2 * 3000


def test_cancellation_gives_exact_zero():
    """{x, -x}: every strategy returns exactly 0."""
    rng = np.random.default_rng(3)
    x = _rand(rng, 1, 2000)[0]
    for st in (ST.PRE, ST.POST, ST.AUTO):
        r = ST.allreduce_strategy([x, -x], st)
        assert np.all(decode(r["codes"], E4M3) == 0) and np.all(r["g_hat"] == 0)


def test_identical_ranks_prescaling_is_one_quantization():
    """N = 4 identical tensors, pre-scaling: x/4 is exact and E4M3's grid is the same in
    every normal binade, so E4M3(x/4) = E4M3(x)/4 and the sum of 4 is E4M3(x) again:
    g_hat = fl(dec(E4M3(t s)) * fl(1/s)) wherever |t s|/4 >= 2^-6."""
    rng = np.random.default_rng(4)
    t = _rand(rng, 1, 4000)[0]
    r = ST.allreduce_strategy([t] * 4, ST.PRE)
    s = r["s"]
    x = t * s
    one = decode(encode(x, E4M3), E4M3).astype(np.float32) * F32(F32(1) / s)
    normal = np.abs(x) / 4 >= 2.0 ** -6
    assert normal.sum() > 1000
    assert np.array_equal(r["g_hat"][normal], one[normal])
    assert r["overflow"] == 0


def _ladder(N):
    """amax 448 (so s = fl(448/448) = 1 exactly) plus 2^-k, k = 0..20, on every rank."""
    v = np.array([448.0] + [2.0 ** -k for k in range(21)], np.float32)
    return [v.copy() for _ in range(N)]


def test_underflow_and_overflow_closed_forms():
    """Ranks hold identical ladders. Pre-scaling at N = 2^p encodes 2^-(k+p): the code
    is zero iff 2^-(k+p) <= 2^-10 (2^-10 is the 0 / 2^-9 midpoint, ties to even 0).
    Post: rank codes vanish iff k >= 10; the sum of N copies of 448 exceeds 448 once per
    element with 448 (one overflow); pre's 448/N sums back to exactly 448 (none)."""
    for p in (1, 3, 7):
        N = 2 ** p
        gs = _ladder(N)
        pre = ST.allreduce_strategy(gs, ST.PRE)
        post = ST.allreduce_strategy(gs, ST.POST)
        assert pre["s"] == 1.0 and post["s"] == 1.0
        assert pre["underflow"] == N * sum(1 for k in range(21) if k + p >= 10)
        assert post["underflow"] == N * sum(1 for k in range(21) if k >= 10)
        assert post["overflow"] == 1 and pre["overflow"] == 0
        assert pre["events"] == post["events"] == (N + 1) * 22
        # the surviving pre-scaled ladder sums back exactly: g_hat = 2^-k for k + p <= 9
        for k in range(21):
            if k + p <= 9:
                assert pre["g_hat"][1 + k] == F32(2.0 ** -k)


def test_snr_closed_form():
    """N = 1, s = 1: 1.03125 = 1 + 2^-5 rounds to 1 in E4M3 (3 mantissa bits), 448 is
    exact, so SNR = 10 log10((448^2 + K 1.03125^2) / (K 2^-10))."""
    K = 37
    g = np.array([448.0] + [1.03125] * K, np.float32)
    r = ST.allreduce_strategy([g], ST.POST)
    ref = 10 * math.log10((448.0 ** 2 + K * 1.03125 ** 2) / (K * 2.0 ** -10))
    assert abs(r["snr_db"] - ref) < 1e-9
    exact = ST.allreduce_strategy([np.array([448.0, 1.0, -2.0], np.float32)], ST.POST)
    assert exact["snr_db"] == float("inf")


def test_all_underflow_construction():
    """Tiny gradients, pre-scaling, N = 128: every nonzero rank value except
    the one carrying amax underflows."""
    N, n = 128, 50
    gs = [np.full(n, 1e-3, np.float32) for _ in range(N)]
    gs[0][0] = 1e3                      # amax: s = 448/1000, 1e-3 s / 128 < 2^-10
    r = ST.allreduce_strategy(gs, ST.PRE)
    assert r["underflow"] == N * n - 1


def test_prescaling_orders_against_postscaling():
    """Monotone consequences of Eq. 1 vs Eq. 2 at N = 2^p with the same s: pre's rank
    inputs are post's divided by N, so everything post loses to underflow pre loses too,
    and pre's codes are at most 448/N, whose sum never exceeds 448 (no overflow)."""
    rng = np.random.default_rng(5)
    for sigma in (1e-6, 1e-3, 1.0):
        gs = [(rng.lognormal(0, 2, 3000) * sigma * rng.choice([-1, 1], 3000)).astype(np.float32)
              for _ in range(16)]
        pre, post = ST.allreduce_strategy(gs, ST.PRE), ST.allreduce_strategy(gs, ST.POST)
        assert pre["underflow"] >= post["underflow"]
        assert pre["overflow"] == 0 and post["overflow"] >= 0
