"""GPU parity of fp8lm_allreduce_strategy (pre-, post-, auto-scaling FP8 all-reduce and
the Fig. 6 statistics; §2.1 Eq. 1-6, Fig. 6; readings R28-R30) against
oracle/strategies.py: codes, scales, mu and every event count bit-exact; the binary64
error sums to 1e-12 relative (their summation order differs)."""
import numpy as np
import pytest
import torch

from oracle import strategies as ST

pytestmark = pytest.mark.gpu

F32 = np.float32


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2310_18313_b200 as B
    return B


def _ensemble(N, n, seed, sigma=1e-3, rho=0.5, zeros=False):
    """log-normal magnitudes with random signs, a common component across ranks (rho)"""
    rng = np.random.default_rng(seed)
    common = rng.lognormal(0, 2, n) * rng.choice([-1.0, 1.0], n)
    out = []
    for _ in range(N):
        own = rng.lognormal(0, 2, n) * rng.choice([-1.0, 1.0], n)
        g = (sigma * (rho * common + np.sqrt(1 - rho * rho) * own)).astype(np.float32)
        if zeros:
            g[rng.random(n) < 0.05] = 0.0
        out.append(g)
    return out


def _compare(B, gs, strategy, mu=1.0, steps=1, offset=0):
    N, n = len(gs), gs[0].size
    dev = torch.device("cuda")
    # an offset view exercises the unaligned (scalar) kernels
    flat = torch.zeros(N * n + offset, dtype=torch.float32, device=dev)
    flat[offset:] = torch.from_numpy(np.concatenate(gs)).to(dev)
    g = flat[offset:].view(N, n) if offset == 0 else None
    mu_d = torch.tensor([mu], dtype=torch.float32, device=dev)
    stats = B.commstats_buffer(dev)
    mu_h = F32(mu)
    for step in range(steps):
        if offset:
            codes = torch.empty(n, dtype=torch.uint8, device=dev)
            B._binding._check(B.lib.fp8lm_allreduce_strategy(
                B.STRATEGIES[strategy], flat.data_ptr() + 4 * offset, N, n, mu_d.data_ptr(),
                codes.data_ptr(), stats.data_ptr(), 0), "strategy")
        else:
            codes, _ = B.allreduce_strategy(g, strategy, mu_d, stats=stats)
        d = B.commstats_read(stats)
        ref = ST.allreduce_strategy(gs, {"pre": ST.PRE, "post": ST.POST, "auto": ST.AUTO}[strategy], mu_h)
        c = codes.cpu().numpy()
        assert np.array_equal(c, ref["codes"]), (strategy, step, int(np.sum(c != ref["codes"])))
        assert d["s"] == ref["s"] and d["scale"] == ref["scale"] and d["scale_inv"] == ref["scale_inv"]
        for k in ("underflow", "overflow", "events", "sat"):
            assert d[k] == ref[k], (k, d[k], ref[k])
        assert d["sig2"] == pytest.approx(ref["sig2"], rel=1e-12, abs=1e-300)
        assert d["err2"] == pytest.approx(ref["err2"], rel=1e-12, abs=1e-300)
        if strategy == "auto":
            assert d["mu_next"] == ref["mu_next"] and float(mu_d.item()) == ref["mu_next"]
            mu_h = ref["mu_next"]
        else:
            assert d["mu_next"] == 1.0 and float(mu_d.item()) == mu
    return d


@pytest.mark.parametrize("strategy", ["pre", "post", "auto"])
@pytest.mark.parametrize("N,n", [(1, 1000), (2, 4096), (3, 70001), (8, 20000), (128, 6000)])
def test_strategy_parity(B, strategy, N, n):
    gs = _ensemble(N, n, seed=N * 1000 + n, zeros=True)
    _compare(B, gs, strategy, mu=1.0 if strategy != "auto" else 0.25, steps=3 if strategy == "auto" else 1)


@pytest.mark.parametrize("strategy", ["pre", "post", "auto"])
def test_strategy_unaligned_and_ragged(B, strategy):
    gs = _ensemble(5, 1001, seed=7)
    _compare(B, gs, strategy, offset=1)
    _compare(B, _ensemble(4, 3, seed=8), strategy)          # smaller than one vector


def test_strategy_closed_forms_on_gpu(B):
    """the oracle's ladder construction (tests/test_oracle_strategies.py) on the GPU"""
    v = np.array([448.0] + [2.0 ** -k for k in range(21)], np.float32)
    for p in (1, 3, 7):
        N = 2 ** p
        d_pre = _compare(B, [v.copy() for _ in range(N)], "pre")
        d_post = _compare(B, [v.copy() for _ in range(N)], "post")
        assert d_pre["underflow"] == N * sum(1 for k in range(21) if k + p >= 10)
        assert d_post["overflow"] == 1 and d_pre["overflow"] == 0


def test_auto_mu_converges_and_beats_post_on_overflow(B):
    """mu halves while the aggregated codes saturate, then the overflow rate of auto is
    below post-scaling's on the same ensemble (Fig. 6(c))."""
    dev = torch.device("cuda")
    gs = _ensemble(128, 50000, seed=9, rho=0.9)
    g = torch.from_numpy(np.stack(gs)).to(dev)
    mu = torch.ones(1, device=dev)
    st = B.commstats_buffer(dev)
    for _ in range(12):
        B.allreduce_strategy(g, "auto", mu, stats=st)
    auto = B.commstats_read(st)
    B.allreduce_strategy(g, "post", stats=st)
    post = B.commstats_read(st)
    assert auto["mu_used"] < 1.0
    assert auto["overflow_rate"] < post["overflow_rate"]
    assert auto["snr_db"] > post["snr_db"]
