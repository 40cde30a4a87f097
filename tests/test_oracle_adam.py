"""Pins of oracle/adam.py (§2.2; App. B; hyper-parameters P:301)."""
import math

import numpy as np
import torch

from oracle import adam as A
from oracle import adam as OA
from oracle.codec import E4M3, FP16, decode

F32 = np.float32


def test_hyper_params_closed_form():
    hp = A.hyper_params(3e-4, 1)
    assert hp.beta1 == F32(0.9) and hp.beta2 == F32(0.95)
    assert hp.step_size == F32(3e-4 / 0.1)                            # lr / (1 - beta1)
    assert hp.inv_bc2_sqrt == F32(1 / math.sqrt(0.05))
    assert hp.decay == F32(1 - 3e-5)                                  # wd = 0.1
    assert hp.eps == F32(1e-8)
    hp = A.hyper_params(1e-3, 10 ** 6)                                 # bias corrections -> 1
    assert hp.step_size == F32(1e-3) and hp.inv_bc2_sqrt == F32(1.0)


def test_fp32_arithmetic_matches_torch_adamw_float64():
    """With quantization bypassed, the binary32 sequence R16 tracks textbook AdamW
    (decoupled decay, bias correction, eps after sqrt) — torch.optim.AdamW in float64."""
    rng = np.random.default_rng(11)
    n = 4096
    w0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    lr, wd = 1e-3, 0.1
    p = torch.tensor(w0.astype(np.float64), requires_grad=True)
    opt = torch.optim.AdamW([p], lr=lr, betas=(0.9, 0.95), eps=1e-8, weight_decay=wd,
                            foreach=False)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    w = w0.copy()
    for t in range(1, 11):
        g = (rng.standard_normal(n) * 10.0 ** rng.uniform(-5, -2)).astype(np.float32)
        p.grad = torch.tensor(g.astype(np.float64))
        opt.step()
        m, v, w = A.adam_math(g, m, v, w, A.hyper_params(lr, t, weight_decay=wd))
        ref = p.detach().numpy()
        assert np.max(np.abs(w - ref) / (np.abs(ref) + 1e-3)) < 1e-5, t


def test_step1_sign_descent_closed_form():
    """From zero moments: m^ = g, v^ = g^2, so w' = w(1 - lr wd) - lr g/(|g| + eps)."""
    rng = np.random.default_rng(12)
    g = (rng.standard_normal(1000) * 1e-3).astype(np.float32)
    w = (rng.standard_normal(1000) * 0.02).astype(np.float32)
    lr = 3e-4
    _, _, w1 = A.adam_math(g, np.zeros_like(g), np.zeros_like(g), w, A.hyper_params(lr, 1))
    g64 = g.astype(np.float64)
    ref = w.astype(np.float64) * (1 - lr * 0.1) - lr * g64 / (np.abs(g64) + 1e-8)
    assert np.allclose(w1, ref, rtol=1e-5, atol=1e-9)


def _half_ulp(x, fmt):
    e = np.floor(np.log2(np.maximum(np.abs(x), fmt.min_normal)))
    return 2.0 ** (e - fmt.mbits) / 2


def test_jit_state_encoding_within_half_ulp_and_attains_max():
    rng = np.random.default_rng(13)
    n = 50000
    w0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    st = A.init_state(w0)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    res = A.adam_step(g, st, A.hyper_params(1e-3, 1))
    new = res["state"]
    for stt, x, fmt, mx in ((new.m1, res["m"], E4M3, 448.0), (new.v, res["v"], FP16, 65504.0),
                            (new.master, res["w"], FP16, 65504.0), (new.w8, res["w"], E4M3, 448.0)):
        scaled = x.astype(np.float64) * float(stt.scale)
        dec = decode(stt.codes, fmt)
        # one rounding of fl(x * s): within half a format ulp (+ the binary32 product rounding)
        assert np.all(np.abs(dec - scaled) <= _half_ulp(scaled, fmt) + 1e-7 * np.abs(scaled))
        assert np.max(np.abs(dec)) == mx                      # JIT scale maps amax to max
        assert stt.scale == F32(F32(mx) / stt.amax)
        assert stt.scale_inv == F32(F32(1) / stt.scale)
    assert np.all(res["v"] >= 0) and np.all(new.v.codes < 0x8000)


def test_zero_gradient_fixed_point():
    """zero gradient, zero moments, wd = 0 -> parameters unchanged."""
    w0 = np.array([0.5, -0.25, 0.125, 0.0], np.float32)     # exactly representable master
    st = A.init_state(w0)
    res = A.adam_step(np.zeros(4, np.float32), st, A.hyper_params(1e-3, 1, weight_decay=0.0))
    assert np.array_equal(res["state"].master.codes, st.master.codes)
    assert np.array_equal(res["w"], w0)
    assert res["state"].m1.scale == 1.0 and res["state"].v.scale == 1.0


def test_exact_master_step_closed_form():
    """Master weights chosen exactly representable at their JIT FP16 scale (65504/0.5):
    w' = w(1 - lr wd) - step_size * m'/(sqrt(v') / sqrt(1-b2) + eps), in float64."""
    w0 = np.array([0.5, -0.25, 0.125, 0.0], np.float32)
    st = A.init_state(w0)
    assert np.array_equal(st.master.value(), w0)
    g = np.array([1.5e-3, -2.4e-4, 1.07e-3, 3.3e-6], np.float32)
    lr = 3e-4
    res = A.adam_step(g, st, A.hyper_params(lr, 1))
    g64 = g.astype(np.float64)
    ref = w0 * (1 - lr * 0.1) - (lr / 0.1) * (0.1 * g64) / (np.sqrt(0.05 * g64 ** 2) / math.sqrt(0.05) + 1e-8)
    assert np.allclose(res["w"], ref, rtol=2e-6, atol=1e-10)


def test_bytes_per_param():
    assert A.bytes_per_param() == 6                      # Eq. 8
    assert A.bytes_per_param(4, 4, 4, 4) == 16           # Eq. 7


def test_skip_leaves_state():
    st = A.init_state(np.linspace(-1, 1, 64).astype(np.float32))
    res = A.adam_step(np.full(64, np.nan, np.float32), st, A.hyper_params(1e-3, 1), skip=True)
    assert np.array_equal(res["state"].master.codes, st.master.codes)
    assert res["state"].master.scale == st.master.scale


# ---------------------------------------------------------------- delayed state scaling
def _random_state(rng, n, step_scale=1.0):
    w0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    st = OA.init_state(w0)
    hist = OA.init_history(st)
    for t in range(1, 4):                        # a few JIT steps: non-trivial m1 / v
        g = (rng.standard_t(3, size=n) * 1e-3 * step_scale).astype(np.float32)
        st = OA.adam_step(g, st, OA.hyper_params(1e-3, t))["state"]
    return st, hist


def test_delayed_bounds_never_saturate_moments():
    """R25: the a-priori bounds put |m'| and v' at or below the format max — no code of m1
    or v ever saturates, on random states and on the equality case (aligned extremes)."""
    rng = np.random.default_rng(31)
    for trial in range(30):
        n = 5000
        st, hist = _random_state(rng, n, 10.0 ** rng.uniform(-2, 2))
        gsi = np.float32(10.0 ** rng.uniform(-9, -5))
        codes = rng.integers(-448, 449, size=n).astype(np.float32)
        if trial % 3 == 0:                       # extremes of m and g aligned
            codes[0] = 448.0
            st.m1.codes[0] = 0x7E
        g = (decode(OA.encode(codes, E4M3), E4M3).astype(np.float32) * gsi).astype(np.float32)
        res = OA.adam_step_delayed(g, st, OA.hyper_params(1e-3, 5), gsi, hist, 5)
        s_m, s_v, _, _ = res["scales"]
        assert np.all(np.abs(res["m"].astype(np.float64) * s_m) <= 448.0 * (1 + 2 ** -22))
        assert np.all(res["v"].astype(np.float64) * s_v <= 65504.0 * (1 + 2 ** -22))


def test_delayed_encoding_half_ulp_and_history_ring():
    rng = np.random.default_rng(32)
    st, hist = _random_state(rng, 20000)
    g = (rng.standard_t(3, size=20000) * 1e-3).astype(np.float32)
    gsi = np.float32(np.abs(g).max() / 448.0)
    hist = hist.copy()
    for step in range(1, 20):
        res = OA.adam_step_delayed(g, st, OA.hyper_params(1e-3, step), gsi, hist, step)
        new = res["state"]
        for stt, x, fmt in ((new.m1, res["m"], E4M3), (new.v, res["v"], FP16), (new.master, res["w"], FP16)):
            scaled = x.astype(np.float64) * float(stt.scale)
            dec = decode(stt.codes, fmt)
            assert np.all(np.abs(dec - scaled) <= _half_ulp(scaled, fmt) + 1e-7 * np.abs(scaled))
        # exact amax recorded; slot (step-1) % 16 of the ring receives it
        assert new.master.amax == np.float32(np.abs(res["w"]).max())
        assert res["hist"][(step - 1) % OA.HIST] == new.master.amax
        others = [i for i in range(OA.HIST) if i != (step - 1) % OA.HIST]
        assert np.array_equal(res["hist"][others], hist[others])
        # master keeps 16x headroom over the history maximum: never saturates here
        assert np.max(np.abs(decode(new.master.codes, FP16))) < 65504.0 / 8
        st, hist = new, res["hist"]


def test_delayed_update_arithmetic_is_the_jit_one():
    """Delayed scaling changes only the encoding: m', v', w' equal the JIT step's."""
    rng = np.random.default_rng(33)
    st, hist = _random_state(rng, 3000)
    g = (rng.standard_normal(3000) * 1e-3).astype(np.float32)
    a = OA.adam_step(g, st, OA.hyper_params(1e-3, 4))
    b = OA.adam_step_delayed(g, st, OA.hyper_params(1e-3, 4), np.float32(1e-6), hist, 4)
    for k in ("m", "v", "w"):
        assert np.array_equal(a[k], b[k])


def test_delayed_recorded_bound_attained_never_exceeded_and_tight():
    """R25 (recorded-amax bound): B_m = fl(fl(b1 M) + fl((1-b1) G)) (1 + 2^-20), M the largest
    dequantized m the recorded exact amax can give, G = fl(448 g_sinv).  Over 60 delayed
    steps from the initial state: no m1 / v code ever saturates; in the aligned case
    (the largest m and a code-448 gradient of the same sign at the same element) |m'| is
    the bound's own sum, encoding at the format max and not beyond; and the headroom
    log2(B_m / max|m'|) stays below 2 binades after the first 10 steps (the round-1
    format-ceiling bound kept 6 on average and up to 15: profiles/r2/f1_headroom.json)."""
    rng = np.random.default_rng(41)
    n = 4096
    st = OA.init_state((rng.standard_normal(n) * 0.02).astype(np.float32))
    hist = OA.init_history(st)
    heads = []
    for step in range(1, 61):
        gsi = np.float32(10.0 ** rng.uniform(-7, -6))
        codes = rng.integers(-300, 301, size=n).astype(np.float32)
        aligned = step > 1 and step % 5 == 0
        if aligned:
            i = int(np.argmax(np.abs(st.m1.value())))
            codes[i] = 448.0 if st.m1.value()[i] >= 0 else -448.0
        g = (decode(OA.encode(codes, E4M3), E4M3).astype(np.float32) * gsi).astype(np.float32)
        hp = OA.hyper_params(1e-3, step)
        b_m, b_v = OA.delayed_moment_bounds(st, gsi, hp)
        res = OA.adam_step_delayed(g, st, hp, gsi, hist, step)
        s_m, s_v, _, _ = res["scales"]
        m, v = res["m"].astype(np.float64), res["v"].astype(np.float64)
        assert np.all(np.abs(m) * s_m <= 448.0 * (1 + 2 ** -22)) and np.all(v * s_v <= 65504.0 * (1 + 2 ** -22))
        assert np.all(np.abs(decode(res["state"].m1.codes, E4M3)) <= 448.0)
        if aligned:      # the bound is attained (up to its slack) at the aligned element
            assert np.abs(m).max() == np.float64(np.float32(b_m / OA.BOUND_SLACK)) or \
                np.abs(m).max() >= float(b_m) * (1 - 2 ** -20)
        if step > 10:
            heads.append(math.log2(float(b_m) / np.abs(m).max()))
        st, hist = res["state"], res["hist"]
    assert max(heads) < 2.0, max(heads)
