"""Oracle of the precision-decoupled FP8 AdamW step (§2.2).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

State per parameter tensor (Eq. 8: 2 + 1 + 1 + 2 = 6 bytes/param):
  * gradient      FP8 E4M3 codes + scale     (the all-reduce output, §2.1 Eq. 6)
  * first moment  FP8 E4M3 codes + scale     ("can tolerate a high quantization error
                                              and can be assigned with low-precision FP8")
  * second moment FP16 + scale (R17)         ("allocating a 16-bit higher precision")
  * master weight FP16 + scale               ("FP16 with tensor scaling")
plus the FP8 E4M3 weight copy w8 + scale written back for the next forward
(BASELINE.json north_star; R20).

Scaling tensors hold (codes, scale, scale_inv, amax); logical value =
decode(code) * scale_inv (R8).  State scales are JUST-IN-TIME (App. B: "the
operator first produces ... the output in higher precision, then calculates the
maximum absolute value of the output, and finally applies this scaling factor"):
computed from the exact amax of the new binary32 values (R18).

AdamW with decoupled weight decay, beta1 = 0.9, beta2 = 0.95, weight decay 0.1
(P:301); eps = 1e-8 and bias correction (R15); the binary32 op sequence (R16):
    m  = fl(dec8(cm) * m_sinv);  v = fl(dec16(hv) * v_sinv);  w = fl(dec16(hw) * w_sinv)
    m' = fl(fl(b1*m) + fl(omb1*g))
    v' = fl(fl(b2*v) + fl(fl(omb2*g)*g))
    den = fl(fl(sqrt(v') * inv_bc2_sqrt) + eps)       (sqrt correctly rounded)
    u  = fl(m' / den)
    w' = fl(fl(w*decay) - fl(step_size*u))
with the host scalars of ``hyper_params`` (computed in float64, rounded once; R24).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict

import numpy as np

from .codec import E4M3, FP16, decode_f32, encode

F32 = np.float32
E4M3_MAX = F32(448.0)
FP16_MAX = F32(65504.0)


@dataclass
class AdamHP:
    beta1: np.float32
    beta2: np.float32
    one_minus_beta1: np.float32
    one_minus_beta2: np.float32
    eps: np.float32
    decay: np.float32          # fl(1 - lr*wd)
    step_size: np.float32      # fl(lr / (1 - beta1^t))
    inv_bc2_sqrt: np.float32   # fl(1 / sqrt(1 - beta2^t))


def hyper_params(lr: float, step: int, beta1: float = 0.9, beta2: float = 0.95,
                 eps: float = 1e-8, weight_decay: float = 0.1) -> AdamHP:
    """Per-step scalars, each computed in float64 and rounded once to binary32 (R24).
    Defaults are the paper's; eps is R15.  ``step`` counts from 1."""
    assert step >= 1
    return AdamHP(
        beta1=F32(beta1), beta2=F32(beta2),
        one_minus_beta1=F32(1.0 - beta1), one_minus_beta2=F32(1.0 - beta2),
        eps=F32(eps),
        decay=F32(1.0 - lr * weight_decay),
        step_size=F32(lr / (1.0 - beta1 ** step)),
        inv_bc2_sqrt=F32(1.0 / math.sqrt(1.0 - beta2 ** step)),
    )


@dataclass
class ScaledTensor:
    """The paper's scaling tensor: codes + per-tensor scale."""
    codes: np.ndarray
    fmt: object
    scale: np.float32 = F32(1.0)
    scale_inv: np.float32 = F32(1.0)
    amax: np.float32 = F32(0.0)

    def value(self) -> np.ndarray:
        return decode_f32(self.codes, self.fmt) * F32(self.scale_inv)

    def copy(self) -> "ScaledTensor":
        return ScaledTensor(self.codes.copy(), self.fmt, self.scale, self.scale_inv, self.amax)


def jit_scale(a: np.float32, fmt_max: np.float32) -> np.float32:
    """JIT state scale fl(max / amax); amax == 0 or an overflowing ratio -> 1 (R18)."""
    if a == 0:
        return F32(1.0)
    s = F32(fmt_max / F32(a))
    if not np.isfinite(s):
        return F32(1.0)
    return s


def encode_scaled(x: np.ndarray, fmt, fmt_max: np.float32, a: np.float32) -> ScaledTensor:
    s = jit_scale(a, fmt_max)
    codes = encode(np.asarray(x, dtype=np.float32) * s, fmt)       # fl(x * s), one rounding
    return ScaledTensor(codes, fmt, s, F32(F32(1.0) / s), F32(a))


@dataclass
class OptState:
    m1: ScaledTensor       # E4M3
    v: ScaledTensor        # FP16 (scaled, R17)
    master: ScaledTensor   # FP16 (scaled)
    w8: ScaledTensor       # E4M3 weight copy

    def copy(self) -> "OptState":
        return OptState(self.m1.copy(), self.v.copy(), self.master.copy(), self.w8.copy())


def init_state(w0: np.ndarray) -> OptState:
    """Initial state (step 14 of SURVEY §8c): zero moments at scale 1; master and w8
    JIT-encoded from the FP32 initial weights."""
    w0 = np.asarray(w0, dtype=np.float32)
    n = w0.size
    aw = F32(np.abs(w0).max()) if n else F32(0.0)
    return OptState(
        m1=ScaledTensor(np.zeros(n, np.uint8), E4M3),
        v=ScaledTensor(np.zeros(n, np.uint16), FP16),
        master=encode_scaled(w0, FP16, FP16_MAX, aw),
        w8=encode_scaled(w0, E4M3, E4M3_MAX, aw),
    )


def adam_math(g: np.ndarray, m: np.ndarray, v: np.ndarray, w: np.ndarray, hp: AdamHP):
    """The binary32 AdamW arithmetic (R16) on dequantized inputs -> (m', v', w')."""
    g, m, v, w = (np.asarray(x, dtype=np.float32) for x in (g, m, v, w))
    m_new = (hp.beta1 * m) + (hp.one_minus_beta1 * g)
    v_new = (hp.beta2 * v) + ((hp.one_minus_beta2 * g) * g)
    den = (np.sqrt(v_new) * hp.inv_bc2_sqrt) + hp.eps
    u = m_new / den
    w_new = (w * hp.decay) - (hp.step_size * u)
    return m_new.astype(F32), v_new.astype(F32), w_new.astype(F32)


def adam_step(g_hat: np.ndarray, st: OptState, hp: AdamHP, skip: bool = False) -> Dict:
    """One FP8 AdamW step for one tensor.  ``g_hat`` = dequantized gradient (binary32).

    Phase 1 computes m', v', w' and their exact amaxes; phase 2 encodes with the JIT
    scales (App. B "multiple passes").  ``skip`` leaves the state unchanged (R14).
    Returns dict(state=new OptState, m=m', v=v', w=w')."""
    if skip:
        return dict(state=st.copy(), m=None, v=None, w=None)
    g = np.asarray(g_hat, dtype=np.float32)
    m_new, v_new, w_new = adam_math(g, st.m1.value(), st.v.value(), st.master.value(), hp)
    am = F32(np.abs(m_new).max()) if m_new.size else F32(0.0)
    av = F32(v_new.max()) if v_new.size else F32(0.0)          # v' >= 0
    aw = F32(np.abs(w_new).max()) if w_new.size else F32(0.0)
    new = OptState(
        m1=encode_scaled(m_new, E4M3, E4M3_MAX, am),
        v=encode_scaled(v_new, FP16, FP16_MAX, av),
        master=encode_scaled(w_new, FP16, FP16_MAX, aw),
        w8=encode_scaled(w_new, E4M3, E4M3_MAX, aw),
    )
    return dict(state=new, m=m_new, v=v_new, w=w_new)


def bytes_per_param(master: int = 2, grad: int = 1, m1: int = 1, m2: int = 2) -> int:
    """Eq. 7 / Eq. 8 accounting."""
    return master + grad + m1 + m2


# ---------------------------------------------------------------- delayed state scaling
# App. B: "selecting the scaling factor based on the maximum absolute values
# observed in a certain number of preceding iterations ... necessitates the storage of a
# history of maximum values".  Reading R25-R27: the new state scales are
# fixed BEFORE the update, so AdamW becomes ONE pass (12 B/param instead of 18):
#   m1 (E4M3): s_m = 448 / B_m, B_m = beta1 M + (1-beta1) G, M the largest dequantized m
#              the previous step's recorded amax can give, G = 448 g_sinv the reduced
#              gradient's ceiling: an a-priori bound on |m'|, never saturates (R25);
#   v  (FP16): s_v = 65504 / B_v, B_v = beta2 V + (1-beta2) G^2 likewise (R25);
#   master (FP16): s_w = 65504 / (16 H_w), w8 (E4M3): s_8 = 448 / H_w, where H_w is the
#              maximum of the last HIST exact amax(w') values (R26; 16x headroom costs the
#              FP16 master no precision, the w8 copy saturates like any delayed scaling).
# The exact amax of the new values is still recorded (history, diagnostics) (R27).
HIST = 16                              # history length
W_HEADROOM = F32(16.0)
BOUND_SLACK = F32(1.0 + 2.0 ** -20)    # covers the binary32 roundings of the bound itself


def delayed_moment_bounds(st: OptState, g_scale_inv: np.float32, hp: AdamHP, bound: str = "recorded"):
    """(B_m, B_v): a-priori bounds on max|m'| and max v' before the update (R25).

    bound = "recorded" (R25, the method): from the previous step's exact recorded amax
    (R27), through the largest stored code it can produce,
    M = fl(dec(E4M3(fl(A_m s_m))) m_sinv), V = fl(dec(F16(fl(A_v s_v))) v_sinv) (RN is
    monotone, so every dequantized m, v is at most M, V).  Both use G = fl(448 g_sinv),
    the saturation ceiling of the reduced gradient, and the R16 update's own op sequence,
    so |m'| <= B_m and v' <= B_v by monotonicity; x (1 + 2^-20) as in R25.
    bound = "prior" (round 1's reading, kept for tests/f1_headroom.py only): the format
    ceilings |m| <= 448 m_sinv, v <= 65504 v_sinv — the previous BOUNDS, which compound
    and start from the zero state's scale 1: 6 binades of m headroom and 30 of v on
    average over 200 steps (profiles/r2/f1_headroom.json)."""
    gsi = F32(g_scale_inv)
    G = F32(E4M3_MAX * gsi)
    if bound == "prior":
        M = F32(E4M3_MAX * F32(st.m1.scale_inv))
        V = F32(FP16_MAX * F32(st.v.scale_inv))
        b_m = F32(F32(F32(hp.beta1 * E4M3_MAX) * F32(st.m1.scale_inv)) +
                  F32(F32(hp.one_minus_beta1 * E4M3_MAX) * gsi))
        b_v = F32(F32(F32(hp.beta2 * FP16_MAX) * F32(st.v.scale_inv)) +
                  F32(F32(hp.one_minus_beta2 * G) * G))
    else:
        cm = encode(np.array([F32(st.m1.amax) * F32(st.m1.scale)], np.float32), E4M3)
        M = F32(decode_f32(cm, E4M3)[0] * F32(st.m1.scale_inv))
        cv = encode(np.array([F32(st.v.amax) * F32(st.v.scale)], np.float32), FP16)
        V = F32(decode_f32(cv, FP16)[0] * F32(st.v.scale_inv))
        b_m = F32(F32(hp.beta1 * M) + F32(hp.one_minus_beta1 * G))
        b_v = F32(F32(hp.beta2 * V) + F32(F32(hp.one_minus_beta2 * G) * G))
    return F32(b_m * BOUND_SLACK), F32(b_v * BOUND_SLACK)


def delayed_scales(st: OptState, g_scale_inv: np.float32, hp: AdamHP, w_hist, bound: str = "recorded") -> tuple:
    """(s_m, s_v, s_w, s_8), each a binary32 op sequence (the kernel's, R25-R26)."""
    b_m, b_v = delayed_moment_bounds(st, g_scale_inv, hp, bound)
    h_w = F32(np.max(np.asarray(w_hist, dtype=np.float32)))
    return (jit_scale(b_m, E4M3_MAX), jit_scale(b_v, FP16_MAX),
            jit_scale(F32(h_w * W_HEADROOM), FP16_MAX), jit_scale(h_w, E4M3_MAX))


def encode_with(x: np.ndarray, fmt, s: np.float32, a: np.float32) -> ScaledTensor:
    codes = encode(np.asarray(x, dtype=np.float32) * F32(s), fmt)   # fl(x * s)
    return ScaledTensor(codes, fmt, F32(s), F32(F32(1.0) / F32(s)), F32(a))


def init_history(st: OptState) -> np.ndarray:
    """Ring of HIST exact amax(w) values; starts with amax(w0)."""
    h = np.zeros(HIST, dtype=np.float32)
    h[0] = st.master.amax
    return h


def adam_step_delayed(g_hat: np.ndarray, st: OptState, hp: AdamHP, g_scale_inv: np.float32,
                      w_hist: np.ndarray, step: int, skip: bool = False, bound: str = "recorded") -> Dict:
    """One FP8 AdamW step with delayed state scaling (one pass).  ``step`` >= 1 selects the
    history slot (step - 1) % HIST that receives this step's exact amax(w').
    Returns dict(state, hist, m, v, w, scales)."""
    if skip:
        return dict(state=st.copy(), hist=np.array(w_hist, np.float32), m=None, v=None, w=None)
    s_m, s_v, s_w, s_8 = delayed_scales(st, g_scale_inv, hp, w_hist, bound)
    g = np.asarray(g_hat, dtype=np.float32)
    m_new, v_new, w_new = adam_math(g, st.m1.value(), st.v.value(), st.master.value(), hp)
    am = F32(np.abs(m_new).max()) if m_new.size else F32(0.0)
    av = F32(v_new.max()) if v_new.size else F32(0.0)
    aw = F32(np.abs(w_new).max()) if w_new.size else F32(0.0)
    new = OptState(
        m1=encode_with(m_new, E4M3, s_m, am),
        v=encode_with(v_new, FP16, s_v, av),
        master=encode_with(w_new, FP16, s_w, aw),
        w8=encode_with(w_new, E4M3, s_8, aw),
    )
    hist = np.array(w_hist, dtype=np.float32)
    hist[(step - 1) % HIST] = aw
    return dict(state=new, hist=hist, m=m_new, v=v_new, w=w_new, scales=(s_m, s_v, s_w, s_8))
