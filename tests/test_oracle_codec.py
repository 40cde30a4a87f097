"""Pins of oracle/codec.py against what the paper and the mathematics fix (task rule ③).

* Table 5 ranges from a golden file.
* Exhaustive 256-code structure: classes, round trip, monotonicity.
* Every RNE midpoint, saturation thresholds, underflow threshold, NaN.
* An independent brute-force nearest-code encoder (tests/_bruteforce.py).
* Third-party encoders: torch clamp+cast (E4M3/E5M2; torch's casts do not
  saturate, so clamp first) and numpy float16 (after clamp).
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle.codec import E4M3, E5M2, FP16, codec_table, decode, encode
from tests._bruteforce import E4M3_BF, E5M2_BF, FP16_BF

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FMTS = {"e4m3": E4M3, "e5m2": E5M2, "f16": FP16}


def test_table5_ranges():
    g = json.load(open(os.path.join(GOLD, "table5_ranges.json")))
    for name, fmt in FMTS.items():
        row = g[name]
        maxv = float(decode([fmt.max_code], fmt)[0])
        assert maxv == row["max_normal"]
        # min normal = code with exponent field 1, mantissa 0; min subnormal = code 1
        minn = float(decode([1 << fmt.mbits], fmt)[0])
        mins = float(decode([1], fmt)[0])
        assert abs(minn - row["min_normal"]) / row["min_normal"] < 5e-3
        assert abs(mins - row["min_subnormal"]) / row["min_subnormal"] < 5e-3
        assert minn == fmt.min_normal and mins == fmt.min_subnormal


def test_e4m3_code_classes():
    rows = codec_table(E4M3)
    classes = [r[2] for r in rows]
    assert classes.count("nan") == 2 and rows[0x7F][2] == "nan" and rows[0xFF][2] == "nan"
    assert classes.count("inf") == 0
    assert classes.count("zero") == 2
    assert classes.count("subnormal") == 14           # mantissa 1..7, both signs
    assert rows[0x7E][1] == 448.0 and rows[0xFE][1] == -448.0
    assert rows[0x38][1] == 1.0                        # 2^(7-7)


def test_e5m2_code_classes():
    rows = codec_table(E5M2)
    classes = [r[2] for r in rows]
    assert classes.count("inf") == 2 and rows[0x7C][1] == np.inf and rows[0xFC][1] == -np.inf
    assert classes.count("nan") == 6
    assert rows[0x7B][1] == 57344.0
    assert rows[0x3C][1] == 1.0


@pytest.mark.parametrize("fmt", [E4M3, E5M2, FP16], ids=lambda f: f.name)
def test_roundtrip_and_monotone(fmt):
    codes = np.arange(1 << fmt.nbits)
    vals = decode(codes, fmt)
    finite = np.isfinite(vals)
    rt = encode(vals[finite].astype(np.float32), fmt)
    assert np.array_equal(rt.astype(np.int64), codes[finite])
    pos = np.arange(fmt.max_code + 1)
    assert np.all(np.diff(decode(pos, fmt)) > 0)


@pytest.mark.parametrize("fmt", [E4M3, E5M2, FP16], ids=lambda f: f.name)
def test_every_midpoint_ties_to_even(fmt):
    pos = np.arange(fmt.max_code + 1)
    v = decode(pos, fmt)
    mids = (v[:-1] + v[1:]) / 2.0                      # exact in float64
    mids32 = mids.astype(np.float32)
    assert np.array_equal(mids32.astype(np.float64), mids)   # midpoints are binary32 values
    got = encode(mids32, fmt).astype(np.int64)
    even = np.where(pos[:-1] % 2 == 0, pos[:-1], pos[1:])
    assert np.array_equal(got, even)
    assert np.array_equal(encode(-mids32, fmt).astype(np.int64), even | (1 << (fmt.nbits - 1)))
    # one binary32 ulp either side of the midpoint goes to the nearer code
    up = np.nextafter(mids32, np.float32(np.inf))
    dn = np.nextafter(mids32, np.float32(0))
    assert np.array_equal(encode(up, fmt).astype(np.int64), pos[1:])
    assert np.array_equal(encode(dn, fmt).astype(np.int64), pos[:-1])
    if fmt is E4M3:
        assert len(mids) == 126


def test_saturation_and_specials():
    f32 = np.float32
    # E4M3: 464 = 448 + half ulp is a tie -> even 448; anything larger saturates (satfinite)
    assert encode([f32(464.0)], E4M3)[0] == 0x7E
    assert encode([np.nextafter(f32(464.0), f32(1e9))], E4M3)[0] == 0x7E
    assert encode([f32(1e30), f32(np.inf), f32(-np.inf)], E4M3).tolist() == [0x7E, 0x7E, 0xFE]
    assert encode([f32(np.nan)], E4M3)[0] == 0x7F
    # E5M2 saturates instead of overflowing to inf (reading R11)
    assert encode([f32(61440.0), f32(59392.0), f32(np.inf)], E5M2).tolist() == [0x7B] * 3
    # FP16 satfinite
    assert encode([f32(65519.0), f32(65520.0), f32(1e9)], FP16).tolist() == [0x7BFF] * 3
    # underflow: half the min subnormal ties to zero; anything above rounds up
    h = f32(2.0 ** -10)
    assert encode([h, -h], E4M3).tolist() == [0x00, 0x80]
    assert encode([np.nextafter(h, f32(1))], E4M3)[0] == 0x01
    assert encode([f32(2.0 ** -17)], E5M2)[0] == 0
    assert encode([f32(-0.0)], E4M3)[0] == 0x80
    # binary32 subnormals flush to (signed) zero in every format
    tiny = np.array([1e-45, -1e-40], dtype=np.float32)
    assert encode(tiny, E4M3).tolist() == [0x00, 0x80]


def _probe_inputs(n_random=1 << 20, seed=0):
    """Structured + random binary32 inputs spanning every exponent and rounding case."""
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 1 << 32, size=n_random, dtype=np.uint64).astype(np.uint32)
    # structured: every exponent x top-5 mantissa bits x low-bit patterns, both signs
    e = np.arange(256, dtype=np.uint32)
    top = np.arange(32, dtype=np.uint32)
    low = np.array([0, 1, 0x1FFFF, 0x20000, 0x3FFFF, 0x3FFFE, 0x15555], dtype=np.uint32)
    E, Tm, L = np.meshgrid(e, top, low, indexing="ij")
    s = (E << 23) | (Tm << 18) | L
    s = np.concatenate([s.ravel(), s.ravel() | np.uint32(0x80000000)])
    return np.concatenate([bits, s]).view(np.float32)


@pytest.mark.parametrize("fmt,bf", [(E4M3, E4M3_BF), (E5M2, E5M2_BF), (FP16, FP16_BF)],
                         ids=["e4m3", "e5m2", "f16"])
def test_vs_bruteforce_nearest_code(fmt, bf):
    x = _probe_inputs()
    got = encode(x, fmt).astype(np.int64)
    ref, nan = bf.encode(x)
    assert np.array_equal(got[~nan], ref[~nan])
    assert np.all(np.isnan(decode(got[nan], fmt)))


def _torch_ref(x, fmt):
    t = torch.from_numpy(x)
    if fmt is E4M3:
        return t.clamp(-448, 448).to(torch.float8_e4m3fn).view(torch.uint8).numpy().astype(np.int64)
    if fmt is E5M2:
        return t.clamp(-57344, 57344).to(torch.float8_e5m2).view(torch.uint8).numpy().astype(np.int64)
    return np.clip(x, -65504, 65504).astype(np.float16).view(np.uint16).astype(np.int64)


@pytest.mark.parametrize("fmt", [E4M3, E5M2, FP16], ids=lambda f: f.name)
def test_vs_third_party_casts(fmt):
    x = _probe_inputs(seed=1)
    got = encode(x, fmt).astype(np.int64)
    ref = _torch_ref(x, fmt)
    nan = np.isnan(x)
    assert np.array_equal(got[~nan], ref[~nan])


@pytest.mark.slow
@pytest.mark.parametrize("fmt", [E4M3, E5M2], ids=lambda f: f.name)
def test_exhaustive_2pow32_vs_torch(fmt):
    """All 2^32 binary32 bit patterns (opt-in: -m slow; several minutes)."""
    chunk = 1 << 24
    for start in range(0, 1 << 32, chunk):
        x = np.arange(start, start + chunk, dtype=np.uint64).astype(np.uint32).view(np.float32)
        got = encode(x, fmt).astype(np.int64)
        ref = _torch_ref(x, fmt)
        nan = np.isnan(x)
        assert np.array_equal(got[~nan], ref[~nan]), hex(start)
