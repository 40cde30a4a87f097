"""Oracle codec: FP8 E4M3 / E5M2 and FP16, decode + saturating round-to-nearest-even encode.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions (App. A, P:741-745 and Table 5):
  * E4M3: 1 sign, 4 exponent, 3 mantissa bits; "values up to +/-448 and NaN".
    No infinities; exponent-all-ones is used for finite values and only
    S.1111.111 is NaN (so that 448 = 1.75 * 2^8 is representable).  Bias 7.
    Min normal 2^-6 = 1.56e-2, min subnormal 2^-9 = 1.95e-3 (Table 5).
  * E5M2: 1 sign, 5 exponent, 2 mantissa bits; "values up to +/-57344, +/- inf and
    NaN".  IEEE-style: exponent-all-ones is inf (mantissa 0) or NaN.  Bias 15.
    Min normal 2^-14 = 6.10e-5, min subnormal 2^-16 = 1.53e-5 (Table 5).
  * FP16 (IEEE binary16, S1E5M10), max 65504, min normal 6.10e-5, min subnormal
    5.96e-8 (Table 5) — used for the second moment and master weights.

Encode reading (R11): round-to-nearest-even on the exact input value,
then SATURATE: any value whose rounded magnitude exceeds the format's max, and
+/-inf, become +/-max ("satfinite").  NaN becomes the canonical NaN code.  Values
at or below half the minimum subnormal become signed zero (the tie goes to the
even code, zero).  The paper fixes no rounding mode; FP8 "roughly follows the IEEE
754 standard" whose default is RNE.

Implementation: one generic mini-float routine parameterised by (exponent bits,
mantissa bits, bias, max); all arithmetic in float64, where every binary32 input
and every grid point of the three formats is exact, so the only rounding is the
explicit ``np.rint`` (round half to even) on the grid index.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Format:
    name: str
    ebits: int
    mbits: int
    bias: int
    maxval: float
    ieee_specials: bool     # True: exponent all-ones = inf/NaN (E5M2, FP16); False: E4M3
    nan_code: int           # canonical (positive) NaN code produced by encode

    @property
    def nbits(self) -> int:
        return 1 + self.ebits + self.mbits

    @property
    def emin(self) -> int:           # exponent of the min normal
        return 1 - self.bias

    @property
    def min_normal(self) -> float:
        return 2.0 ** self.emin

    @property
    def min_subnormal(self) -> float:
        return 2.0 ** (self.emin - self.mbits)

    @property
    def max_code(self) -> int:       # positive code of +max
        return self.encode_scalar(self.maxval)

    def encode_scalar(self, x: float) -> int:
        return int(encode(np.array([x], dtype=np.float64), self, _allow_f64=True)[0])


E4M3 = Format("e4m3", 4, 3, 7, 448.0, False, 0x7F)
E5M2 = Format("e5m2", 5, 2, 15, 57344.0, True, 0x7E)
FP16 = Format("f16", 5, 10, 15, 65504.0, True, 0x7E00)


def _code_dtype(fmt: Format):
    return np.uint8 if fmt.nbits == 8 else np.uint16


def decode(codes, fmt: Format) -> np.ndarray:
    """Exact value of each code as float64: (-1)^s * 2^(e-bias) * (1 + m/2^M), or the
    subnormal 2^(1-bias) * m/2^M when e == 0; NaN / inf codes per the format."""
    c = np.asarray(codes).astype(np.int64)
    sign = (c >> (fmt.nbits - 1)) & 1
    e = (c >> fmt.mbits) & ((1 << fmt.ebits) - 1)
    m = c & ((1 << fmt.mbits) - 1)
    emax_field = (1 << fmt.ebits) - 1
    normal = np.ldexp(1.0 + m / float(1 << fmt.mbits), (e - fmt.bias).astype(np.int64))
    subnormal = np.ldexp(m.astype(np.float64), fmt.emin - fmt.mbits)
    v = np.where(e == 0, subnormal, normal)
    if fmt.ieee_specials:
        v = np.where((e == emax_field) & (m == 0), np.inf, v)
        v = np.where((e == emax_field) & (m != 0), np.nan, v)
    else:
        v = np.where((e == emax_field) & (m == (1 << fmt.mbits) - 1), np.nan, v)
    return np.where(sign == 1, -v, v)


def encode(x, fmt: Format, _allow_f64: bool = False) -> np.ndarray:
    """Saturating RNE encode of binary32 values (R11).  Returns uint8 / uint16 codes."""
    x = np.asarray(x)
    if not _allow_f64:
        x = x.astype(np.float32)        # the method quantizes binary32 values
    with np.errstate(invalid="ignore"):
        a64 = np.abs(x.astype(np.float64))
    neg = np.signbit(x)
    nan = np.isnan(a64)
    inf = np.isinf(a64)
    fin = ~(nan | inf)
    a = np.where(fin, a64, 0.0)

    # binade exponent e = floor(log2 a), clamped below at the min-normal exponent
    _, E = np.frexp(a)                      # a = f * 2^E with f in [0.5, 1)
    e = np.maximum(E.astype(np.int64) - 1, fmt.emin)
    ulp = np.ldexp(1.0, e - fmt.mbits)      # grid spacing in that binade
    q = np.rint(a / ulp)                    # round half to even (exact division)
    v = q * ulp                             # rounded magnitude (exact)
    v = np.where(inf, np.inf, v)
    v = np.minimum(v, fmt.maxval)           # satfinite: overflow and inf -> max

    # bit pattern of the (exactly representable) magnitude v
    sub = v < fmt.min_normal
    mant_sub = np.rint(v / fmt.min_subnormal).astype(np.int64)
    _, E2 = np.frexp(np.where(sub, 1.0, v))
    exp_field = E2.astype(np.int64) - 1 + fmt.bias
    frac = np.ldexp(np.where(sub, 1.0, v), -(E2.astype(np.int64) - 1)) - 1.0
    mant_norm = np.rint(frac * (1 << fmt.mbits)).astype(np.int64)
    mag = np.where(sub, mant_sub, (exp_field << fmt.mbits) | mant_norm)
    code = np.where(neg, mag | (1 << (fmt.nbits - 1)), mag)
    code = np.where(nan, fmt.nan_code, code)
    return code.astype(_code_dtype(fmt))


def roundtrip(x, fmt: Format) -> np.ndarray:
    """decode(encode(x)) as float64."""
    return decode(encode(x, fmt), fmt)


def is_nan_code(codes, fmt: Format) -> np.ndarray:
    return np.isnan(decode(codes, fmt))


def code_class(code: int, fmt: Format) -> str:
    v = float(decode(np.array([code]), fmt)[0])
    if np.isnan(v):
        return "nan"
    if np.isinf(v):
        return "inf"
    if v == 0.0:
        return "zero"
    return "subnormal" if abs(v) < fmt.min_normal else "normal"


def codec_table(fmt: Format):
    """All 2^8 codes as rows (bits_hex, value, class) — SPEC.md's codec-table idea."""
    assert fmt.nbits == 8
    vals = decode(np.arange(256), fmt)
    return [(f"0x{c:02X}", float(vals[c]), code_class(c, fmt)) for c in range(256)]


# float32 helpers for the pipeline: decode to binary32 (exact for every FP8/FP16 value)
def decode_f32(codes, fmt: Format) -> np.ndarray:
    return decode(codes, fmt).astype(np.float32)


if __name__ == "__main__":   # python -m oracle.codec e4m3
    import sys
    f = {"e4m3": E4M3, "e5m2": E5M2}[sys.argv[1] if len(sys.argv) > 1 else "e4m3"]
    print("bits_hex,value,class")
    for row in codec_table(f):
        print(f"{row[0]},{row[1]!r},{row[2]}")
