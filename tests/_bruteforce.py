"""Independent second encoder used only to PIN the oracle codec (not part of the oracle).

Method: enumerate every finite code of the format, decode it from the bit fields
(sign, exponent, mantissa, bias) with a scalar formula of its own, sort, and for
each input pick the nearest grid value by |x - v| with exact rational comparison
(float64 holds every value involved exactly), ties to the code with even mantissa
LSB; saturate beyond max.  Shares nothing with oracle/codec.py's frexp/rint method.
"""
from __future__ import annotations

import math

import numpy as np


def _value(code: int, ebits: int, mbits: int, bias: int, ieee: bool):
    nbits = 1 + ebits + mbits
    s = (code >> (nbits - 1)) & 1
    e = (code >> mbits) & ((1 << ebits) - 1)
    m = code & ((1 << mbits) - 1)
    if ieee and e == (1 << ebits) - 1:
        return None                      # inf / NaN: not a finite grid point
    if (not ieee) and e == (1 << ebits) - 1 and m == (1 << mbits) - 1:
        return None                      # E4M3 NaN
    if e == 0:
        mag = math.ldexp(m, 1 - bias - mbits)
    else:
        mag = math.ldexp((1 << mbits) + m, e - bias - mbits)
    return -mag if s else mag


class BruteForce:
    def __init__(self, ebits, mbits, bias, ieee):
        self.nbits = 1 + ebits + mbits
        pos = []
        for c in range(1 << (self.nbits - 1)):
            v = _value(c, ebits, mbits, bias, ieee)
            if v is not None:
                pos.append((v, c))
        pos.sort()
        self.vals = np.array([v for v, _ in pos], dtype=np.float64)
        self.codes = np.array([c for _, c in pos], dtype=np.int64)
        self.maxval = self.vals[-1]

    def encode(self, x):
        with np.errstate(invalid="ignore"):
            x = np.asarray(x, dtype=np.float32).astype(np.float64)
        out = np.empty(x.shape, dtype=np.int64)
        neg = np.signbit(x)
        a = np.abs(x)
        nan = np.isnan(a)
        a = np.where(nan, 0.0, np.minimum(a, self.maxval))   # inf and above max -> max
        hi = np.searchsorted(self.vals, a, side="left")       # vals[hi] >= a
        hi = np.minimum(hi, len(self.vals) - 1)
        lo = np.maximum(hi - 1, 0)
        dlo = a - self.vals[lo]
        dhi = self.vals[hi] - a
        pick_hi = (dhi < dlo) | ((dhi == dlo) & ((self.codes[hi] & 1) == 0))
        pick_hi = np.where(self.vals[hi] == a, True, pick_hi)
        c = np.where(pick_hi, self.codes[hi], self.codes[lo])
        c = np.where(neg, c | (1 << (self.nbits - 1)), c)
        out[...] = c
        return out, nan


E4M3_BF = BruteForce(4, 3, 7, False)
E5M2_BF = BruteForce(5, 2, 15, True)
FP16_BF = BruteForce(5, 10, 15, True)
