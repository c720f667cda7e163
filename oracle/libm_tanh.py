"""Python restatement of the host libm's double tanh (the device copy is
paper_1611_09482_b200/csrc/libm_tanh.cuh).

TEST INFRASTRUCTURE ONLY: tests/test_oracle_plain.py checks it against
math.tanh, which is what the reference's numba kernel calls (kernel.py:54-55),
to pin the algorithm the device port follows: fdlibm's tanh over expm1 with
glibc's Estrin evaluation of expm1's correction polynomial, compiled with a*b+c
contracted to fused multiply-adds (as glibc's x86-64 build is). Exact FMA is
emulated with rationals; every other operation is a plain IEEE double op.
"""

from __future__ import annotations

import math
import struct
from fractions import Fraction


def _fma(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))  # one rounding


def _hi(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0] >> 32


def _from_hi(h: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", (h & 0xFFFFFFFF) << 32))[0]


LN2_HI, LN2_LO, INVLN2 = 6.93147180369123816490e-01, 1.90821492927058770002e-10, 1.44269504088896338700e+00
Q1, Q2, Q3 = -3.33333333333331316428e-02, 1.58730158725481460165e-03, -7.93650757867487942473e-05
Q4, Q5 = 4.00821782732936239552e-06, -2.01099218183624371326e-07


def expm1(x: float) -> float:
    """fdlibm expm1 for the arguments tanh passes (|x| <= 44)."""
    hx = _hi(x)
    xsb, hx = hx & 0x80000000, hx & 0x7FFFFFFF
    if hx >= 0x4043687A and xsb:
        return -1.0
    c, k = 0.0, 0
    if hx > 0x3FD62E42:
        if hx < 0x3FF0A2B2:
            hi, lo, k = (x - LN2_HI, LN2_LO, 1) if not xsb else (x + LN2_HI, -LN2_LO, -1)
        else:
            k = int(_fma(INVLN2, x, -0.5 if xsb else 0.5))
            t = float(k)
            hi, lo = _fma(-t, LN2_HI, x), t * LN2_LO
        x = hi - lo
        c = (hi - x) - lo
    elif hx < 0x3C900000:
        return x
    hfx = 0.5 * x
    hxs = x * hfx
    r1 = _fma(hxs * hxs * (hxs * hxs), _fma(hxs, Q5, Q4),
              _fma(hxs * hxs, _fma(hxs, Q3, Q2), _fma(hxs, Q1, 1.0)))
    t = _fma(-r1, hfx, 3.0)
    e = hxs * ((r1 - t) / _fma(-x, t, 6.0))
    if k == 0:
        return x - _fma(x, e, -hxs)
    twopk = _from_hi(0x3FF00000 + (k << 20))
    e = _fma(x, e - c, -c) - hxs
    if k == -1:
        return _fma(0.5, x - e, -0.5)
    if k == 1:
        return -2.0 * (e - (x + 0.5)) if x < -0.25 else _fma(2.0, x - e, 1.0)
    if k <= -2 or k > 56:
        return (1.0 - (e - x)) * twopk - 1.0
    if k < 20:
        return (_from_hi(0x3FF00000 - (0x200000 >> k)) - (e - x)) * twopk
    return ((x - (e + _from_hi((0x3FF - k) << 20))) + 1.0) * twopk


def tanh(x: float) -> float:
    jx = _hi(x)
    ix = jx & 0x7FFFFFFF
    if ix >= 0x7FF00000:
        return math.tanh(x)
    if ix < 0x40360000:
        if x == 0.0:
            return x
        if ix < 0x3C800000:
            return x * (1.0 + x)
        if ix >= 0x3FF00000:
            z = 1.0 - 2.0 / (expm1(2.0 * abs(x)) + 2.0)
        else:
            t = expm1(-2.0 * abs(x))
            z = -t / (t + 2.0)
    else:
        z = 1.0
    return -z if jx & 0x80000000 else z
