"""Exact-rational IEEE-754 binary64/binary32 arithmetic for pinning the oracle.

Written independently of ``oracle/``: every operation is computed exactly with
``fractions.Fraction`` and rounded once, to nearest-even, by ``rn`` below (with
gradual underflow and overflow to infinity), following the IEEE-754 rules for
special operands.  ``v1_hypot`` then restates Listing 2
on top of these operations, so a mistake in the C oracle's compilation (a
contracted fma, FTZ, x87 double rounding, a wrong min/max NaN rule) shows up
as a bit mismatch.
"""
from __future__ import annotations

import math
import struct
from fractions import Fraction

import numpy as np

FMT = {
    64: dict(prec=53, emin=-1022, emax=1023),
    32: dict(prec=24, emin=-126, emax=127),
}
INF, NAN = float("inf"), float("nan")


def rn(v: Fraction, bits: int = 64) -> float:
    """Round the exact rational v to the nearest binary{bits} value (ties to even)."""
    f = FMT[bits]
    if v == 0:
        return 0.0
    sign = -1.0 if v < 0 else 1.0
    a = abs(v)
    # exponent e with 2^e <= a < 2^(e+1)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    qe = max(e - (f["prec"] - 1), f["emin"] - (f["prec"] - 1))
    q = Fraction(2) ** qe
    m = a / q
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    if fl == 0:
        return sign * 0.0
    if fl.bit_length() + qe > f["emax"] + 1:
        return sign * INF
    val = math.ldexp(fl, qe)
    if bits == 32:
        val = float(np.float32(val))  # exact: val is representable
    return sign * val


def rn_sqrt(v: Fraction, bits: int = 64) -> float:
    """RN(sqrt(v)) exactly, v >= 0."""
    if v == 0:
        return 0.0
    f = FMT[bits]
    # sqrt(v) in [2^e, 2^(e+1))
    e = (v.numerator.bit_length() - v.denominator.bit_length()) // 2
    while Fraction(2) ** (2 * e) > v:
        e -= 1
    while Fraction(2) ** (2 * e + 2) <= v:
        e += 1
    qe = max(e - (f["prec"] - 1), f["emin"] - (f["prec"] - 1))
    # floor(sqrt(v) / 2^qe) = isqrt(floor(v / 4^qe))
    w = v / (Fraction(2) ** (2 * qe))
    fl = math.isqrt(w.numerator // w.denominator)
    half = Fraction(2 * fl + 1, 2)
    if half * half < w or (half * half == w and fl % 2 == 1):
        fl += 1
    if fl.bit_length() + qe > f["emax"] + 1:
        return INF
    val = math.ldexp(fl, qe)
    if bits == 32:
        val = float(np.float32(val))
    return val


def _isnan(x):
    return x != x


def fmin(x, y):  # IEEE minNum: a NaN operand is ignored
    if _isnan(x):
        return y
    if _isnan(y):
        return x
    return x if x <= y else y


def fmax(x, y):
    if _isnan(x):
        return y
    if _isnan(y):
        return x
    return x if x >= y else y


def div(x, y, bits=64):
    if _isnan(x) or _isnan(y):
        return NAN
    if math.isinf(x) and math.isinf(y):
        return NAN
    if x == 0 and y == 0:
        return NAN
    sgn = math.copysign(1.0, x) * math.copysign(1.0, y)
    if math.isinf(x):
        return sgn * INF
    if math.isinf(y):
        return sgn * 0.0
    if y == 0:
        return sgn * INF
    r = rn(Fraction(x) / Fraction(y), bits)
    return math.copysign(abs(r), sgn) if r == 0 else r


def fma(a, b, c, bits=64):
    if _isnan(a) or _isnan(b) or _isnan(c):
        return NAN
    if math.isinf(a) or math.isinf(b) or math.isinf(c):
        prod = a * b  # exact enough for the sign/inf decision here
        if _isnan(prod):
            return NAN
        s = prod + c
        return s
    return rn(Fraction(a) * Fraction(b) + Fraction(c), bits)


def sqrt(x, bits=64):
    if _isnan(x) or x < 0:
        return NAN
    if math.isinf(x):
        return INF
    return rn_sqrt(Fraction(x), bits)


def mul(x, y, bits=64):
    if _isnan(x) or _isnan(y):
        return NAN
    if (math.isinf(x) and y == 0) or (math.isinf(y) and x == 0):
        return NAN
    if math.isinf(x) or math.isinf(y):
        return math.copysign(1.0, x) * math.copysign(1.0, y) * INF
    return rn(Fraction(x) * Fraction(y), bits)


def v1_hypot(x: float, y: float, bits: int = 64) -> float:
    """Listing 2 on exact-rational IEEE operations."""
    X, Y = abs(x), abs(y)
    m, M = fmin(X, Y), fmax(X, Y)
    q = div(m, M, bits)
    Q = fmax(q, 0.0)
    S = fma(Q, Q, 1.0, bits)
    s = sqrt(S, bits)
    return mul(M, s, bits)


def exact_norm(xs, bits: int = 64) -> float:
    """RN(sqrt(sum x_i^2)) with exact rational arithmetic (finite inputs)."""
    S = sum((Fraction(float(v)) ** 2 for v in xs), Fraction(0))
    return rn_sqrt(S, bits)


def bits_of(x: float, bits: int = 64) -> int:
    if bits == 64:
        return struct.unpack("<Q", struct.pack("<d", x))[0]
    return struct.unpack("<I", struct.pack("<f", x))[0]


def same(a: float, b: float, bits: int = 64) -> bool:
    """Bitwise equality (NaNs compare by being NaN)."""
    if _isnan(a) and _isnan(b):
        return True
    return bits_of(float(a), bits) == bits_of(float(b), bits)
