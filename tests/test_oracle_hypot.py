"""Pins for the oracle's v1_hypot (Listing 2).

Nothing here re-calls the oracle's own arithmetic as the expected value: the
expectations are closed forms, IEEE facts, or ``ieee_exact`` (an independent
exact-rational implementation of every IEEE operation)."""
import math
import struct

import mpmath
import numpy as np
import pytest

import ieee_exact as ie
import oracle

rng = np.random.default_rng(20250906)
DMAX = np.finfo(np.float64).max
DMIN_SUB = 5e-324
SMAX = float(np.finfo(np.float32).max)
SMIN_SUB = float(np.float32(1.4e-45))


def d2b(x):
    return struct.unpack("<Q", struct.pack("<d", float(x)))[0]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("x,y,h", [(3, 4, 5), (6, 8, 10), (0.75, 1.0, 1.25), (3 * 2.0 ** 40, 2.0 ** 42, 5 * 2.0 ** 40),
                                   (3 * 2.0 ** -40, 2.0 ** -38, 5 * 2.0 ** -40)])
def test_pythagorean_triples_exact(dt, x, y, h):
    # q = 3/4 is dyadic: S = 1 + 9/16 = 25/16 and s = 5/4 are exact, so h = M*s = h exactly.
    assert oracle.v1_hypot(x, y, dt) == h
    assert oracle.v1_hypot(-y, x, dt) == h


@pytest.mark.parametrize("bits", [64, 32])
@pytest.mark.parametrize("x,y,h", [(5, 12, 13), (8, 15, 17), (20, 21, 29), (7, 24, 25)])
def test_pythagorean_triples_non_dyadic(bits, x, y, h):
    # q = m/M is inexact: the result is the exact-rational Listing 2 value, within 2 ulp of h.
    dt = np.float64 if bits == 64 else np.float32
    r = float(oracle.v1_hypot(x, y, dt))
    assert ie.same(r, ie.v1_hypot(float(x), float(y), bits), bits)
    ulp = math.ulp(h) if bits == 64 else float(np.spacing(np.float32(h)))
    assert abs(r - h) <= 2 * ulp


@pytest.mark.parametrize("dt,tiny,big", [(np.float64, DMIN_SUB, DMAX), (np.float32, SMIN_SUB, SMAX)])
def test_zero_identity_and_zero_zero(dt, tiny, big):
    # v1(x, 0) = |x| exactly: q = 0, S = 1, s = 1, h = M
    for x in [1.0, -2.5, tiny, -tiny, big, -big, 1e-30, 3.0e30]:
        x = float(dt(x))
        assert ie.same(oracle.v1_hypot(x, 0.0, dt), abs(x), 64 if dt == np.float64 else 32)
        assert ie.same(oracle.v1_hypot(0.0, x, dt), abs(x), 64 if dt == np.float64 else 32)
    # v1(0,0): q = 0/0 = NaN, Q = fmax(NaN, 0) = 0, S=1, h = +0
    for a, b in [(0.0, 0.0), (-0.0, 0.0), (-0.0, -0.0)]:
        r = oracle.v1_hypot(a, b, dt)
        assert r == 0 and math.copysign(1.0, float(r)) == 1.0


def test_v1_equal_arguments_sqrt2():
    # v1(1,1): q=1, S=2, s=RN(sqrt 2) = 0x3FF6A09E667F3BCD (IEEE sqrt of 2)
    assert d2b(oracle.v1_hypot(1.0, 1.0)) == 0x3FF6A09E667F3BCD
    assert oracle.v1_hypot(1.0, 1.0) == math.sqrt(2.0)
    # v1(sqrt2, sqrt2) = RN(sqrt2 * RN(sqrt2)) = 2 + 2^-51 (exact-rational check)
    s2 = math.sqrt(2.0)
    assert oracle.v1_hypot(s2, s2) == 2.0 + 2.0 ** -51
    assert ie.v1_hypot(s2, s2) == 2.0 + 2.0 ** -51


@pytest.mark.parametrize("bits", [64, 32])
def test_matches_exact_rational_ieee(bits):
    """20k pairs over many magnitude regimes: oracle (gcc/glibc) == exact IEEE."""
    dt = np.float64 if bits == 64 else np.float32
    n = 4000
    emax = 1023 if bits == 64 else 127
    emin = -1074 if bits == 64 else -149
    pairs = []
    # (a) moderate uniform
    pairs += list(zip(rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)))
    # (b) wide exponents, independent
    e1 = rng.integers(emin, emax, n)
    e2 = rng.integers(emin, emax, n)
    pairs += list(zip(np.ldexp(rng.uniform(1, 2, n), e1), np.ldexp(rng.uniform(1, 2, n), e2)))
    # (c) close exponents (q near 1, the rounding-sensitive regime)
    e = rng.integers(emin + 60, emax - 2, n)
    pairs += list(zip(np.ldexp(rng.uniform(1, 2, n), e), np.ldexp(rng.uniform(1, 2, n), e + rng.integers(-3, 3, n))))
    # (d) subnormal / tiny pairs
    t = np.ldexp(1.0, emin)
    pairs += list(zip(rng.integers(0, 2 ** 20, n) * t, rng.integers(0, 2 ** 20, n) * t))
    # (e) q tiny around the S==1 threshold (q ~ 2^-27 .. 2^-26 for fp64)
    thr = -27 if bits == 64 else -12
    pairs += list(zip(np.ldexp(rng.uniform(1, 2, n), thr + rng.integers(-2, 2, n)), rng.uniform(1, 2, n)))
    mism = 0
    for x, y in pairs:
        x, y = float(dt(x)), float(dt(y))
        if not (math.isfinite(x) and math.isfinite(y)):
            continue
        got = float(oracle.v1_hypot(x, y, dt))
        exp = ie.v1_hypot(x, y, bits)
        if not ie.same(got, exp, bits):
            mism += 1
    assert mism == 0


@pytest.mark.parametrize("bits", [64, 32])
def test_special_values_reading_R4(bits):
    """Listing 2 taken literally for non-finite inputs (reading R4)."""
    dt = np.float64 if bits == 64 else np.float32
    inf, nan = float("inf"), float("nan")
    s2 = math.sqrt(2.0) if bits == 64 else float(np.sqrt(np.float32(2.0)))
    cases = [
        ((nan, 3.0), ie.mul(3.0, s2, bits)),  # m=M=3 -> q=1 -> S=2 -> 3*RN(sqrt2)
        ((nan, 0.0), 0.0),                     # m=M=0 -> q NaN -> Q=0 -> +0
        ((inf, 3.0), inf), ((3.0, -inf), inf), ((inf, inf), inf),
        ((inf, nan), inf), ((inf, 0.0), inf),
    ]
    for (x, y), exp in cases:
        got = float(oracle.v1_hypot(x, y, dt))
        assert ie.same(got, exp, bits), (x, y, got, exp)
        assert ie.same(got, ie.v1_hypot(x, y, bits), bits)
    assert math.isnan(float(oracle.v1_hypot(nan, nan, dt)))


@pytest.mark.parametrize("bits", [64, 32])
def test_symmetry_bitwise(bits):
    dt = np.float64 if bits == 64 else np.float32
    xs = np.ldexp(rng.uniform(-2, 2, 3000), rng.integers(-60, 60, 3000)).astype(dt)
    ys = np.ldexp(rng.uniform(-2, 2, 3000), rng.integers(-60, 60, 3000)).astype(dt)
    for x, y in zip(xs, ys):
        a = oracle.v1_hypot(x, y, dt)
        for b in (oracle.v1_hypot(y, x, dt), oracle.v1_hypot(-x, y, dt), oracle.v1_hypot(x, -y, dt),
                  oracle.v1_hypot(-y, -x, dt)):
            assert ie.same(float(a), float(b), bits)


@pytest.mark.parametrize("bits", [64, 32])
def test_reH_envelope(bits):
    """e:reH: (1+eps'-) < v1/hypot < (1+eps'+) on random pairs."""
    dt = np.float64 if bits == 64 else np.float32
    mpmath.mp.prec = 300
    eps = mpmath.mpf(2) ** (-53 if bits == 64 else -24)
    lo = (1 - eps) ** mpmath.mpf(2.5) * mpmath.sqrt(1 - eps * (2 - eps) / 2)
    hi = (1 + eps) ** mpmath.mpf(2.5) * mpmath.sqrt(1 + eps * (2 + eps) / 2)
    n = 20000
    xs = np.ldexp(rng.uniform(-2, 2, n), rng.integers(-30, 30, n)).astype(dt)
    ys = np.ldexp(rng.uniform(-2, 2, n), rng.integers(-30, 30, n)).astype(dt)
    worst = mpmath.mpf(0)
    for x, y in zip(xs, ys):
        if x == 0 and y == 0:
            continue
        h = mpmath.mpf(float(oracle.v1_hypot(x, y, dt)))
        H = mpmath.sqrt(mpmath.mpf(float(x)) ** 2 + mpmath.mpf(float(y)) ** 2)
        r = h / H
        assert lo < r < hi
        worst = max(worst, abs(r - 1) / eps)
    assert worst < 3.0  # first-order size of the envelope (~3 eps)


def test_monotone_in_each_argument():
    """A hypot suited for the method is non-decreasing in |x|, |y|;
    sampled on a grid for v1_hypot."""
    y = 0.7
    grid = np.sort(rng.uniform(0, 3, 10000))
    vals = [oracle.v1_hypot(g, y) for g in grid]
    assert all(a <= b for a, b in zip(vals, vals[1:]))


def test_no_spurious_overflow_or_underflow():
    # (1.2e308, 1.2e308): true value 1.697e308 < DBL_MAX; q <= 1 so nothing
    # intermediate overflows; h = RN(1.2e308 * RN(sqrt2)) is finite.
    h = oracle.v1_hypot(1.2e308, 1.2e308)
    assert math.isfinite(h) and abs(h / (1.2e308 * math.sqrt(2.0)) - 1) < 1e-15
    # the true value above DBL_MAX overflows to +inf (correct, not spurious)
    assert oracle.v1_hypot(1.5e308, 1.5e308) == float("inf")
    # tiny normals: no flush to zero
    t = 2.0 ** -1000
    assert oracle.v1_hypot(3 * t, 4 * t) == 5 * t
    # subnormal pair (inexact underflow regime): still nonzero
    assert oracle.v1_hypot(DMIN_SUB, DMIN_SUB) == DMIN_SUB


@pytest.mark.parametrize("bits", [64, 32])
def test_cr_hypot_is_exact_rounding(bits):
    """oracle cr_hypot == RN(sqrt(x^2+y^2)) computed by the independent
    exact-rational code (ieee_exact), incl. subnormal, huge and close pairs."""
    dt = np.float64 if bits == 64 else np.float32
    emin, emax = (-1074, 1020) if bits == 64 else (-149, 125)
    n = 3000
    xs = np.concatenate([rng.uniform(-2, 2, n), np.ldexp(rng.uniform(1, 2, n), rng.integers(emin, emax, n)),
                         rng.integers(1, 1 << 20, n) * np.ldexp(1.0, emin)]).astype(dt)
    ys = np.concatenate([rng.uniform(-2, 2, n), np.ldexp(rng.uniform(1, 2, n), rng.integers(emin, emax, n)),
                         rng.integers(1, 1 << 20, n) * np.ldexp(1.0, emin)]).astype(dt)
    ys[:500] = (xs[:500] * dt(1.0000001)).astype(dt)
    got = oracle.cr_hypot_array(xs, ys)
    for x, y, g in zip(xs, ys, got):
        if not (math.isfinite(x) and math.isfinite(y)):
            continue
        assert ie.same(float(g), ie.exact_norm([float(x), float(y)], bits), bits)


def test_cr_hypot_specials_and_closed_forms():
    inf, nan = float("inf"), float("nan")
    assert oracle.cr_hypot(3, 4) == 5 and oracle.cr_hypot(5, 12) == 13 and oracle.cr_hypot(8, 15) == 17
    assert oracle.cr_hypot(1, 1) == math.sqrt(2.0)
    assert oracle.cr_hypot(inf, nan) == inf and oracle.cr_hypot(nan, -inf) == inf
    assert math.isnan(oracle.cr_hypot(nan, 1.0))
    assert oracle.cr_hypot(-2.5, 0.0) == 2.5 and oracle.cr_hypot(0.0, 0.0) == 0.0
    assert oracle.cr_hypot(1.5e308, 1.5e308) == inf and math.isfinite(oracle.cr_hypot(1.2e308, 1.2e308))
    assert oracle.cr_hypot(DMAX, 1.0) == DMAX
