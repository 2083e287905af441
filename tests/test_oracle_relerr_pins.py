"""Value pins for oracle.relerr (e:relerr) and for the
e:reH / Thm-3 bound at eps_S.

Every accuracy gate of the suite ("<= 64 eps", "< 3 eps", "<= Thm-3 bound")
runs through these two functions, so they are pinned against values fixed by
the definitions themselves, not against their own formulas:

* relerr: results exactly one or two units of eps_x away from a power of two
  (the spacing of the floats there is 2 eps_x above and eps_x below, P:67-69,
  and numpy's finfo states the machine epsilon 2 eps_x independently), the
  operand order (the exact norm is the denominator, e:relerr), binade
  invariance, and the degenerate cases.
* the bound: a second-order Taylor expansion of e:reH worked by hand,
  (1+e)^(5/2) sqrt(1 + e(2+e)/2) = 1 + 3e + (13/4) e^2 + O(e^3), and of its
  d-th power, 1 + 3d e + (13d/4 + 9 d(d-1)/2) e^2 + O(e^3); a wrong eps_S
  (e.g. 2^-23) moves the second-order term by ~2e-7 and fails.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import bounds

F64, F32 = np.float64, np.float32


def test_eps_is_half_the_machine_epsilon():
    # eps_S = 2^-24, eps_D = 2^-53 (rounding to nearest); numpy's
    # finfo.eps is the gap between 1 and the next float, 2 eps_x
    assert oracle.EPS[np.dtype(F64)] == np.finfo(F64).eps / 2 == 2.0 ** -53
    assert oracle.EPS[np.dtype(F32)] == float(np.finfo(F32).eps) / 2 == 2.0 ** -24


@pytest.mark.parametrize("dt", [F64, F32])
def test_relerr_one_spacing_above_one_is_two(dt):
    up = np.nextafter(dt(1), dt(2))                     # 1 + 2 eps_x
    assert float(up) == 1 + float(np.finfo(dt).eps)
    assert oracle.relerr(up, dt(1), dt) == 2.0
    down = np.nextafter(dt(1), dt(0))                   # 1 - eps_x
    assert oracle.relerr(down, dt(1), dt) == 1.0


def test_relerr_literal_values():
    # the two pins of VERDICT r1: one ulp above 1 in each precision is 2 eps_x
    assert oracle.relerr(F32(1 + 2.0 ** -23), 1.0, F32) == 2.0
    assert oracle.relerr(1 + 2.0 ** -52, 1.0) == 2.0
    # the same in the fp32 scale is 2^29 eps_D when read as fp64
    assert oracle.relerr(F32(1 + 2.0 ** -23), 1.0, F64) == 2.0 ** 30


@pytest.mark.parametrize("dt", [F64, F32])
@pytest.mark.parametrize("k", [-1000, -100, -3, 0, 7, 60, 1000])
def test_relerr_binade_invariance(dt, k):
    if dt == F32:
        k = max(-120, min(120, k))
    ref = np.ldexp(dt(1), k)
    r = np.nextafter(ref, dt(np.inf))
    assert oracle.relerr(r, ref, dt) == 2.0
    r2 = np.nextafter(r, dt(np.inf))
    assert oracle.relerr(r2, ref, dt) == 4.0


def test_relerr_denominator_is_the_exact_norm():
    # e:relerr divides by ||x||'_F (the exact value), not by the computed one
    one, up = 1.0, 1 + 2.0 ** -52
    assert oracle.relerr(up, one) == 2.0
    below = oracle.relerr(one, up)
    assert below < 2.0
    assert below == float(Fraction(2) / (1 + Fraction(1, 2 ** 52)))


def test_relerr_degenerate():
    assert oracle.relerr(0.0, 0.0) == 0.0
    assert oracle.relerr(1e-300, 0.0) == float("inf")
    assert oracle.relerr(3.0, 3.0, F32) == 0.0
    # the sign of the difference does not matter
    assert oracle.relerr(1.0 - 2.0 ** -53, 1.0) == oracle.relerr(1.0 + 2.0 ** -52, 1.0) / 2


def _taylor_reH_pow(d: int, e: Fraction) -> Fraction:
    """((1+e)^(5/2) sqrt(1+e(2+e)/2))^d = 1 + 3d e + (13d/4 + 9 d(d-1)/2) e^2 + O(e^3),
    worked by hand: (1+e)^(5/2) = 1 + 5e/2 + 15e^2/8 + ..., sqrt(1 + e + e^2/2)
    = 1 + e/2 + e^2/8 + ..., product 1 + 3e + 13e^2/4 + ...; the d-th power of
    1 + a e + b e^2 is 1 + d a e + (d b + d(d-1)/2 a^2) e^2 + ..."""
    return 1 + 3 * d * e + (Fraction(13, 4) * d + Fraction(9, 2) * d * (d - 1)) * e * e


@pytest.mark.parametrize("dt,bits", [(F32, 32), (F64, 64)])
@pytest.mark.parametrize("d", [1, 2, 12, 30])
def test_reH_bound_second_order(dt, bits, d):
    e = Fraction(1, 2 ** (24 if bits == 32 else 53))
    want = float((_taylor_reH_pow(d, e) - 1) / e)       # in units of eps
    # the neglected terms are O(d^3 e^2): < 1e-9 for d <= 30 at eps_S
    assert abs(oracle.ub_relerr_H(d, dt) - want) < 1e-9
    assert abs(bounds.ub_depths(d, 0, bits) - want) < 1e-9
    lo, hi = bounds.hypot_envelope("v1", bits)
    assert abs(float((hi - 1) / bounds._eps(bits)) - float((_taylor_reH_pow(1, e) - 1) / e)) < 1e-12


def test_reH_bound_eps_S_is_not_eps_D():
    # the second-order term distinguishes the precisions: 3 + 13/4 eps
    s1 = oracle.ub_relerr_H(1, F32)
    d1 = oracle.ub_relerr_H(1, F64)
    assert abs((s1 - 3.0) / 2.0 ** -24 - 3.25) < 1e-6
    assert abs(d1 - 3.0) < 1e-14
    # eps_S: the single-node bound covers every fp32 v1_hypot of random pairs
    # against the correctly rounded hypot (exact rationals)
    rng = np.random.default_rng(7)
    x = (rng.uniform(-1, 1, 2000) * np.ldexp(1.0, rng.integers(-30, 30, 2000))).astype(F32)
    y = (rng.uniform(-1, 1, 2000) * np.ldexp(1.0, rng.integers(-30, 30, 2000))).astype(F32)
    h = oracle.v1_hypot_array(x, y)
    worst = 0.0
    for a, b, r in zip(x, y, h):
        ex = Fraction(float(a)) ** 2 + Fraction(float(b)) ** 2
        # relerr against the real hypot: |r - sqrt(ex)| / (sqrt(ex) eps) <= bound
        # <=> (r/sqrt(ex)) in [lo, hi] <=> r^2 / ex in [lo^2, hi^2]
        q = Fraction(float(r)) ** 2 / ex
        worst = max(worst, abs(float(q) - 1) / 2 / 2.0 ** -24)
        assert q <= Fraction(1 + 3.0000003 * 2.0 ** -24) ** 2
    assert worst <= s1
