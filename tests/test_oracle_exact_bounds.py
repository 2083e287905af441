"""Pins for the exact reference (O2), the Thm-3 bounds and the accuracy claims.

exact(): checked against Python exact rationals + math.isqrt (ieee_exact) and
closed forms.  Bounds: the closed forms reproduce the paper's Table 3
(tests/golden/table3_ub_relerr_D.txt, transcribed from PAPER.md P:679-708)."""
import math
import os

import mpmath
import numpy as np
import pytest

import ieee_exact as ie
import nrmf_inputs as gen
import oracle

rng = np.random.default_rng(99)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table3_ub_relerr_D.txt")


@pytest.mark.parametrize("bits", [64, 32])
def test_exact_vs_fraction_isqrt(bits):
    dt = np.float64 if bits == 64 else np.float32
    emin = -1074 if bits == 64 else -149
    emax = 1000 if bits == 64 else 120
    for trial in range(300):
        n = int(rng.integers(1, 40))
        kind = trial % 4
        if kind == 0:
            x = rng.uniform(-1, 1, n)
        elif kind == 1:
            x = np.ldexp(rng.uniform(1, 2, n), rng.integers(emin + 52 if bits == 64 else emin + 23, emax, n))
        elif kind == 2:
            x = rng.integers(-2 ** 20, 2 ** 20, n) * np.ldexp(1.0, emin)  # subnormal sums
        else:
            e = int(rng.integers(-200, 200)) if bits == 64 else int(rng.integers(-40, 40))
            x = np.ldexp(rng.uniform(1, 2, n), e + rng.integers(-2, 2, n))
        x = x.astype(dt)
        assert ie.same(float(oracle.exact(x)), ie.exact_norm(x, bits), bits)


def test_exact_closed_forms():
    assert oracle.exact(np.array([3.0, 4.0])) == 5.0
    assert oracle.exact(np.array([3.0, 4.0], dtype=np.float32)) == 5.0
    assert oracle.exact(np.ones(4)) == 2.0
    for k in range(0, 12):
        c = 0.3
        # sqrt(n c^2) with n = 4^k is c * 2^k exactly (power-of-two scaling of |c|)
        assert oracle.exact(np.full(4 ** k, c)) == c * 2 ** k
    assert oracle.exact(np.array([5e-324])) == 5e-324
    assert oracle.exact(np.zeros(5)) == 0.0
    assert oracle.exact(np.zeros(0)) == 0.0
    big = np.finfo(np.float64).max
    assert oracle.exact(np.array([big, big])) == float("inf")
    assert oracle.exact(np.array([big])) == big
    assert oracle.exact(np.array([big * 0.7, big * 0.7])) == ie.exact_norm([big * 0.7, big * 0.7])
    assert oracle.exact(np.array([np.inf, 1.0])) == float("inf")
    assert math.isnan(oracle.exact(np.array([np.nan, np.inf])))
    # order independence (exact sum)
    x = gen.normal(1, 5000)
    assert oracle.exact(x) == oracle.exact(x[::-1]) == oracle.exact(np.sort(x))


def test_exact_rounding_near_ties():
    """sqrt(1 + 2^-52 + 2^-106) etc.: values whose square root lies a hair above
    or below a rounding midpoint; the integer sqrt with sticky must round right."""
    for x in ([1.0, 2.0 ** -26], [1.0, 2.0 ** -26 * 1.0000001], [1.0, 2.0 ** -27 * 3],
              [1.0, 1.0, 2.0 ** -30], [1.0 + 2.0 ** -52, 2.0 ** -26]):
        assert ie.same(float(oracle.exact(np.array(x))), ie.exact_norm(x))


def _golden():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            ln, k, L, A, Hh = line.split()
            rows.append((int(k), mpmath.mpf(L), mpmath.mpf(A), mpmath.mpf(Hh)))
    assert len(rows) == 30
    return rows


def _sig18(a, b):
    """Agreement to the 18 printed significant digits (relative 5e-18)."""
    return abs(a - b) <= abs(b) * mpmath.mpf("6e-18")


def test_table3_H_column_closed_form():
    """ub relerr[H_D] for n = 2^k is ((1+eps'+)^k - 1)/eps with eps'+ from
    e:reH (Thm 3 with equal children)."""
    for k, _, _, Hh in _golden():
        assert _sig18(mpmath.mpf(oracle.ub_relerr_H(k)), Hh) or \
            _sig18(((oracle.reH_plus()) ** k - 1) / mpmath.mpf(2) ** -53, Hh), k


def test_table3_A_and_L_columns():
    """A_D: ((1+eps)^k - 1)/eps (cr_hypot, c = 1).  L_D (Thm 1,
    e:ubr P:646-650): (sqrt((1+eps)^(n-1))*(1+eps) - 1)/eps with n = 2^k."""
    mpmath.mp.prec = 2048
    eps = mpmath.mpf(2) ** -53
    for k, L, A, _ in _golden():
        assert _sig18(((1 + eps) ** k - 1) / eps, A), k
        n = 2 ** k
        assert _sig18((mpmath.sqrt((1 + eps) ** (n - 1)) * (1 + eps) - 1) / eps, L), k


def test_growth_laws():
    """Table 3 / P:661-663: logarithmic growth for H (steps of ~3 per doubling)."""
    prev = None
    for k in range(1, 31):
        v = oracle.ub_relerr_H(k)
        if prev is not None:
            assert abs((v - prev) - 3.0) < 1e-6
        prev = v


@pytest.mark.parametrize("dt,make", [
    (np.float64, lambda s, n: gen.uniform_pm1(s, n)),
    (np.float64, lambda s, n: gen.normal(s, n)),
    (np.float32, lambda s, n: gen.sme(s, n)),
    (np.float32, lambda s, n: gen.normal(s, n, dtype=np.float32)),
])
def test_accuracy_within_bound_and_64eps(dt, make):
    """relerr (e:relerr) of the tile-lane tree against the exact
    reference is within the Thm-3 bound for its depth and within 64 eps; on
    these moderately varying inputs it is also below 3 eps as the paper
    observes for all recursive algorithms."""
    n = (1 << 18) + 333
    depth = 12 + 7  # lg T + lg P2 (P2 = 128 tiles)
    for seed in (1, 2, 3):
        x = make(seed, n).astype(dt)
        r = oracle.nrmf(x)
        e = oracle.relerr(r, oracle.exact(x), dt)
        assert e <= oracle.ub_relerr_H(depth, dt)
        assert e <= 64
        assert e < 3


def test_extreme_range_variants_reading_R9():
    """C5 readings: 'lit' overflows (exact +inf and tree +inf, no NaN); 'fin' and
    'fin2' stay finite and within 64 eps (small n here; full n on the GPU)."""
    n = 1 << 16
    x = gen.extreme(1, n, "lit")
    assert np.all(np.isfinite(x))
    assert oracle.exact(x) == float("inf") and oracle.nrmf(x) == float("inf")
    for v in ("fin", "fin2"):
        x = gen.extreme(2, n, v)
        ex = oracle.exact(x)
        assert math.isfinite(ex)
        assert oracle.relerr(oracle.nrmf(x), ex) <= 64


# --------------------------------------------------------------- SURVEY f4
from oracle import bounds as B  # noqa: E402


def test_table3_by_the_recurrences():
    """Thm 1 (e:13) and Thm 3 (e:8, evaluated recursively over Listing 1's
    tree with the clamp convention) reproduce all 90 printed values of
    Table 3 to their 18 digits."""
    for k, L, A, Hh in _golden():
        n = 2 ** k
        assert _sig18(B.bounds_L(n)[1], L), k
        assert _sig18(B.bounds_R(n, "cr")[1], A), k
        assert _sig18(B.bounds_R(n, "v1")[1], Hh), k


def test_bounds_properties():
    # lb <= 0 <= ub, growth laws: L doubles per doubling of n,
    # A steps by 1 and H by ~3 per doubling
    for k in range(10, 30):
        n = 2 ** k
        for lb, ub in (B.bounds_L(n), B.bounds_R(n, "cr"), B.bounds_R(n, "v1")):
            assert lb <= 0 <= ub
        assert 1.9 <= B.bounds_L(2 * n)[1] / B.bounds_L(n)[1] <= 2.1
        assert abs(B.bounds_R(2 * n, "cr")[1] - B.bounds_R(n, "cr")[1] - 1) < 1e-6
        assert abs(B.bounds_R(2 * n, "v1")[1] - B.bounds_R(n, "v1")[1] - 3) < 1e-6
    # non-power-of-two n: Listing 1's ceil split, bound of ceil(lg n) levels
    for n in (3, 5, 7, 1000, 12345):
        d = (n - 1).bit_length()
        assert abs(B.bounds_R(n, "v1")[1] - B.ub_depths(d)) < 1e-9


def test_C_bound_about_twice_L():
    """for large n the single-accumulator C bounds are about twice
    those of L."""
    for n in (2 ** 10, 2 ** 14):
        r = float(B.bounds_C(n)[1] / B.bounds_L(n)[1])
        assert 1.8 < r < 2.2


def test_tile_tree_bound_f1():
    """The A-style top makes the 64-eps target a theorem at n = 2^30 fp64
    (SURVEY f1): 12 v1 levels + 18 cr levels -> 54 eps; all-v1 gives 90."""
    assert abs(B.ub_depths(*B.tile_tree_depths(1 << 30)) - 90) < 1e-6
    ub = B.ub_depths(*B.tile_tree_depths(1 << 30, top="cr"))
    assert 53.9 < ub < 54.1 and ub < 64
