"""oracle.bounds -- TEST INFRASTRUCTURE ONLY.

High-precision evaluator of the paper's relative-error-bound recurrences
(mpmath, 256+ bits), used by the tests to bound every computed norm:

  bounds_L(n)              Thm 1, e:13, the xNRM2 model L
  bounds_C(n, c)           Thm 2, e:3, iterative hypot C
  bounds_R(n, kind)        Thm 3, e:8, over Listing 1's split tree
  hypot_envelope(kind)     e:reH for v1_hypot; (1 -+ eps) for cr_hypot
  ub_depths(d_v1, d_cr)    a tree whose root-to-leaf paths hold at most d_v1
                           v1_hypot and d_cr cr_hypot rounding nodes

Normalised bounds are in units of eps (e:ubr).  Conventions (SPEC
S:359-360, R12): Thm 1 iterates n-1 update factors; in Thm 3 the
quotient factor 1+eps_/ of (e:8) is a min/max ratio, hence clamped to <= 1,
so an equal-children node contributes exactly one hypot factor.  With these
the evaluator reproduces all 90 values of Table 3 (tests/golden).
"""
from __future__ import annotations

from functools import lru_cache

import mpmath

PREC = 512


def _eps(bits: int):
    return mpmath.mpf(2) ** (-53 if bits == 64 else -24)


def hypot_envelope(kind: str = "v1", bits: int = 64):
    """(1+eps'-, 1+eps'+): e:reH for v1_hypot; 1-+eps for cr_hypot."""
    mpmath.mp.prec = PREC
    e = _eps(bits)
    if kind == "cr":
        return 1 - e, 1 + e
    lo = (1 - e) ** mpmath.mpf(2.5) * mpmath.sqrt(1 - e * (2 - e) / 2)
    hi = (1 + e) ** mpmath.mpf(2.5) * mpmath.sqrt(1 + e * (2 + e) / 2)
    return lo, hi


def bounds_L(n: int, bits: int = 64):
    """Thm 1, e:13: (lb, ub) of relerr[L] in eps, single accumulator."""
    mpmath.mp.prec = PREC
    e = _eps(bits)
    etam = (1 - e) ** (n - 1)   # 1 + eta_n^-
    etap = (1 + e) ** (n - 1)   # 1 + eta_n^+
    lb = (mpmath.sqrt(etam) * (1 - e) - 1) / e
    ub = (mpmath.sqrt(etap) * (1 + e) - 1) / e
    return lb, ub


def bounds_C(n: int, bits: int = 64):
    """Thm 2, e:3 with cr_hypot, iterated from eps_1 = 0 for i = 2..n."""
    mpmath.mp.prec = PREC
    e = _eps(bits)
    em = ep = mpmath.mpf(0)
    for _ in range(2, n + 1):
        em = mpmath.sqrt(1 + em * (2 + em)) * (1 - e) - 1
        ep = mpmath.sqrt(1 + ep * (2 + ep)) * (1 + e) - 1
    return em / e, ep / e


def _combine(p, q, env):
    """e:8: bounds of the parent of two subtrees with bounds p, q."""
    (pm, pp), (qm, qp) = p, q
    lo, hi = env
    # k: the child with the larger upper factor, l: the other
    if pp >= qp:
        (km, kp), (lm, lp) = (pm, pp), (qm, qp)
    else:
        (km, kp), (lm, lp) = (qm, qp), (pm, pp)
    sm = (1 + lm) / (1 + kp)                      # 1 + eps_/^-
    sp = min(mpmath.mpf(1), (1 + lp) / (1 + km))  # 1 + eps_/^+, a ratio <= 1 (clamp)
    xm, xp = sm - 1, sp - 1
    nm = mpmath.sqrt(1 + xm * (2 + xm)) * (1 + km) * lo - 1
    np_ = mpmath.sqrt(1 + xp * (2 + xp)) * (1 + kp) * hi - 1
    return nm, np_


@lru_cache(maxsize=None)
def _bounds_R_raw(n: int, kind: str, bits: int):
    mpmath.mp.prec = PREC
    if n == 1:
        return mpmath.mpf(0), mpmath.mpf(0)
    env = hypot_envelope(kind, bits)
    if n == 2:
        return env[0] - 1, env[1] - 1
    p = (n >> 1) + (n & 1)
    return _combine(_bounds_R_raw(p, kind, bits), _bounds_R_raw(n - p, kind, bits), env)


def bounds_R(n: int, kind: str = "v1", bits: int = 64):
    """Thm 3 over Listing 1's tree (ceil split): (lb, ub) of relerr in eps."""
    e = _eps(bits)
    m, p = _bounds_R_raw(n, kind, bits)
    return m / e, p / e


def ub_depths(d_v1: int, d_cr: int = 0, bits: int = 64) -> float:
    """Upper bound (in eps) for a tree whose every root-to-leaf path contains
    at most d_v1 v1_hypot and d_cr cr_hypot rounding nodes (Thm 3 with the
    clamp: each rounding node multiplies the upper factor by its envelope)."""
    mpmath.mp.prec = PREC
    e = _eps(bits)
    return float((hypot_envelope("v1", bits)[1] ** d_v1 * hypot_envelope("cr", bits)[1] ** d_cr - 1) / e)


def tile_tree_depths(n: int, bits: int = 64, top: str = "v1"):
    """(d_v1, d_cr) for the tile-lane tree of n elements:
    lg T levels inside a tile (v1), lg P2 levels above (v1 or cr)."""
    T = 4096
    nt = max(1, -(-n // T))
    P2 = 1
    while P2 < nt:
        P2 <<= 1
    lt, lp = 12, P2.bit_length() - 1
    return (lt + lp, 0) if top == "v1" else (lt, lp)
