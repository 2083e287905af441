"""Pins for the oracle's tree evaluators (Listing 1, the tile-lane tree, columns,
shards).  Expected values come from the paper's worked examples (e:r P:473-481,
the n=16 lane display P:912-932), from ``ieee_exact`` (exact-rational Listing 2),
from index arithmetic, or from invariants -- never from the oracle itself."""
import math

import numpy as np
import pytest

import ieee_exact as ie
import nrmf_inputs as gen
import oracle

rng = np.random.default_rng(7)
BITS = {np.float64: 64, np.float32: 32}
LANES = {np.float64: 64, np.float32: 128}
JJ = {np.float64: 64, np.float32: 32}
T = 4096


def H(a, b, bits=64):
    return ie.v1_hypot(float(a), float(b), bits)


def test_listing1_n7_is_e_r():
    """e:r: R([x1..x7]) = h(h(h(x1,x2),h(x3,x4)), h(h(x5,x6),|x7|))."""
    for _ in range(50):
        x = rng.uniform(-3, 3, 7)
        exp = H(H(H(x[0], x[1]), H(x[2], x[3])), H(H(x[4], x[5]), abs(x[6])))
        assert ie.same(float(oracle.R_H(x)), exp)
        # the tile-lane tree with one lane and J = 8 is the same tree (padding
        # the 8th leaf with +0 gives v1(x7, 0) = |x7| exactly)
        assert ie.same(float(oracle.nrmf(x, lanes=1, J=8)), exp)


def test_listing1_split_lengths():
    """Listing 1 splits n into p = ceil(n/2), q = n - p: n=5 ->
    h(h(h(x1,x2),|x3|), h(x4,x5)); n=3 -> h(h(x1,x2), |x3|)."""
    x = rng.uniform(-1, 1, 5)
    assert ie.same(float(oracle.R_H(x)), H(H(H(x[0], x[1]), abs(x[2])), H(x[3], x[4])))
    assert ie.same(float(oracle.R_H(x[:3])), H(H(x[0], x[1]), abs(x[2])))
    assert float(oracle.R_H(x[:1])) == abs(x[0])


@pytest.mark.parametrize("k", [0, 1, 2, 5, 10, 13])
def test_one_lane_tree_is_listing1_on_powers_of_two(k):
    x = rng.normal(size=2 ** k)
    assert ie.same(float(oracle.nrmf(x, lanes=1, J=max(2 ** k, 1))), float(oracle.R_H(x)))


def test_lane_example_n16_p4():
    """with p = 4, n = 16, lane l holds
    sqrt((x_l^2 + x_{l+4}^2) + (x_{l+8}^2 + x_{l+12}^2)), grouped as displayed;
    the 4 lanes are then reduced by R over the stored lane array
    -- contiguous pairs, v1_hypot at every node (reading R1)."""
    for dt in (np.float64, np.float32):
        b = BITS[dt]
        x = rng.uniform(-2, 2, 16).astype(dt)
        L = [H(H(x[l], x[l + 4], b), H(x[l + 8], x[l + 12], b), b) for l in range(4)]
        exp = H(H(L[0], L[1], b), H(L[2], L[3], b), b)
        assert ie.same(float(oracle.nrmf(x, lanes=4, J=4)), exp, b)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", [1, 2, 63, 64, 4095, 4096, 4097, 9000, 3 * 4096 + 5])
def test_one_hot_every_position_class(dt, n):
    """One nonzero element c anywhere: every node is v1(a, 0) = a or v1(0,0) = 0,
    so the result is |c| exactly.  Pins the index mapping and neutral padding."""
    positions = sorted(set([0, n - 1, n // 2] + list(rng.integers(0, n, 12))))
    for p in positions:
        x = np.zeros(n, dtype=dt)
        c = dt(-1.7e-3) if p % 2 else dt(12345.678)
        x[p] = c
        assert oracle.nrmf(x) == abs(c)


def y_index(i, dt):
    """Position of element i in the transposed order:
    tile tau = i // T, lane l = (i % T) % lanes, j = (i % T) // lanes,
    y = tau*T + l*J + j."""
    lanes, J = LANES[dt], JJ[dt]
    tau, r = divmod(i, T)
    j, l = divmod(r, lanes)
    return tau * T + l * J + j


def lca_depth(a, b):
    """Length of the common prefix of two leaf positions in a balanced tree:
    larger = deeper lowest common ancestor."""
    return (a ^ b).bit_length()


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_two_and_three_hot_tree_shape(dt):
    """Two nonzeros: v1(x_a, x_b) whatever their positions.  Three nonzeros: the
    pair whose leaves share the deepest common ancestor in the transposed order
    (index arithmetic only) is combined first: v1(v1(x_a,x_b), x_c)."""
    b = BITS[dt]
    n = 5 * T + 77
    for _ in range(60):
        idx = rng.choice(n, size=3, replace=False)
        vals = [dt(v) for v in rng.uniform(0.5, 2.0, 3)]
        x = np.zeros(n, dtype=dt)
        x[idx[0]], x[idx[1]] = vals[0], vals[1]
        assert ie.same(float(oracle.nrmf(x)), H(vals[0], vals[1], b), b)
        x[idx[2]] = vals[2]
        ys = [y_index(int(i), dt) for i in idx]
        pairs = [(0, 1, 2), (0, 2, 1), (1, 2, 0)]
        a, bb, c = min(pairs, key=lambda p: lca_depth(ys[p[0]], ys[p[1]]))
        exp = H(H(vals[a], vals[bb], b), vals[c], b)
        assert ie.same(float(oracle.nrmf(x)), exp, b)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_zero_and_empty(dt):
    assert oracle.nrmf(np.zeros(0, dtype=dt)) == 0
    r = oracle.nrmf(np.zeros(10000, dtype=dt))
    assert r == 0 and math.copysign(1, float(r)) == 1
    r = oracle.nrmf(-np.zeros(3, dtype=dt))
    assert r == 0 and math.copysign(1, float(r)) == 1


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("k", [1, 2, 3, 6])
def test_constant_vector_full_tree(dt, k):
    """n = 4^k elements equal to c with n = P2*T or n <= T fully populating a
    perfect tree of depth d = 2k: every level maps a -> v1(a, a) = RN(a*RN(sqrt2))
    (Q = 1, S = 2), so the result is that map applied d times to |c|
    (closed form from Listing 2 with q = 1); and it is within the Thm-3 bound
    of |c|*sqrt(n) = |c|*2^k."""
    b = BITS[dt]
    n = 4 ** k
    if n > T or T % n:
        pytest.skip("needs a full tile")
    c = dt(-0.3)
    x = np.full(n, c, dtype=dt)
    r = float(oracle.nrmf(x, lanes=n if n < LANES[dt] else LANES[dt], J=max(1, n // LANES[dt])))
    s2 = ie.sqrt(2.0, b)
    v = abs(float(c))
    for _ in range(2 * k):
        v = ie.mul(v, s2, b)
    assert r == v
    assert oracle.relerr(r, abs(float(c)) * 2 ** k, dt) <= oracle.ub_relerr_H(2 * k, dt)


def test_constant_ones_production_tree():
    """All-ones, n = 4^k for the production tree (tile of 4096, 2^12 leaves per
    tile): every node has equal children, so result = (x -> RN(x RN(sqrt2)))^lg n (1)."""
    for k in (6, 7, 8):
        n = 4 ** k
        r = float(oracle.nrmf(np.ones(n)))
        v = 1.0
        for _ in range(2 * k):
            v = ie.mul(v, math.sqrt(2.0))
        assert r == v
        assert abs(r - 2.0 ** k) / 2.0 ** k <= 2 * 2.0 ** -53 * (2 * k)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_power_of_two_scaling_bitwise(dt):
    """x -> 2^s x scales every exact intermediate by 2^s, so the result scales
    bitwise when nothing under/overflows (S, s are scale-free)."""
    x = gen.uniform_pm1(3, 20000, dtype=dt)
    r = oracle.nrmf(x)
    for s in ([-300, -7, 5, 300] if dt == np.float64 else [-40, -3, 9, 40]):
        xs = np.ldexp(x, s).astype(dt)
        assert oracle.nrmf(xs) == np.ldexp(r, s).astype(dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_permutation_within_bound(dt):
    """A permutation goes through a different tree (different bits), but both
    results are within the Thm-3 bound of the permutation-invariant exact norm."""
    n = 3 * T + 11
    x = gen.normal(5, n, dtype=dt)
    ex = oracle.exact(x)
    d = 12 + 2  # lg T + lg P2 (P2 = 4 tiles)
    ub = oracle.ub_relerr_H(d, dt)
    for _ in range(5):
        xp = x[rng.permutation(n)]
        assert oracle.exact(xp) == ex
        assert oracle.relerr(oracle.nrmf(xp), ex, dt) <= ub
    assert oracle.relerr(oracle.nrmf(x), ex, dt) <= ub


def test_extremes_no_overflow_underflow():
    big = 0.7 * np.finfo(np.float64).max
    r = oracle.nrmf(np.array([big, -big]))
    assert math.isfinite(r) and r > big
    assert oracle.nrmf(np.array([big, big, big])) == float("inf")   # true norm > DBL_MAX
    t = np.full(64, 2.0 ** -1000)        # x^2 = 2^-2000 underflows in a naive sum of squares
    r = oracle.nrmf(t)
    assert r > 0 and oracle.relerr(r, 8 * 2.0 ** -1000) <= oracle.ub_relerr_H(6)
    # all-subnormal input: inexact underflow (excluded by Thm 3) loses
    # relative accuracy, but the result does not flush to zero
    assert oracle.nrmf(np.full(64, 2.0 ** -1060)) > 0
    assert oracle.nrmf(np.array([5e-324])) == 5e-324


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_nan_padding_reading_R4(dt):
    """v1(NaN, 0) = +0 (Listing 2 literally), so padding is *not* neutral for a
    NaN input: a lone NaN in a 1-element array gives |NaN| at n = 1 but the
    tile tree pads it with zeros -> +0.  Documented reading R4."""
    x = np.array([np.nan], dtype=dt)
    assert math.isnan(oracle.nrmf(x, lanes=1, J=1))   # no padding: |NaN|
    assert oracle.nrmf(x) == 0                        # padded: v1(NaN, 0) = +0
    # NaN's lane meets a +0 leaf first and collapses to +0; the other lane holds 3
    x = np.array([np.nan, 3.0], dtype=dt)
    assert oracle.nrmf(x) == 3.0


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n,G", [(1, 2), (5, 8), (4096, 2), (4097, 2), (4097, 8), (3 * 4096 + 1, 4),
                                 (17 * 4096 - 3, 8), (40000, 1), (40000, 2), (40000, 4), (40000, 8)])
def test_shards_combine_to_global(dt, n, G):
    """Canonical shards are aligned subtrees; combining the rank values with the
    rank tree reproduces the global tree bitwise (including the NaN reading)."""
    x = gen.normal(11, n, dtype=dt)
    g = oracle.nrmf(x)
    sh = oracle.shard_norms(x, G)
    assert oracle.combine_ranks(sh) == g
    ranges = oracle.shard_ranges(n, G)
    assert sum(c for _, c, _ in ranges) == n
    assert all(a % T == 0 for a, c, _ in ranges if c)
    # NaN in the last element: same bits at every G
    x[-1] = np.nan
    g = oracle.nrmf(x)
    assert ie.same(float(oracle.combine_ranks(oracle.shard_norms(x, G))), float(g), BITS[dt])


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_columns(dt):
    """e:F: column norms then the norm over columns.  With r = ld = T
    the column-major matrix is the vector of tiles, so frob == nrmf(vec A)."""
    r, c = 4096, 24
    A = gen.colscaled_normal(2, r, c, dtype=dt)
    col, frob = oracle.cols(A, r, c, r)
    for j in range(c):
        assert col[j] == oracle.nrmf(A[j * r:(j + 1) * r])
    assert frob == oracle.nrmf(A)
    # per-column power-of-two scaling: col_j * 2^-k_j is the unscaled column norm
    A0 = gen.colscaled_normal(2, r, c, klo=0, khi=0, dtype=dt)
    col0, _ = oracle.cols(A0, r, c, r)
    ratio = np.log2(col / col0)
    assert np.all(ratio == np.round(ratio))
    # ragged rows and ld > r
    r2, ld2 = 1000, 1003
    A2 = gen.colscaled_normal(4, r2, 7, ld=ld2, dtype=dt)
    col2, frob2 = oracle.cols(A2, r2, 7, ld2)
    for j in range(7):
        assert col2[j] == oracle.nrmf(A2[j * ld2:j * ld2 + r2])
    assert frob2 == oracle.combine(col2)
    # empty shapes
    col3, frob3 = oracle.cols(np.zeros(0, dtype=dt), 0, 3, 0)
    assert np.all(col3 == 0) and frob3 == 0


def test_A_top_reading_R1_f1():
    """top="cr": Listing 1 with cr_hypot (A) above the tiles, v1
    inside.  One tile: identical to the v1 tree.  e:r shape for A on n=7.
    Shards + rank tree reproduce it.  Error within the A/H mixed bound."""
    x = rng.uniform(-3, 3, 7)
    C = lambda a, b: ie.exact_norm([float(a), float(b)])  # noqa: E731
    exp = C(C(C(x[0], x[1]), C(x[2], x[3])), C(C(x[4], x[5]), abs(x[6])))
    assert ie.same(float(oracle.R_A(x)), exp)
    y = gen.normal(3, 4000)
    assert oracle.nrmf(y, top="cr") == oracle.nrmf(y)           # no node above the single tile
    z = gen.normal(4, 37 * T + 5)
    a, v = oracle.nrmf(z, top="cr"), oracle.nrmf(z)
    tiles = oracle.tiles(z)
    assert a == oracle.combine(tiles, top="cr") and v == oracle.combine(tiles)
    for G in (2, 4, 8):
        assert oracle.combine_ranks(oracle.shard_norms(z, G, top="cr"), top="cr") == a
    import mpmath
    mpmath.mp.prec = 200
    eps = mpmath.mpf(2) ** -53
    ub = float(((oracle.reH_plus()) ** 12 * (1 + eps) ** 6 - 1) / eps)   # 12 v1 levels, 6 cr levels
    assert oracle.relerr(a, oracle.exact(z)) <= ub


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("r,c", [(5, 7), (4096, 9), (4100, 3), (1, 33), (300, 64)])
def test_cols_block_shards_combine_to_global_frob(dt, r, c):
    """Column blocks: each rank's Frobenius subtree over its
    canonical column block, padded to P2c/G, combined by the rank tree, equals
    the global Frobenius norm bitwise for every G = 1..8 (powers of two) --
    including a NaN column norm, for which +0 padding is not neutral (R4)."""
    A = gen.normal(r * 10 + c, r * c, dtype=dt)
    for with_nan in (False, True):
        if with_nan:
            A = A.copy()
            A[(c - 1) * r:] = np.nan           # last column all NaN: its norm is NaN
        _, efr = oracle.cols(A, r, c, r)
        for G in (1, 2, 4, 8):
            vals = oracle.cols_shard_frobs(A, r, c, r, G)
            got = oracle.combine_ranks(vals)
            assert np.asarray(got, dtype=dt).tobytes() == np.asarray(efr, dtype=dt).tobytes(), (G, with_nan)


# ------------------------------------------------------------ golden fixtures
import os as _os
import re as _re

_GOLD = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "golden")


def _golden(name):
    out = {}
    with open(_os.path.join(_GOLD, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                k, v = line.split(":", 1)
                out[k.strip()] = v.strip()
    return out


def _eval_tree(expr, env, bits):
    """Evaluate h(a,b) / abs(a) / names with the exact-rational Listing 2."""
    tok = _re.findall(r"[A-Za-z_][A-Za-z_0-9]*|[(),]", expr)
    pos = 0

    def parse():
        nonlocal pos
        t = tok[pos]
        pos += 1
        if t in ("h", "abs"):
            assert tok[pos] == "("
            pos += 1
            a = parse()
            if t == "abs":
                assert tok[pos] == ")"
                pos += 1
                return abs(a)
            assert tok[pos] == ","
            pos += 1
            b = parse()
            assert tok[pos] == ")"
            pos += 1
            return H(a, b, bits)
        return env[t]
    v = parse()
    assert pos == len(tok)
    return v


def test_golden_e_r_n7():
    """tests/golden/e_r_n7.txt: the oracle's Listing 1 and the
    one-lane tile tree with J = 8 evaluate exactly the transcribed tree."""
    g = _golden("e_r_n7.txt")
    for _ in range(50):
        x = rng.uniform(-3, 3, 7)
        env = {f"x{i + 1}": float(x[i]) for i in range(7)}
        exp = _eval_tree(g["tree"], env, 64)
        assert ie.same(float(oracle.R_H(x)), exp)
        assert ie.same(float(oracle.nrmf(x, lanes=1, J=8)), exp)


def test_golden_lane_example_p4_n16():
    """tests/golden/lane_example_p4_n16.txt: the
    oracle with p = 4 lanes, J = 4 is the transcribed lane trees + R."""
    g = _golden("lane_example_p4_n16.txt")
    for dt in (np.float64, np.float32):
        b = BITS[dt]
        for _ in range(20):
            x = rng.uniform(-2, 2, 16).astype(dt)
            env = {f"x{i + 1}": float(x[i]) for i in range(16)}
            for l in range(1, 5):
                env[f"lane{l}"] = _eval_tree(g[f"lane{l}"], env, b)
            exp = _eval_tree(g["final"], env, b)
            assert ie.same(float(oracle.nrmf(x, lanes=4, J=4)), exp, b)
