"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded CPU implementation of the xNRMF hot path
(arXiv 2509.06220), written from the paper (see ``nrmf_oracle.c`` for the
line-by-line citations).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2509_06220_b200`` (the product), and
the product never imports it.

Functions (and what pins each, independently of this package)
  v1_hypot(x, y, dtype)              Listing 2 -- exact-rational IEEE
                                     re-implementation, closed forms, e:reH envelope
  cr_hypot(x, y, dtype)              correctly rounded hypot (f1) -- exact rationals
  R_H(x), R_A(x)                     Listing 1, literal, with v1 / cr
                                     hypot -- e:r for n = 7, ceil splits
  nrmf(x, lanes=None, J=None, top=)  the tile-lane tree -- lane
                                     example P:912-932, one/two/three-hot vectors,
                                     constants, scaling, zero/empty
  tiles(x, tau0, count)              tile values (sampled parity at full size)
  cols(A, r, c, ld)                  column norms + Frobenius norm (e:F) -- column
                                     == vector tree, frob == nrmf(vec A) at r = T
  shard_ranges / shard_norms /       canonical shards and per-rank subtrees --
  combine_ranks / combine            == the global tree for G = 1..8
  cols_shard_ranges /                canonical column blocks and their Frobenius
  cols_shard_frobs                   subtrees -- == the global frob for G = 1..8
  exact(x)                           exactly rounded RN(sqrt(sum x^2))
                                     -- Python Fraction + isqrt, closed forms
  relerr(r, ref, dtype)              e:relerr -- results one/two float
                                     spacings from powers of two (numpy's finfo
                                     eps), operand order, binade invariance
  ub_relerr_H(depth, dtype)          Thm 3 + e:reH bound -- Table 3 at
                                     eps_D; a hand-worked second-order Taylor
                                     expansion at eps_S and eps_D
  bounds.py                          Thm 1-3 recurrences -- all 90 Table 3 values

Parity unpinned: the absolute result values on random data -- the paper
prints none; they are pinned only by the same-tree evaluation plus the bound
against the exact reference.

Tree constants (frozen, tree version 1): fp64 lanes=64, J=64; fp32 lanes=128,
J=32; tile T = 4096.  These are restated here from DESIGN.md §3, not imported
from the CUDA side.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nrmf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

TREE = {np.dtype(np.float64): (64, 64), np.dtype(np.float32): (128, 32)}
EPS = {np.dtype(np.float64): 2.0 ** -53, np.dtype(np.float32): 2.0 ** -24}

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fno-finite-math-only",
          "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, vp, ip = ctypes.c_int64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)
        d, f = ctypes.c_double, ctypes.c_float
        L.oracle_v1_hypot_d.argtypes = [d, d]; L.oracle_v1_hypot_d.restype = d
        L.oracle_v1_hypot_s.argtypes = [f, f]; L.oracle_v1_hypot_s.restype = f
        L.oracle_v1_hypot_array_d.argtypes = [i64, vp, vp, vp]; L.oracle_v1_hypot_array_d.restype = None
        L.oracle_v1_hypot_array_s.argtypes = [i64, vp, vp, vp]; L.oracle_v1_hypot_array_s.restype = None
        L.oracle_R_H_d.argtypes = [i64, vp]; L.oracle_R_H_d.restype = d
        L.oracle_R_H_s.argtypes = [i64, vp]; L.oracle_R_H_s.restype = f
        ci = ctypes.c_int
        L.oracle_nrmf_tree_d.argtypes = [vp, i64, i64, i64, i64, ci, ip]; L.oracle_nrmf_tree_d.restype = d
        L.oracle_nrmf_tree_s.argtypes = [vp, i64, i64, i64, i64, ci, ip]; L.oracle_nrmf_tree_s.restype = f
        L.oracle_cr_hypot_d.argtypes = [d, d]; L.oracle_cr_hypot_d.restype = d
        L.oracle_cr_hypot_s.argtypes = [f, f]; L.oracle_cr_hypot_s.restype = f
        L.oracle_cr_hypot_array_d.argtypes = [i64, vp, vp, vp]; L.oracle_cr_hypot_array_d.restype = None
        L.oracle_cr_hypot_array_s.argtypes = [i64, vp, vp, vp]; L.oracle_cr_hypot_array_s.restype = None
        L.oracle_R_A_d.argtypes = [i64, vp]; L.oracle_R_A_d.restype = d
        L.oracle_R_A_s.argtypes = [i64, vp]; L.oracle_R_A_s.restype = f
        L.oracle_tiles_d.argtypes = [vp, i64, i64, i64, i64, i64, vp]; L.oracle_tiles_d.restype = ctypes.c_int
        L.oracle_tiles_s.argtypes = [vp, i64, i64, i64, i64, i64, vp]; L.oracle_tiles_s.restype = ctypes.c_int
        L.oracle_nrmf_cols_d.argtypes = [i64, i64, i64, vp, i64, i64, ctypes.c_int, vp, vp]
        L.oracle_nrmf_cols_d.restype = ctypes.c_int
        L.oracle_nrmf_cols_s.argtypes = [i64, i64, i64, vp, i64, i64, ctypes.c_int, vp, vp]
        L.oracle_nrmf_cols_s.restype = ctypes.c_int
        for sfx in ("d", "s"):
            getattr(L, "exact_acc_" + sfx).argtypes = [vp, i64, vp, ip]
            getattr(L, "exact_acc_" + sfx).restype = None
            getattr(L, "exact_round_" + sfx).argtypes = [vp, ctypes.c_int]
            getattr(L, "exact_acc_words_" + sfx).restype = ctypes.c_int
        L.exact_round_d.restype = d
        L.exact_round_s.restype = f
        L.exact_acc_merge.argtypes = [vp, vp, ctypes.c_int]; L.exact_acc_merge.restype = None
        L.exact_nrm_d.argtypes = [vp, i64]; L.exact_nrm_d.restype = d
        L.exact_nrm_s.argtypes = [vp, i64]; L.exact_nrm_s.restype = f
        _lib = L
    return _lib


def _arr(x, dtype=None):
    x = np.ascontiguousarray(x, dtype=dtype)
    if x.dtype not in (np.float64, np.float32):
        raise TypeError(f"oracle: unsupported dtype {x.dtype}")
    return x


def _is64(x) -> bool:
    return x.dtype == np.float64


def v1_hypot(x, y, dtype=np.float64):
    """Listing 2, one pair.  Returns a numpy scalar of ``dtype``."""
    if np.dtype(dtype) == np.float64:
        return np.float64(lib().oracle_v1_hypot_d(float(x), float(y)))
    return np.float32(lib().oracle_v1_hypot_s(float(np.float32(x)), float(np.float32(y))))


def v1_hypot_array(x, y):
    """Listing 2 applied elementwise to two equal-length arrays."""
    x = _arr(x)
    y = _arr(y, x.dtype)
    assert x.size == y.size
    out = np.empty_like(x)
    f = lib().oracle_v1_hypot_array_d if _is64(x) else lib().oracle_v1_hypot_array_s
    f(x.size, x.ctypes.data, y.ctypes.data, out.ctypes.data)
    return out


def cr_hypot(x, y, dtype=np.float64):
    """Correctly rounded hypot: RN(sqrt(x^2+y^2)) exactly (IEEE specials)."""
    if np.dtype(dtype) == np.float64:
        return np.float64(lib().oracle_cr_hypot_d(float(x), float(y)))
    return np.float32(lib().oracle_cr_hypot_s(float(np.float32(x)), float(np.float32(y))))


def cr_hypot_array(x, y):
    """cr_hypot applied elementwise."""
    x = _arr(x)
    y = _arr(y, x.dtype)
    out = np.empty_like(x)
    f = lib().oracle_cr_hypot_array_d if _is64(x) else lib().oracle_cr_hypot_array_s
    f(x.size, x.ctypes.data, y.ctypes.data, out.ctypes.data)
    return out


def R_A(x):
    """Listing 1 with cr_hypot (the A algorithm)."""
    x = _arr(x)
    assert x.size >= 1
    f = lib().oracle_R_A_d if _is64(x) else lib().oracle_R_A_s
    return x.dtype.type(f(x.size, x.ctypes.data))


def R_H(x):
    """Listing 1 (scalar recursive, ceil split) with v1_hypot; n >= 1."""
    x = _arr(x)
    assert x.size >= 1
    f = lib().oracle_R_H_d if _is64(x) else lib().oracle_R_H_s
    return x.dtype.type(f(x.size, x.ctypes.data))


def nrmf(x, lanes: int | None = None, J: int | None = None, p2_min: int = 1, top: str = "v1"):
    """The tile-lane tree.  lanes/J default to the production tree of x's dtype.
    lanes=1, J>=n (power of two) is Listing 1; lanes=8 is Z_D with an
    R-with-v1_hypot final reduction.  top="cr": the levels
    above the tiles use cr_hypot (the A-style final reduction)."""
    x = _arr(x)
    dl, dj = TREE[x.dtype]
    lanes = dl if lanes is None else lanes
    J = dj if J is None else J
    assert lanes & (lanes - 1) == 0 and J & (J - 1) == 0
    ok = ctypes.c_int(1)
    f = lib().oracle_nrmf_tree_d if _is64(x) else lib().oracle_nrmf_tree_s
    r = f(x.ctypes.data, x.size, lanes, J, p2_min, 1 if top == "cr" else 0, ctypes.byref(ok))
    if not ok.value:
        raise MemoryError("oracle: allocation failed")
    return x.dtype.type(r)


def tiles(x, tau0: int = 0, count: int | None = None, lanes=None, J=None):
    """Tile values tau0 .. tau0+count-1 of the tile-lane tree of x."""
    x = _arr(x)
    dl, dj = TREE[x.dtype]
    lanes = dl if lanes is None else lanes
    J = dj if J is None else J
    T = lanes * J
    nt = -(-x.size // T)
    count = nt - tau0 if count is None else count
    out = np.empty(count, dtype=x.dtype)
    f = lib().oracle_tiles_d if _is64(x) else lib().oracle_tiles_s
    if not f(x.ctypes.data, x.size, lanes, J, tau0, count, out.ctypes.data):
        raise MemoryError("oracle: allocation failed")
    return out


def cols(A, r: int, c: int, ld: int, lanes=None, J=None, top: str = "v1"):
    """Column norms of the column-major r x c matrix stored in flat A (leading
    dimension ld), and the Frobenius norm (R_H over the padded column norms)."""
    A = _arr(A)
    dl, dj = TREE[A.dtype]
    lanes = dl if lanes is None else lanes
    J = dj if J is None else J
    col = np.empty(c, dtype=A.dtype)
    frob = np.zeros(1, dtype=A.dtype)
    f = lib().oracle_nrmf_cols_d if _is64(A) else lib().oracle_nrmf_cols_s
    if not f(r, c, ld, A.ctypes.data, lanes, J, 1 if top == "cr" else 0, col.ctypes.data, frob.ctypes.data):
        raise MemoryError("oracle: allocation failed")
    return col, A.dtype.type(frob[0])


def combine(values, top: str = "v1"):
    """R_H (or R_A for top="cr") over the list padded with +0 to a power of two
    (the rank tree)."""
    v = _arr(values)
    if v.size == 0:
        return v.dtype.type(0)
    p = 1
    while p < v.size:
        p <<= 1
    pad = np.zeros(p, dtype=v.dtype)
    pad[: v.size] = v
    return R_A(pad) if top == "cr" else R_H(pad)


def shard_ranges(n: int, G: int, T: int = 4096):
    """Canonical contiguous shards: NT = ceil(n/T) tiles,
    P2 = pow2 >= NT; if G <= P2 rank g owns tiles [g*P2/G, (g+1)*P2/G), else
    rank g < P2 owns tile g.  Returns [(offset, count, p2_local)] per rank
    (p2_local = 0 for a rank that owns no part of the tree)."""
    nt = -(-n // T)
    P2 = 1
    while P2 < nt:
        P2 <<= 1
    out = []
    for g in range(G):
        if G <= P2:
            per = P2 // G
            t0, t1 = g * per, (g + 1) * per
            p2l = per
        else:
            t0, t1 = (g, g + 1) if g < P2 else (P2, P2)
            p2l = 1 if g < P2 else 0
        a, b = min(t0 * T, n), min(t1 * T, n)
        out.append((a, b - a, p2l))
    return out


def cols_shard_ranges(c: int, G: int):
    """Canonical column blocks: P2c = pow2 >= c column leaves;
    if G <= P2c rank g owns columns [g*P2c/G, (g+1)*P2c/G), else rank g < P2c
    owns column g.  Returns [(col_offset, col_count, p2_local)] per rank."""
    return shard_ranges(c, G, 1)


def cols_shard_frobs(A, r: int, c: int, ld: int, G: int, top: str = "v1"):
    """Each rank's Frobenius subtree (R_H over its column norms padded with +0
    to p2_local), in rank order (None for a rank owning no part of the tree)."""
    col, _ = cols(A, r, c, ld, top=top)
    res = []
    for (a, cnt, p2l) in cols_shard_ranges(c, G):
        if p2l == 0:
            res.append(None)
            continue
        pad = np.zeros(p2l, dtype=col.dtype)
        pad[:cnt] = col[a:a + cnt]
        res.append(combine(pad, top=top))
    return res


def shard_norms(x, G: int, top: str = "v1"):
    """Value of each rank's aligned subtree (oracle), in rank order."""
    x = _arr(x)
    dl, dj = TREE[x.dtype]
    res = []
    for (a, cnt, p2l) in shard_ranges(x.size, G, dl * dj):
        if p2l == 0:
            res.append(None)
        else:
            res.append(nrmf(x[a:a + cnt], p2_min=p2l, top=top))
    return res


def combine_ranks(values, top: str = "v1"):
    """Rank tree: R_H (R_A) over the values of ranks that own part of the tree."""
    vals = [v for v in values if v is not None]
    return combine(np.array(vals, dtype=type(vals[0])), top=top)


def exact(x, threads: int | None = None):
    """RN(sqrt(sum x_i^2)) computed exactly (integer superaccumulator).
    Large inputs are accumulated in disjoint chunks on host threads; integer
    addition is exact and associative, so the result does not depend on it."""
    x = _arr(x)
    L = lib()
    if threads is None:
        threads = min(os.cpu_count() or 1, 16) if x.size >= (1 << 22) else 1
    if threads <= 1:
        f = L.exact_nrm_d if _is64(x) else L.exact_nrm_s
        return x.dtype.type(f(x.ctypes.data, x.size))
    from concurrent.futures import ThreadPoolExecutor
    sfx = "d" if _is64(x) else "s"
    words = getattr(L, "exact_acc_words_" + sfx)()
    acc_f = getattr(L, "exact_acc_" + sfx)
    bounds = np.linspace(0, x.size, threads + 1).astype(np.int64)
    accs = [np.zeros(words, dtype=np.uint64) for _ in range(threads)]
    flags = [ctypes.c_int(0) for _ in range(threads)]

    def work(k):
        a, b = int(bounds[k]), int(bounds[k + 1])
        acc_f(x.ctypes.data + a * x.itemsize, b - a, accs[k].ctypes.data, ctypes.byref(flags[k]))

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    for k in range(1, threads):
        L.exact_acc_merge(accs[0].ctypes.data, accs[k].ctypes.data, words)
    fl = 0
    for v in flags:
        fl |= v.value
    return x.dtype.type(getattr(L, "exact_round_" + sfx)(accs[0].ctypes.data, fl))


def relerr(r, ref, dtype=np.float64) -> float:
    """e:relerr: |ref - r| / (ref * eps_x), evaluated exactly."""
    eps = Fraction(EPS[np.dtype(dtype)])
    R, F = Fraction(float(r)), Fraction(float(ref))
    if F == 0:
        return 0.0 if R == 0 else float("inf")
    return float(abs(F - R) / (F * eps))


def reH_plus(dtype=np.float64):
    """1 + eps'^+ of e:reH as an mpmath number (256 bits)."""
    import mpmath
    mpmath.mp.prec = 256
    e = mpmath.mpf(EPS[np.dtype(dtype)])
    return (1 + e) ** mpmath.mpf(2.5) * mpmath.sqrt(1 + e * (2 + e) / 2)


def ub_relerr_H(depth: int, dtype=np.float64) -> float:
    """Upper bound on relerr (in eps units) for a v1_hypot tree whose longest
    root-to-leaf path has `depth` rounding nodes: Thm 3 (e:8) with equal
    children bounds gives 1+eps_[n]^+ = (1+eps_[k]^+)(1+eps'^+) per level."""
    import mpmath
    mpmath.mp.prec = 256
    e = mpmath.mpf(EPS[np.dtype(dtype)])
    return float(((reH_plus(dtype)) ** depth - 1) / e)
