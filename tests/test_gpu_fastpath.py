"""GPU check of the fast node sequences against the CUDA
IEEE-correct intrinsics: wherever a fast node does not flag itself `bad`, its
result equals the exact-intrinsic node bit for bit; the fp32 square root is
checked exhaustively on [1, 2], the fp32 division on every dividend mantissa
against a sample of divisors, fp64 sqrt/node on large random and
near-midpoint samples."""
import ctypes
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "fastcheck.cu")
LIB = os.path.join(HERE, "csrc", "libfastcheck.so")


@pytest.fixture(scope="module")
def fc():
    deps = [SRC, os.path.join(HERE, "..", "paper_2509_06220_b200", "csrc", "nrmf_device.cuh")]
    if not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in deps):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
                               "-Xcompiler", "-fPIC", "-shared", "-o", LIB, SRC])
    L = ctypes.CDLL(LIB)
    L.fastcheck.argtypes = [ctypes.c_int, ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_int,
                            ctypes.POINTER(ctypes.c_ulonglong)]
    L.fastcheck.restype = ctypes.c_int

    def run(which, seed=1, n=1 << 26, mode=0):
        out = (ctypes.c_ulonglong * 3)()
        assert L.fastcheck(which, seed, n, mode, out) == 0
        return out[0], out[1], out[2]
    return run


@pytest.mark.parametrize("mode", [0, 1])
def test_fp64_node_fast_equals_exact(fc, mode):
    checked, fast, mism = fc(0, seed=11 + mode, n=1 << 28, mode=mode)
    assert checked == 1 << 28 and mism == 0
    assert fast > (checked // 3 if mode == 0 else checked - checked // 1000)


@pytest.mark.parametrize("mode", [0, 1])
def test_fp32_node_fast_equals_exact(fc, mode):
    checked, fast, mism = fc(1, seed=21 + mode, n=1 << 28, mode=mode)
    assert checked == 1 << 28 and mism == 0
    assert fast > checked // 3


def test_fp32_sqrt_exhaustive_on_1_2(fc):
    checked, _, mism = fc(2)
    assert checked == (1 << 23) + 1 and mism == 0


def test_fp32_div_all_dividends_sampled_divisors(fc):
    checked, _, mism = fc(3, n=512)     # every dividend x 2048 divisors x 3 scales
    assert checked > 4e10 and mism == 0


@pytest.mark.slow
def test_fp32_div_exhaustive(fc):
    """Every (dividend, divisor) mantissa pair, dividend scaled by 1, 1/2 and
    2^-12 (q = m/M covers [2^-13, 2)): fast sequence == __fdiv_rn."""
    checked, _, mism = fc(3, n=1)
    assert checked > 1.5e14 and mism == 0


def test_fp64_sqrt_random_and_near_midpoints(fc):
    checked, _, mism = fc(4, seed=5, n=1 << 30)
    assert checked == 1 << 30 and mism == 0


@pytest.mark.parametrize("which", [5, 6], ids=["fp64", "fp32"])
def test_internal_node_unchecked_in_fast_domain(fc, which):
    """Internal nodes of a tile run without a range check: in
    the whole fast domain of M -- which the leaf check plus the 12-level growth
    bound guarantees for every internal node -- the unchecked fast node equals
    the exact node bit for bit, for any 0 <= m <= M (q near 1, tiny q,
    subnormal and zero m)."""
    checked, fast, mism = fc(which, seed=31 + which, n=1 << 28)
    assert checked == 1 << 28 and fast == checked and mism == 0


def test_fp64_division_near_midpoints(fc):
    """2^30 divisions m/M constructed to lie within about an ulp of m of a
    rounding midpoint of the quotient (m = RN(M*c), c a midpoint, +-2 ulps),
    over 60 quotient binades and scales across the fast domain: the fast
    sequence equals __ddiv_rn on every one."""
    checked, _, mism = fc(7, seed=77, n=1 << 30)
    assert checked == 1 << 30 and mism == 0


@pytest.mark.parametrize("which", [8, 9], ids=["fp64", "fp32"])
def test_fast_domain_edges(fc, which):
    """M within 64 ulps of every edge of the fast domain (2^-900 / 2^1012 /
    2^1021; fp32 2^-80 / 2^116 / 2^125) and q near 2^-69 (2^-12) and near 1:
    unflagged leaf nodes and in-domain internal nodes equal the exact node."""
    checked, fast, mism = fc(which, seed=91 + which, n=1 << 26)
    assert checked == 1 << 26 and mism == 0 and fast > 0


@pytest.mark.parametrize("which", [10, 11], ids=["fp64", "fp32"])
def test_safe_node_equals_exact_node_everywhere(fc, which):
    """The safe node (v1h_safe_n: the fast sequences on power-of-two-scaled
    operands, the tile fallback) equals the IEEE-intrinsic node of Listing 2
    for every kind of operand: full range incl. subnormals, +-0, +-inf, NaN,
    values near the format's maximum (h overflows), q near 1, M at the edges
    of the scaling ranges; scalar and packed (4 chains) forms."""
    checked, _, mism = fc(which, seed=101 + which, n=1 << 28)
    assert checked == 1 << 28 and mism == 0
