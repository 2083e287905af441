"""the A-style top levels (NRMF_TOP_CR): cr_hypot above the tile
level.  GPU cr_hypot is checked against the oracle's exact cr_hypot (exact
integer RN(sqrt(x^2+y^2))), and every entry point with top="cr" against the
oracle's tree with cr_hypot above the tiles, bit for bit."""
import ctypes
import os
import subprocess

import numpy as np
import pytest
import torch

import nrmf_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
T = 4096


@pytest.fixture(scope="module")
def nrmf():
    assert torch.cuda.is_available()
    from paper_2509_06220_b200 import _build
    _build.build()
    import paper_2509_06220_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="module")
def fc():
    src = os.path.join(HERE, "csrc", "fastcheck.cu")
    lib = os.path.join(HERE, "csrc", "libfastcheck.so")
    deps = [src] + [os.path.join(HERE, "..", "paper_2509_06220_b200", "csrc", f)
                    for f in ("nrmf_device.cuh", "nrmf_crhypot.cuh")]
    if not os.path.exists(lib) or any(os.path.getmtime(d) > os.path.getmtime(lib) for d in deps):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
                               "-Xcompiler", "-fPIC", "-shared", "-o", lib, src])
    L = ctypes.CDLL(lib)
    L.crhypot_array.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    return L


def bits(v, dt):
    return np.asarray(v, dtype=dt).tobytes()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_device_cr_hypot_vs_exact(fc, dt):
    rng = np.random.default_rng(31)
    n = 1 << 20
    emin, emax = (-1074, 1023) if dt == np.float64 else (-149, 127)
    a = np.ldexp(rng.uniform(1, 2, n), rng.integers(emin, emax, n))
    b = np.ldexp(rng.uniform(1, 2, n), rng.integers(emin, emax, n))
    k = n // 4
    b[:k] = a[:k] * np.ldexp(rng.uniform(0.5, 1, k), -rng.integers(0, 30, k))   # close exponents
    a[k:2 * k] = rng.integers(1, 1 << 40, k) * np.ldexp(1.0, emin)               # subnormal / tiny
    b[k:2 * k] = rng.integers(1, 1 << 40, k) * np.ldexp(1.0, emin)
    a[2 * k:2 * k + 64] = [3, 5, 8, 20, 7, 0, np.inf, np.nan] * 8
    b[2 * k:2 * k + 64] = [4, 12, 15, 21, 24, 0, np.nan, 1.0] * 8
    a = (a * np.where(rng.integers(0, 2, n) == 1, -1, 1)).astype(dt)
    b = b.astype(dt)
    da, db = dev(a), dev(b)
    out = torch.empty_like(da)
    assert fc.crhypot_array(1 if dt == np.float64 else 0, n, da.data_ptr(), db.data_ptr(), out.data_ptr()) == 0
    got = out.cpu().numpy()
    exp = oracle.cr_hypot_array(a, b)
    nan = np.isnan(exp)
    assert np.array_equal(np.isnan(got), nan)
    assert got[~nan].tobytes() == exp[~nan].tobytes()


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", [1, 4096, 4097, 9 * T + 1, 300 * T + 77, (1 << 22) + 3])
def test_vector_top_cr(nrmf, dt, n):
    x = gen.normal(n, n, dtype=dt)
    r = nrmf.norm(dev(x), top="cr").cpu().numpy()
    assert bits(r, dt) == bits(oracle.nrmf(x, top="cr"), dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("r,c", [(4096, 300), (9000, 33), (1000, 77)])
def test_cols_top_cr(nrmf, dt, r, c):
    A = gen.colscaled_normal(5, r, c, dtype=dt)
    col, fr = nrmf.cols(dev(A).as_strided((r, c), (1, r)), top="cr")
    ecol, efr = oracle.cols(A, r, c, r, top="cr")
    assert col.cpu().numpy().tobytes() == ecol.tobytes()
    assert bits(fr.cpu().numpy(), dt) == bits(efr, dt)


def test_host_and_dist_top_cr(nrmf):
    import torch.distributed as td
    x = gen.normal(9, 3 * 512 * T + 5)
    exp = bits(oracle.nrmf(x, top="cr"), np.float64)
    assert bits(nrmf.norm(torch.from_numpy(x).pin_memory(), top="cr").numpy(), np.float64) == exp
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29534")
    created = not td.is_initialized()
    if created:
        td.init_process_group("gloo", rank=0, world_size=1)
    try:
        assert bits(nrmf.dist(dev(x), x.size, top="cr").cpu().numpy(), np.float64) == exp
    finally:
        for c in list(nrmf._comms.values()):
            c.close()
        nrmf._comms.clear()
        if created:
            td.destroy_process_group()


@pytest.mark.slow
def test_c3_top_cr_bound_is_a_theorem(nrmf):
    """n = 2^30: 12 v1 levels in the tile + 18 cr levels above: the Thm-3 bound
    ((1+eps'+)^12 (1+eps)^18 - 1)/eps = 54 < 64."""
    import mpmath
    n = 1 << 30
    x = gen.normal(1, n)
    r = nrmf.norm(dev(x), top="cr").cpu().numpy()
    assert bits(r, np.float64) == bits(oracle.nrmf(x, top="cr"), np.float64)
    mpmath.mp.prec = 200
    eps = mpmath.mpf(2) ** -53
    ub = float(((oracle.reH_plus()) ** 12 * (1 + eps) ** 18 - 1) / eps)
    assert ub < 64
    assert oracle.relerr(r, oracle.exact(x)) <= ub
