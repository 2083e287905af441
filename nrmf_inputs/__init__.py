"""Seeded, counter-based, index-addressable input generators.

Shared by tests, bench.py and the oracle runs.  Holds none of the method's
arithmetic: it only maps (seed, stream, index) to input values, so element i
has the same bits whether it is generated whole, per shard, or per chunk.

The C source is ``gen.c``; ``build()`` compiles it with gcc (OpenMP) into
``libnrmf_gen.so`` next to this file.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libnrmf_gen.so")
_lib = None

# BASELINE.json configs (DESIGN.md §5 input recipe)
C2_ELO, C2_EHI = -20, 20
C4_KLO, C4_KHI = -30, 30
DBL_MAX = np.finfo(np.float64).max


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, u64, i32, f64 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        vp = ctypes.c_void_p
        L.gen_key.argtypes = [u64, u64]; L.gen_key.restype = u64
        L.gen_u64.argtypes = [u64, u64, i64, i64, vp]
        L.gen_uniform_pm1_d.argtypes = [u64, i64, i64, vp]
        L.gen_uniform_pm1_s.argtypes = [u64, i64, i64, vp]
        L.gen_sme_s.argtypes = [u64, i64, i64, i32, i32, vp]
        L.gen_sme_d.argtypes = [u64, i64, i64, i32, i32, vp]
        L.gen_normal_d.argtypes = [u64, i64, i64, vp]
        L.gen_normal_s.argtypes = [u64, i64, i64, vp]
        L.gen_colscaled_normal_d.argtypes = [u64, i64, i64, i64, i64, i32, i32, vp]
        L.gen_colscaled_normal_s.argtypes = [u64, i64, i64, i64, i64, i32, i32, vp]
        L.gen_extreme_d.argtypes = [u64, i64, i64, i32, f64, i64, vp]
        for f in ("gen_u64", "gen_uniform_pm1_d", "gen_uniform_pm1_s", "gen_sme_s", "gen_sme_d",
                  "gen_normal_d", "gen_normal_s", "gen_colscaled_normal_d",
                  "gen_colscaled_normal_s", "gen_extreme_d"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


def _out(out, cnt, dtype):
    if out is None:
        out = np.empty(cnt, dtype=dtype)
    assert out.dtype == dtype and out.size >= cnt and out.flags.c_contiguous
    return out


def u64(seed: int, stream: int, off: int, cnt: int) -> np.ndarray:
    out = np.empty(cnt, dtype=np.uint64)
    lib().gen_u64(seed, stream, off, cnt, _ptr(out))
    return out


def uniform_pm1(seed: int, n: int, off: int = 0, dtype=np.float64, out=None) -> np.ndarray:
    """C1: i.i.d. uniform in [-1, 1)."""
    out = _out(out, n, dtype)
    f = lib().gen_uniform_pm1_d if dtype == np.float64 else lib().gen_uniform_pm1_s
    f(seed, off, n, _ptr(out))
    return out


def sme(seed: int, n: int, off: int = 0, elo: int = C2_ELO, ehi: int = C2_EHI,
        dtype=np.float32, out=None) -> np.ndarray:
    """C2: x = s*m*2^e, s = +-1, m in [1,2), e uniform integer in [elo, ehi]."""
    out = _out(out, n, dtype)
    f = lib().gen_sme_s if dtype == np.float32 else lib().gen_sme_d
    f(seed, off, n, elo, ehi, _ptr(out))
    return out


def normal(seed: int, n: int, off: int = 0, dtype=np.float64, out=None) -> np.ndarray:
    """C3: standard normal (host Box-Muller)."""
    out = _out(out, n, dtype)
    f = lib().gen_normal_d if dtype == np.float64 else lib().gen_normal_s
    f(seed, off, n, _ptr(out))
    return out


def colscaled_normal(seed: int, r: int, c: int, ld: int | None = None, c0: int = 0,
                     cc: int | None = None, klo: int = C4_KLO, khi: int = C4_KHI,
                     dtype=np.float64, out=None) -> np.ndarray:
    """C4: column-major r x c, A_ij = z_ij * 2^k_j.  Returns a flat array of
    cc*ld entries holding columns [c0, c0+cc) (rows r..ld-1 are zero)."""
    ld = r if ld is None else ld
    cc = c - c0 if cc is None else cc
    if out is None:
        out = np.zeros(cc * ld, dtype=dtype)
    f = lib().gen_colscaled_normal_d if dtype == np.float64 else lib().gen_colscaled_normal_s
    f(seed, r, ld, c0, cc, klo, khi, _ptr(out))
    return out


def extreme(seed: int, n: int, variant: str = "fin2", off: int = 0, out=None) -> np.ndarray:
    """C5 extreme-range fp64 (reading R9):
    lit  -- exponents over [-1074, 1023], magnitudes capped at 0.99*DBL_MAX (norm overflows)
    fin  -- exponents over [-1074, 1003] plus one planted +-0.99*DBL_MAX element
    fin2 -- exponents over [-1074, 1008], nothing planted
    """
    vmax = 0.99 * DBL_MAX
    if variant == "lit":
        emax, plant = 1023, -1
    elif variant == "fin":
        emax, plant = 1003, int(u64(seed, 6, 0, 1)[0] % np.uint64(max(n, 1)))
    elif variant == "fin2":
        emax, plant = 1008, -1
    else:
        raise ValueError(variant)
    out = _out(out, n, np.float64)
    lib().gen_extreme_d(seed, off, n, emax, vmax, plant, _ptr(out))
    return out
