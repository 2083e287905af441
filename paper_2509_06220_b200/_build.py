"""Build libnrmf.so in-tree with nvcc for sm_100a (no JIT cache, no fallback)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libnrmf.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("nrmf.cu", "nrmf_dist.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("nrmf_device.cuh", "nrmf_internal.h",
                                                           "nrmf_crhypot.cuh", "nrmf_p2p.cuh")] + [
    os.path.join(ROOT, "include", "nrmf.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # IEEE arithmetic exactly as written: no contraction, correct div/sqrt, no FTZ
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    """Compile libnrmf.so (or a variant with extra -D defines into `out`)."""
    target = out or LIB
    if out is None and not defines and not force and not stale():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, *(f"-D{d}" for d in defines), "-o", target + ".tmp", *SOURCES, "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force=True, verbose=True)
