"""Race stress of the combine protocols: a test build of
the library (-DNRMF_PROBE_JITTER) sleeps a random 0-4 us at every step of the
CTA combine step (deposit, count, claim, slot release), of the last-arriver
climbs (announce, value store, acquire) and of the split kernel's announce,
so that warps interleave in orders deterministic timing never produces.
1000 calls per dtype over persistent grids of 1-5 CTAs (many rounds per CTA,
slot reuse, partial last blocks) and the split kernel: every result must be
the oracle's bits (parity: same tree, any arrival order)."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import nrmf_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tests", "csrc", "libnrmf_jitter.so")
T = 4096


@pytest.fixture(scope="module")
def J():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    sys.path.insert(0, os.path.join(ROOT, "paper_2509_06220_b200"))
    import _build
    deps = _build.DEPS
    if not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in deps):
        _build.build(out=LIB, defines=("NRMF_PROBE_JITTER",))
    L = ctypes.CDLL(LIB)
    i64, vp, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    for f in ("nrmf_d", "nrmf_s"):
        getattr(L, f).argtypes = [i64, vp, vp, vp, sz, vp]
        getattr(L, f).restype = ctypes.c_int
    L.nrmf_workspace_bytes.argtypes = [i64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = sz
    L.nrmf_debug_set_grid.argtypes = [ctypes.c_int]
    return L


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_jittered_combine_keeps_the_bits(J, dt):
    tdt = torch.float64 if dt == np.float64 else torch.float32
    f = J.nrmf_d if dt == np.float64 else J.nrmf_s
    cases = []
    for n in (1000 * T + 123, 333 * T + 7, 64 * T):
        x = gen.normal(n + 3, n, dtype=dt)
        cases.append((n, torch.from_numpy(x).cuda(), np.asarray(oracle.nrmf(x), dtype=dt).tobytes()))
    s = torch.cuda.current_stream().cuda_stream
    runs = 0
    try:
        for grid in (0, 1, 2, 3, 4, 5):          # 0: automatic (split kernel at these sizes)
            J.nrmf_debug_set_grid(grid)
            for n, xd, want in cases:
                ws = torch.zeros(J.nrmf_workspace_bytes(n, xd.element_size()), dtype=torch.uint8, device="cuda")
                outs = torch.empty(56, dtype=tdt, device="cuda")
                for i in range(56):
                    assert f(n, xd.data_ptr(), outs[i:].data_ptr(), ws.data_ptr(), ws.numel(), s) == 0
                torch.cuda.synchronize()
                got = outs.cpu().numpy()
                for i in range(56):
                    assert got[i].tobytes() == want, (grid, n, i)
                runs += 56
    finally:
        J.nrmf_debug_set_grid(0)
    assert runs >= 1000
