"""Dev tool: bit-compare a libnrmf.so variant with the oracle on a few inputs."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nrmf_inputs as gen  # noqa: E402
import oracle  # noqa: E402

L = ctypes.CDLL(sys.argv[1])
for f in ("nrmf_d", "nrmf_s"):
    getattr(L, f).argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                              ctypes.c_void_p]
L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
L.nrmf_workspace_bytes.restype = ctypes.c_size_t
bad = 0
for dt, f in ((np.float64, L.nrmf_d), (np.float32, L.nrmf_s)):
    sizes = [4096, 5 * 4096 + 3, 300 * 4096 + 77, (1 << 22) + 5]
    if os.environ.get("BIG"):  # persistent-kernel sizes (every warp busy, several rounds, ragged ends)
        sizes += [(1 << 25) + 3 * 4096 + 5, 37 * 16 * 2368 * 4096 // 16 + 4095, (1 << 28) + 12345, 1 << 30]
    for n in sizes:
        x = gen.normal(n, n, dtype=dt)
        xd = torch.from_numpy(x).cuda()
        out = torch.empty((), dtype=xd.dtype, device="cuda")
        ws = torch.zeros(L.nrmf_workspace_bytes(n, x.itemsize), dtype=torch.uint8, device="cuda")
        assert f(n, xd.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream) == 0
        ok = out.cpu().numpy().tobytes() == np.asarray(oracle.nrmf(x), dtype=dt).tobytes()
        bad += not ok
        print(dt.__name__, n, "OK" if ok else "MISMATCH", flush=True)
print("ALL OK" if bad == 0 else f"{bad} MISMATCHES")
