"""Dev tool: device time of one libnrmf.so variant per forced warp-group size
(g0) at n = 2^30, fp32 and fp64 -- with a NRMF_PROBE_CHEAP_NODE build this is
the stream loader's own bandwidth ceiling per group size.

    python tools/loader_probe.py lib.so [g0 ...]
"""
import ctypes
import statistics
import sys

import torch


def main():
    L = ctypes.CDLL(sys.argv[1])
    g0s = [int(a) for a in sys.argv[2:]] or [-1, 0, 1, 2, 3, 4]
    for f in ("nrmf_d", "nrmf_s"):
        getattr(L, f).argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    L.nrmf_debug_set_g0.argtypes = [ctypes.c_int]
    n = 1 << 30
    for dt in (torch.float32, torch.float64):
        x = torch.randn(n, dtype=dt, device="cuda")
        esz = x.element_size()
        ws = torch.zeros(L.nrmf_workspace_bytes(n, esz), dtype=torch.uint8, device="cuda")
        out = torch.empty((), dtype=dt, device="cuda")
        f = L.nrmf_d if esz == 8 else L.nrmf_s
        s = torch.cuda.current_stream().cuda_stream
        for g0 in g0s:
            L.nrmf_debug_set_g0(g0)
            for _ in range(3):
                assert f(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s) == 0
            ts = []
            for _ in range(15):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                f(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            print(f"{dt} g0={g0}: {t:.4f} ms  {n * esz / t / 1e6:.0f} GB/s", flush=True)
        L.nrmf_debug_set_g0(-1)
        del x, ws


if __name__ == "__main__":
    main()
