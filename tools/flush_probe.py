"""Dev probe: what an L2 flush (256 MiB write) right before the start event
adds to an event-timed call -- a tiny torch kernel and the C1 call (2^20 fp64,
one graph node) -- with the flush alone, with a no-op kernel between the
flush and the start event, and with no flush.

    python tools/flush_probe.py [lib.so]"""
import ctypes
import sys

import numpy as np
import torch


def timed(fn, pre, reps=30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        pre()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts[5:]))


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2509_06220_b200/libnrmf.so"
    L = ctypes.CDLL(lib)
    L.nrmf_ex_d.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                            ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tiny = torch.zeros(1, device="cuda")
    n = 1 << 20
    x = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
    ws = torch.zeros(L.nrmf_workspace_bytes(n, 8), dtype=torch.uint8, device="cuda")
    out = torch.empty((), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        assert L.nrmf_ex_d(n, x.data_ptr(), out.data_ptr(), 0, ws.data_ptr(), ws.numel(), s.cuda_stream) == 0
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            assert L.nrmf_ex_d(n, x.data_ptr(), out.data_ptr(), 2, ws.data_ptr(), ws.numel(), s.cuda_stream) == 0
        torch.cuda.synchronize()
        pres = {"flush": lambda: flush.zero_(),
                "flush + no-op kernel": lambda: (flush.zero_(), tiny.add_(0)),
                "flush + read 1 MiB": lambda: (flush.zero_(), flush[: 1 << 20].sum()),
                "no flush": lambda: None}
        for name, pre in pres.items():
            a = timed(lambda: tiny.add_(1), pre)
            b = timed(g.replay, pre)
            print(f"{name:22s}: tiny kernel {a:5.2f} us   C1 graph replay {b:5.2f} us")


if __name__ == "__main__":
    main()
