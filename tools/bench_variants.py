"""Dev tool: time nrmf_d / nrmf_s of several libnrmf.so variants on one GPU.

    python tools/bench_variants.py lib1.so lib2.so ...

Inputs are random normal data generated on the device (timing only; parity
is the tests' job).  CUDA-event timing, 2^30 elements, median of 20 reps."""
import ctypes
import statistics
import sys

import torch


def load(path):
    L = ctypes.CDLL(path)
    for f in ("nrmf_d", "nrmf_s"):
        getattr(L, f).argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    return L


def time_one(L, x, reps=20):
    n = x.numel()
    esz = x.element_size()
    ws = torch.zeros(L.nrmf_workspace_bytes(n, esz), dtype=torch.uint8, device="cuda")
    out = torch.empty((), dtype=x.dtype, device="cuda")
    f = L.nrmf_d if esz == 8 else L.nrmf_s
    s = torch.cuda.current_stream().cuda_stream
    call = lambda: f(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s)
    for _ in range(3):
        assert call() == 0
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); call(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), out.item()


def main():
    n = 1 << 30
    xd = torch.randn(n, dtype=torch.float64, device="cuda")
    xs = torch.randn(n, dtype=torch.float32, device="cuda") * 3
    for p in sys.argv[1:]:
        L = load(p)
        td, rd = time_one(L, xd)
        ts, rs = time_one(L, xs)
        print(f"{p}: fp64 {td:.4f} ms ({n*8/td/1e6:.0f} GB/s) r={rd!r}  fp32 {ts:.4f} ms ({n*4/ts/1e6:.0f} GB/s) r={rs!r}",
              flush=True)




def torch_reference():
    n = 1 << 30
    for dt in (torch.float64, torch.float32):
        x = torch.randn(n, dtype=dt, device="cuda")
        for _ in range(3):
            x.sum()
        ts = []
        for _ in range(10):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); x.sum(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        print(f"torch.sum {dt}: {t:.4f} ms ({n * x.element_size() / t / 1e6:.0f} GB/s read)", flush=True)
        del x


if __name__ == "__main__":
    if sys.argv[1:] == ["torch"]:
        torch_reference()
    else:
        main()
