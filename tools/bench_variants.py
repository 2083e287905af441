"""Dev tool: time nrmf_d / nrmf_s of several libnrmf.so variants on one GPU.

    python tools/bench_variants.py lib1.so lib2.so ...

Inputs are random normal data generated on the device (timing only; parity
is the tests' job).  CUDA-event timing, 2^30 elements, median of 20 reps."""
import ctypes
import os
import statistics
import sys
import time

import torch


def load(path):
    L = ctypes.CDLL(path)
    for f in ("nrmf_d", "nrmf_s"):
        getattr(L, f).argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    return L


class Clock:
    """NVML SM-clock sampler (MHz) running while the context is open."""

    def __init__(self):
        import threading
        import pynvml as nv
        nv.nvmlInit()
        self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.samples, self.stop, self.threading = [], None, threading

    def __enter__(self):
        self.samples = []
        self.stop = self.threading.Event()

        def run():
            while not self.stop.is_set():
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                time.sleep(0.002)
        self.t = self.threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join()

    def mhz(self):
        return statistics.mean(self.samples) if self.samples else float("nan")


CLK = None


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
    global CLK
    if CLK is None:
        CLK = Clock()
    with CLK:
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); call(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
    # time normalised to the 1965 MHz max clock (compute-bound kernels scale with the clock)
    time_one.last_mhz = CLK.mhz()
    return statistics.median(ts), out.item()


def main():
    """Variants are timed in interleaved rounds (A B C A B C ...) so that a
    drift of the SM clock over the run (power/thermal) hits all of them alike;
    the report is the per-variant minimum and median over rounds."""
    n = 1 << 30
    rounds = int(os.environ.get("ROUNDS", "3"))
    xd = torch.randn(n, dtype=torch.float64, device="cuda")
    xs = torch.randn(n, dtype=torch.float32, device="cuda") * 3
    libs = [(p, load(p)) for p in sys.argv[1:]]
    res = {p: ([], [], [], [], None, None) for p, _ in libs}
    for _ in range(rounds):
        for p, L in libs:
            td, rd = time_one(L, xd, reps=10)
            cd = time_one.last_mhz
            ts, rs = time_one(L, xs, reps=10)
            cs = time_one.last_mhz
            d, f, nd, nf, _, _ = res[p]
            d.append(td); f.append(ts); nd.append(td * cd / 1965.0); nf.append(ts * cs / 1965.0)
            res[p] = (d, f, nd, nf, rd, rs)
    for p, _ in libs:
        d, f, nd, nf, rd, rs = res[p]
        print(f"{p}: fp64 min {min(d):.4f} med {statistics.median(d):.4f} ms @1965-norm {statistics.median(nd):.4f} | "
              f"fp32 min {min(f):.4f} med {statistics.median(f):.4f} ms @1965-norm {statistics.median(nf):.4f} "
              f"| r={rd!r} {rs!r}", flush=True)




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
