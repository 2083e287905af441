"""Dev tool: A/B timing of libnrmf.so variants at the bench's operating point.

    python tools/ab.py [--lg 30] [--rounds 5] [--reps 20] [--cool 3] lib1.so lib2.so ...

Each round: for each library in turn, let the GPU cool for --cool seconds,
then time --reps back-to-back calls of nrmf_d and of nrmf_s (CUDA events per
call, median) -- the burst regime the driver's 20-step bench sees.  Rounds
interleave the libraries, so drift hits all alike.  Reports per-library
median and min over rounds."""
import argparse
import ctypes
import statistics
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


def timed(L, x, reps):
    n = x.numel()
    ws = torch.zeros(L.nrmf_workspace_bytes(n, x.element_size()), dtype=torch.uint8, device="cuda")
    out = torch.empty((), dtype=x.dtype, device="cuda")
    f = L.nrmf_d if x.element_size() == 8 else L.nrmf_s
    s = torch.cuda.current_stream().cuda_stream
    call = lambda: f(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s)  # noqa: E731
    call()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        call()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev), out.item()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--lg", type=int, default=30)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cool", type=float, default=3.0)
    a = ap.parse_args()
    n = 1 << a.lg
    xd = torch.randn(n, dtype=torch.float64, device="cuda")
    xs = torch.randn(n, dtype=torch.float32, device="cuda")
    libs = [(p, load(p)) for p in a.libs]
    res = {p: ([], [], None) for p in a.libs}
    for _ in range(a.rounds):
        for p, L in libs:
            time.sleep(a.cool)
            td, rd = timed(L, xd, a.reps)
            ts, rs = timed(L, xs, a.reps)
            res[p][0].append(td)
            res[p][1].append(ts)
            res[p] = (res[p][0], res[p][1], (rd, rs))
    for p in a.libs:
        d, s, r = res[p]
        print(f"{p}: fp64 med {statistics.median(d):.4f} min {min(d):.4f} ms | fp32 med {statistics.median(s):.4f} "
              f"min {min(s):.4f} ms | results {r}", flush=True)


if __name__ == "__main__":
    main()
