"""Dev probe: resolution of CUDA-event timing on this box, and a small call
(default C1: 2^20 fp64, one graph node, L2 flushed before every call)
measured two ways: per-call event pairs (bench.py's flushed loop) and by
difference, t(K x [flush; call]) - t(K x [flush]), one event pair around each
whole sequence (intervals of milliseconds: the timer's step does not matter).

    nvcc ... -o tools/timer_probe_k.so tools/timer_probe_k.cu   (see that file)
    python tools/timer_probe.py [lib.so] [lg ...]"""
import ctypes
import sys

import numpy as np
import torch


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2509_06220_b200/libnrmf.so"
    lgs = [int(a) for a in sys.argv[2:]] or [20]
    K = ctypes.CDLL("tools/timer_probe_k.so")
    K.launch_spin.argtypes = [ctypes.c_longlong, ctypes.c_void_p]
    K.launch_ticks.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    L = ctypes.CDLL(lib)
    L.nrmf_ex_d.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                            ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(s):
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        K.launch_ticks(out.data_ptr(), 100000, sp)
        torch.cuda.synchronize()
        print(f"smallest %globaltimer step: {int(out.item())} ns")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # event pairs around globaltimer spins of known length, behind a flush
        print("event-timed spin kernels (flush before each):")
        for ns in (1000, 1500, 2000, 2500, 3000, 4000, 5000, 6000, 8000):
            ts = []
            for _ in range(20):
                flush.zero_()
                e0.record(s)
                K.launch_spin(ns, sp)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            print(f"  spin {ns / 1e3:4.1f} us: event median {np.median(ts):6.2f} us, distinct values "
                  f"{sorted(set(round(t, 2) for t in ts))[:6]}")
        for lg in lgs:
            n = 1 << lg
            x = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
            ws = torch.zeros(L.nrmf_workspace_bytes(n, 8), dtype=torch.uint8, device="cuda")
            res = torch.empty((), dtype=torch.float64, device="cuda")
            assert L.nrmf_ex_d(n, x.data_ptr(), res.data_ptr(), 0, ws.data_ptr(), ws.numel(), sp) == 0
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                assert L.nrmf_ex_d(n, x.data_ptr(), res.data_ptr(), 2, ws.data_ptr(), ws.numel(), sp) == 0
            torch.cuda.synchronize()
            # per-call event pairs
            ts = []
            for _ in range(50):
                flush.zero_()
                e0.record(s)
                g.replay()
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            # by difference over long sequences
            Kn = 200
            seq = {}
            for name, body in (("flush+call", lambda: (flush.zero_(), g.replay())),
                               ("flush+spin0", lambda: (flush.zero_(), K.launch_spin(0, sp))),
                               ("flush", lambda: flush.zero_())):
                vals = []
                for _ in range(3):
                    torch.cuda.synchronize()
                    e0.record(s)
                    for _ in range(Kn):
                        body()
                    e1.record(s)
                    torch.cuda.synchronize()
                    vals.append(e0.elapsed_time(e1) * 1e3 / Kn)
                seq[name] = float(np.median(vals))
            print(f"2^{lg} fp64: per-call events median {np.median(ts):6.2f} us (distinct "
                  f"{sorted(set(round(t, 2) for t in ts))[:5]}); by difference: call {seq['flush+call'] - seq['flush']:6.2f} us, "
                  f"empty kernel {seq['flush+spin0'] - seq['flush']:6.2f} us (flush {seq['flush']:.1f} us)")


if __name__ == "__main__":
    main()
