"""Dev tool: per-warp event times of one small (split-kernel) call, from a
libnrmf.so built with -DNRMF_PROBE_TRACE -DNRMF_PROBE_TRACE2 (one globaltimer
slot per warp and event, no atomics), L2 flushed before the call as in the
bench's C1 step.  Prints each event's spread relative to the first warp's
start, and the event-timed call beside an empty kernel's.

    python tools/trace2_probe.py build/variants/trace2.so [lg_n] [reps]
"""
import ctypes
import sys

import numpy as np
import torch

NAMES = {0: "start", 14: "batch loaded", 5: "batch end", 15: "after CTA barrier", 1: "group value",
         9: "ll store", 6: "ll poll start", 10: "ll polled", 11: "ll cleared", 12: "ll in-lane",
         13: "ll shuffles", 8: "ll root", 3: "ll poll round 1", 2: "ll poll round 2"}


def main():
    L = ctypes.CDLL(sys.argv[1])
    lg = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    for f in ("nrmf_d", "nrmf_s"):
        getattr(L, f).argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    L.nrmf_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_uint]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    n = 1 << lg
    s = torch.cuda.current_stream().cuda_stream
    # reference: an (almost) empty launch, event-timed the same way
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tiny = torch.zeros(1, device="cuda")
    ts = []
    for _ in range(20):
        flush.zero_()
        e0.record(); tiny.add_(1); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"empty-ish kernel (tensor add_), event-timed: median {np.median(ts):.1f} us")
    for dt in (torch.float64, torch.float32):
        x = torch.randn(n, dtype=dt, device="cuda")
        esz = x.element_size()
        ws = torch.zeros(L.nrmf_workspace_bytes(n, esz), dtype=torch.uint8, device="cuda")
        out = torch.empty((), dtype=dt, device="cuda")
        f = L.nrmf_d if esz == 8 else L.nrmf_s
        nw = 4096 * 32
        buf = torch.zeros(nw * 16, dtype=torch.int64, device="cuda")
        acc = {k: [] for k in NAMES}
        tot = []
        for rep in range(reps):
            buf.zero_()
            assert L.nrmf_debug_set_trace(buf.data_ptr(), nw * 16) == 0
            flush.zero_()
            e0.record()
            assert f(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s) == 0
            e1.record()
            torch.cuda.synchronize()
            tot.append(e0.elapsed_time(e1) * 1e3)
            a = buf.cpu().numpy().view(np.uint64).reshape(nw, 16).astype(np.float64)
            t0 = a[:, 0][a[:, 0] > 0].min()
            for k in NAMES:
                col = a[:, k]
                col = col[col > 0]
                if len(col):
                    acc[k].append(((col - t0) / 1e3))
            spins = a[:, 7][a[:, 7] > 0]
            acc.setdefault("spins", []).append(spins)
        L.nrmf_debug_set_trace(None, 0)
        print("  poll rounds per call:", [int(v[0]) if len(v) else None for v in acc["spins"]],
              "(None: the two-warp last step records no round count)")
        print(f"== {dt} n=2^{lg}: event-timed median {np.median(tot):.1f} us over {reps} calls "
              f"(last {reps - 1} averaged below)")
        for k, name in NAMES.items():
            if not acc[k]:
                continue
            v = acc[k][1:] if len(acc[k]) > 1 else acc[k]
            mins = np.mean([x.min() for x in v]); meds = np.mean([np.median(x) for x in v])
            maxs = np.mean([x.max() for x in v])
            print(f"  {name:18s} n={len(v[0]):5d} min {mins:6.2f} med {meds:6.2f} max {maxs:6.2f} us")


if __name__ == "__main__":
    main()
