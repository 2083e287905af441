"""Dev probe: how evenly the persistent kernel's CTAs progress.  One traced call
(libnrmf.so built with -DNRMF_PROBE_TRACE) at n = 2^lg: per CTA, the end time
of its last group and the mean time per group; per warp, the same.  If the
slowest CTAs finish well after the median, a static round-robin of groups
leaves the fast SMs idle at the end (dynamic claiming would rebalance).

    python tools/cta_spread.py build/variants/trace1.so [lg] [d|s]"""
import ctypes
import sys

import numpy as np
import torch


def main():
    L = ctypes.CDLL(sys.argv[1])
    lg = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    dt = torch.float64 if (sys.argv[3] if len(sys.argv) > 3 else "d") == "d" else torch.float32
    for f in ("nrmf_d", "nrmf_s"):
        getattr(L, f).argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    L.nrmf_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_uint]
    n = 1 << lg
    cap = 1 << 21
    buf = torch.zeros(2 * cap, dtype=torch.int64, device="cuda")
    x = torch.randn(n, dtype=dt, device="cuda")
    ws = torch.zeros(L.nrmf_workspace_bytes(n, x.element_size()), dtype=torch.uint8, device="cuda")
    out = torch.empty((), dtype=dt, device="cuda")
    f = L.nrmf_d if x.element_size() == 8 else L.nrmf_s
    s = torch.cuda.current_stream().cuda_stream
    for rep in range(3):
        buf.zero_()
        assert L.nrmf_debug_set_trace(buf.data_ptr(), cap) == 0
        assert f(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s) == 0
        torch.cuda.synchronize()
        L.nrmf_debug_set_trace(None, 0)
        a = buf.cpu().numpy().view(np.uint64).reshape(-1, 2)
        a = a[a[:, 1] != 0]
        typ = (a[:, 0] >> 56).astype(int)
        cta = ((a[:, 0] >> 24) & 0xFFFFFF).astype(int)
        wid = (a[:, 0] & 0xFFFFFF).astype(int)
        t = (a[:, 1] - a[:, 1].min()).astype(np.int64) / 1e3
        g = typ == 1
        ends = {}
        cnt = {}
        for c, w, tt in zip(cta[g], wid[g], t[g]):
            ends[c] = max(ends.get(c, 0.0), tt)
            cnt[c] = cnt.get(c, 0) + 1
        cs = np.array(sorted(ends))
        e = np.array([ends[c] for c in cs])
        k = np.array([cnt[c] for c in cs])
        per = e / k
        print(f"rep {rep}: {dt} n=2^{lg}: {len(cs)} CTAs, groups per CTA {k.min()}..{k.max()}; "
              f"last group end min {e.min():.1f} med {np.median(e):.1f} max {e.max():.1f} us; "
              f"us per group min {per.min():.2f} med {np.median(per):.2f} max {per.max():.2f}")
        if rep == 2:
            order = np.argsort(per)
            print("  slowest CTAs (us/group):", [(int(cs[i]), round(float(per[i]), 2)) for i in order[-8:]])
            print("  fastest CTAs (us/group):", [(int(cs[i]), round(float(per[i]), 2)) for i in order[:8]])


if __name__ == "__main__":
    main()
