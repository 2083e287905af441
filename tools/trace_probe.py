"""Dev tool: globaltimer event trace of one tree-kernel call (a libnrmf.so
built with -DNRMF_PROBE_TRACE): when warps start, finish groups, climb and
exit -- where the time between the last group and the kernel's end goes.

    python tools/trace_probe.py build/variants/trace.so [lg_n] [split_ll 0|1] [pad KiB before ws]
"""
import collections
import ctypes
import sys

import numpy as np
import torch


def main():
    L = ctypes.CDLL(sys.argv[1])
    lg = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    for f in ("nrmf_d", "nrmf_s"):
        getattr(L, f).argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    L.nrmf_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_uint]
    if len(sys.argv) > 3:
        L.nrmf_debug_set_split_ll.argtypes = [ctypes.c_int]
        L.nrmf_debug_set_split_ll(int(sys.argv[3]))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    n = 1 << lg
    cap = 1 << 20
    buf = torch.zeros(2 * cap, dtype=torch.int64, device="cuda")
    for dt in (torch.float32, torch.float64):
        x = torch.randn(n, dtype=dt, device="cuda")
        esz = x.element_size()
        pad = torch.zeros(max(1, int(sys.argv[4]) if len(sys.argv) > 4 else 0) * 1024, dtype=torch.uint8,
                          device="cuda")
        ws = torch.zeros(L.nrmf_workspace_bytes(n, esz), dtype=torch.uint8, device="cuda")
        out = torch.empty((), dtype=dt, device="cuda")
        print(f"ws at {ws.data_ptr():#x}, out at {out.data_ptr():#x}", flush=True)
        f = L.nrmf_d if esz == 8 else L.nrmf_s
        s = torch.cuda.current_stream().cuda_stream
        for rep in range(4):
            assert L.nrmf_debug_set_trace(buf.data_ptr(), cap) == 0
            flush.zero_()                                  # cold L2, as the bench's C1 step
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            assert f(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s) == 0
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        L.nrmf_debug_set_trace(None, 0)
        a = buf.cpu().numpy().view(np.uint64).reshape(-1, 2)
        a = a[a[:, 1] != 0]
        typ = (a[:, 0] >> 56).astype(int)
        lvl = ((a[:, 0] >> 48) & 0xFF).astype(int)
        wid = (a[:, 0] & ((1 << 48) - 1)).astype(np.int64)
        t = (a[:, 1] - a[:, 1].min()).astype(np.int64) / 1e3  # us
        print(f"== {dt} n=2^{lg}: event-timed {ms * 1e3:.1f} us, {len(a)} events")
        for k, name in ((0, "start"), (5, "batch end"), (1, "group end"), (9, "ll store"), (2, "climb start"),
                        (3, "climb end"), (6, "ll poll start"), (10, "ll polled"), (11, "ll cleared"),
                        (12, "ll in-lane"), (13, "ll shuffles"), (8, "ll root"), (4, "exit")):
            tk = t[typ == k]
            if len(tk):
                print(f"  {name:12s} n={len(tk):6d} min {tk.min():8.1f} med {np.median(tk):8.1f} "
                      f"p99 {np.percentile(tk, 99):8.1f} max {tk.max():8.1f} us")
        # climbs: duration per level
        starts = collections.defaultdict(list)
        for i in np.nonzero(typ == 2)[0]:
            starts[(wid[i], lvl[i])].append(t[i])
        durs = collections.defaultdict(list)
        for i in np.nonzero(typ == 3)[0]:
            st = starts[(wid[i], lvl[i])]
            if st:
                durs[lvl[i]].append(t[i] - st.pop(0))
        for k in sorted(durs):
            d = np.array(durs[k])
            print(f"  climb level {k}: n={len(d)} med {np.median(d):.2f} max {d.max():.2f} us")
        # per warp: groups, climbs, exit time
        ge = collections.Counter(wid[typ == 1])
        cl = collections.Counter(wid[typ == 2])
        ex = {w: tt for w, tt in zip(wid[typ == 4], t[typ == 4])}
        last_ge = {}
        for w, tt in zip(wid[typ == 1], t[typ == 1]):
            last_ge[w] = max(last_ge.get(w, 0), tt)
        worst = sorted(ex, key=lambda w: -ex[w])[:8]
        for w in worst:
            print(f"  warp cta {w >> 24} w {w & 0xffffff}: groups {ge[w]} climbs {cl[w]} "
                  f"last group end {last_ge.get(w, 0):.1f} exit {ex[w]:.1f}")
        byg = collections.defaultdict(list)
        for w in ex:
            byg[(ge[w], cl[w])].append(ex[w])
        for key in sorted(byg):
            v = np.array(byg[key])
            print(f"  groups {key[0]} climbs {key[1]}: warps {len(v)} exit med {np.median(v):.1f} max {v.max():.1f}")
        del x, ws


if __name__ == "__main__":
    main()
