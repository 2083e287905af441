"""Dev tool: C1-sized (and other small / unaligned) calls of several
libnrmf.so builds, A/B on one box: each call captured in a CUDA graph (flags
NRMF_WS_CLEAN, as bench.py's capture does), L2 flushed before every replay,
median device time over rounds that interleave the builds (by default by
difference: reps x [flush; call] minus reps x [flush], see --diff).

    python tools/c1_ab.py lib1.so lib2.so ... [--lg 20] [--off 0] [--dtype d]"""
import argparse
import ctypes
import statistics

import torch


def load(path):
    L = ctypes.CDLL(path)
    for f in ("nrmf_ex_d", "nrmf_ex_s"):
        getattr(L, f).argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    L.nrmf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.nrmf_workspace_bytes.restype = ctypes.c_size_t
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--lg", type=int, default=20)
    ap.add_argument("--off", type=int, default=0, help="element offset of the base (1: 8 bytes off for fp64)")
    ap.add_argument("--dtype", default="d")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--flush", type=int, default=1)
    ap.add_argument("--pad", type=int, default=0, help="KiB allocated before each workspace (address probe)")
    ap.add_argument("--wspad", type=int, default=0, help="extra KiB of workspace (layout probe)")
    ap.add_argument("--diff", type=int, default=1,
                    help="1: time reps x [flush; call] and reps x [flush] with one event pair each and report the "
                         "difference per call (per-call event pairs behind a flush carry ~4 us of event overhead "
                         "and ~2.05 us steps on this pool: tools/timer_probe.py); 0: per-call event pairs")
    a = ap.parse_args()
    dt = torch.float64 if a.dtype == "d" else torch.float32
    n = 1 << a.lg
    xb = torch.randn(n + a.off, dtype=dt, device="cuda")
    x = xb[a.off:]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    graphs = []
    for p in a.libs:
        L = load(p)
        keep = torch.zeros(max(1, a.pad) * 1024, dtype=torch.uint8, device="cuda")
        ws = torch.zeros(L.nrmf_workspace_bytes(n, x.element_size()) + a.wspad * 1024, dtype=torch.uint8, device="cuda")
        out = torch.empty((), dtype=dt, device="cuda")
        f = L.nrmf_ex_d if a.dtype == "d" else L.nrmf_ex_s
        s = torch.cuda.Stream()
        call = lambda f=f, ws=ws, out=out, s=s: f(n, x.data_ptr(), out.data_ptr(), 2, ws.data_ptr(), ws.numel(),  # noqa: E731
                                                  s.cuda_stream)
        with torch.cuda.stream(s):
            for _ in range(3):
                assert call() == 0
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            assert call() == 0
        graphs.append((p, g, out, (ws, keep)))
        print(f"{p}: ws at {ws.data_ptr():#x} ({ws.numel()} B), out at {out.data_ptr():#x}, x at {x.data_ptr():#x}", flush=True)
    res = {p: [] for p in a.libs}

    def seq(body):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            body()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / a.reps

    for _ in range(a.rounds):
        for p, g, out, _ in graphs:
            if a.diff:
                t_fc = seq(lambda g=g: (flush.zero_(), g.replay()))
                t_f = seq(lambda: flush.zero_())
                res[p].append(t_fc - t_f)
                continue
            ts = []
            for _ in range(a.reps):
                if a.flush:
                    flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                ts.append((e0, e1))
            torch.cuda.synchronize()
            res[p].append(statistics.median(e0.elapsed_time(e1) for e0, e1 in ts) * 1e3)
    for p, g, out, _ in graphs:
        print(f"{p}: lg {a.lg} off {a.off} {a.dtype}: median {statistics.median(res[p]):.2f} us "
              f"(rounds {', '.join(f'{v:.2f}' for v in res[p])}) result {out.item()!r}", flush=True)


if __name__ == "__main__":
    main()
