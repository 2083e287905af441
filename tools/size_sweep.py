"""Dev tool: device time of nrmf_d / nrmf_s over sizes.

Each measurement replays a CUDA graph of R back-to-back calls (R = 20 for
small n), so host overhead (Python, ctypes, launch) is not in the number."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_06220_b200 as nrmf  # noqa: E402

if len(sys.argv) > 1:            # time another build of the library
    nrmf.LIB_PATH = sys.argv[1]


def t(x, reps):
    out = torch.empty((), dtype=x.dtype, device="cuda")
    R = 20 if x.numel() <= (1 << 24) else 1

    def calls():
        for _ in range(R):
            nrmf.norm(x, out=out)
    g = nrmf.capture(calls)
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / R)
    return statistics.median(ts)


for dt in (torch.float64, torch.float32):
    for lg in (12, 16, 18, 20, 22, 23, 24, 25, 26, 27, 28, 29, 30):
        x = torch.randn(1 << lg, dtype=dt, device="cuda")
        ms = t(x, 20 if lg >= 28 else 50)
        print(f"{str(dt):14s} n=2^{lg:2d}: {ms*1e3:9.1f} us  {x.numel()*x.element_size()/ms/1e6:8.1f} GB/s", flush=True)
        del x
