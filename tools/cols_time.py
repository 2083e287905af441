"""Dev tool: time nrmf.cols on C4 (4096 x 65536 fp64) and other shapes."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_06220_b200 as nrmf  # noqa: E402

if len(sys.argv) > 1:            # time another build of the library
    nrmf.LIB_PATH = sys.argv[1]


def t(A, reps=20):
    for _ in range(3):
        nrmf.cols(A)
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); nrmf.cols(A); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for (r, c, ld, dt) in [(4096, 65536, 4096, torch.float64), (4096, 65536, 4160, torch.float64),
                       (8192, 32768, 8192, torch.float64), (8192, 32768, 8256, torch.float64),
                       (4096, 65536, 4160, torch.float32),
                       (4096, 65536, 4096, torch.float32), (4000, 65536, 4096, torch.float64), (4000, 65536, 4000, torch.float64), (3000, 65536, 3000, torch.float32),
                       (1000, 262144, 1000, torch.float64), (500, 524288, 500, torch.float64), (700, 393216, 700, torch.float64),
                       (1500, 174762, 1500, torch.float32),
                       (1024, 262144, 1024, torch.float64), (2000, 131072, 2000, torch.float32),
                       (300, 262144, 301, torch.float32), (100, 1 << 20, 100, torch.float64),
                       (100, 1 << 20, 101, torch.float64), (500, 524288, 501, torch.float64),
                       (4096, 32768, 4097, torch.float64), (4096, 32768, 4097, torch.float32)]:
    B = torch.randn(c, ld, dtype=dt, device="cuda")
    A = B.t()[:r]
    ms = t(A)
    print(f"cols r={r} c={c} ld={ld} {dt}: {ms:.4f} ms  {r * c * B.element_size() / ms / 1e6:.0f} GB/s", flush=True)
    del A, B
