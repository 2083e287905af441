"""Dev tool: device time of the C5 extreme-range inputs (n = 2^27 fp64, lit /
fin / fin2) for a libnrmf.so build, bits checked against the oracle."""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nrmf_inputs as gen  # noqa: E402
import oracle  # noqa: E402
import paper_2509_06220_b200 as nrmf  # noqa: E402

if len(sys.argv) > 1:
    nrmf.LIB_PATH = sys.argv[1]
n = 1 << 27
for var in ("lit", "fin", "fin2"):
    xh = gen.extreme(1, n, var)
    x = torch.from_numpy(xh).cuda()
    out = torch.empty((), dtype=torch.float64, device="cuda")
    g = nrmf.capture(lambda: nrmf.norm(x, out=out))
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = np.float64(out.item()).tobytes() == np.float64(oracle.nrmf(xh)).tobytes()
    print(f"C5 {var}: {statistics.median(ts):.4f} ms  bit_exact={ok}", flush=True)
