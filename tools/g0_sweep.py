"""Dev tool: device time per warp-group size (forced g0) and size, to fit the
group-size model of launch_tree."""
import ctypes
import random
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2509_06220_b200 as nrmf  # noqa: E402

L = nrmf.lib()
L.nrmf_debug_set_g0.argtypes = [ctypes.c_int]


def t(x, reps=20):
    out = torch.empty((), dtype=x.dtype, device="cuda")
    g = nrmf.capture(lambda: nrmf.norm(x, out=out))
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


# measurements in random order, each after a 1.5 s cool-down (the FP64 kernel
# is power-capped when hot), 3 repetitions -> minimum
random.seed(1)
G0S = (-1, 0, 1, 2, 3, 4)
DTS = (torch.float32, torch.float64) if "--both" in sys.argv else (torch.float32,)
LGS = (26, 28, 29, 30)
for a in sys.argv[1:]:
    if a.startswith("--lg="):
        LGS = tuple(int(v) for v in a[5:].split(","))
cases = [(dt, lg, g0) for dt in DTS for lg in LGS
         for g0 in G0S for _ in range(3)]
random.shuffle(cases)
xs = {}
res = {}
for dt, lg, g0 in cases:
    key = (dt, lg)
    if key not in xs:
        xs[key] = torch.randn(1 << lg, dtype=dt, device="cuda")
    L.nrmf_debug_set_g0(g0)
    time.sleep(1.5 if lg >= 28 else 0.3)
    v = t(xs[key], reps=5) * 1e3
    res.setdefault((dt, lg, g0), []).append(v)
L.nrmf_debug_set_g0(-1)
for dt in DTS:
    for lg in LGS:
        r = {g0: min(res[(dt, lg, g0)]) for g0 in G0S}
        print(f"{str(dt):14s} n=2^{lg}: auto {r[-1]:8.1f}  G1 {r[0]:8.1f}  G2 {r[1]:8.1f}  G4 {r[2]:8.1f}"
              f"  G8 {r[3]:8.1f}  G16 {r[4]:8.1f} us", flush=True)
