"""Dev tool: a short nrmf_d / nrmf_s run of one libnrmf.so variant, for ncu.

    python tools/prof_one.py lib.so [d|s] [reps] [lg_n]"""
import sys

import torch

sys.path.insert(0, "tools")
from bench_variants import load  # noqa: E402

L = load(sys.argv[1])
dt = torch.float64 if (sys.argv[2] if len(sys.argv) > 2 else "d") == "d" else torch.float32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = 1 << (int(sys.argv[4]) if len(sys.argv) > 4 else 30)
x = torch.randn(n, dtype=dt, device="cuda")
ws = torch.zeros(L.nrmf_workspace_bytes(n, x.element_size()), dtype=torch.uint8, device="cuda")
out = torch.empty((), dtype=dt, device="cuda")
f = L.nrmf_d if dt == torch.float64 else L.nrmf_s
for _ in range(reps):
    assert f(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
print("ok", out.item())
