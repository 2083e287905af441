"""Dev tool: energy per call (NVML total-energy counter) and sustained time of
nrmf_d at n=2^30 for libnrmf.so variants, each after a cool-down, 300
back-to-back launches.  Under the board power cap the kernel's energy per node
decides the sustained clock."""
import statistics
import sys
import time

import pynvml as nv
import torch

sys.path.insert(0, "tools")
from bench_variants import load  # noqa: E402

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
n = 1 << 30
x = torch.randn(n, dtype=torch.float64, device="cuda")
for path in sys.argv[1:]:
    L = load(path)
    ws = torch.zeros(L.nrmf_workspace_bytes(n, 8), dtype=torch.uint8, device="cuda")
    out = torch.empty((), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    call = lambda: L.nrmf_d(n, x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    time.sleep(5)                                   # cool down
    e0 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(300)]
    for a, b in evs:
        a.record(); call(); b.record()
    torch.cuda.synchronize()
    e1 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
    ts = [a.elapsed_time(b) for a, b in evs]
    print(f"{path}: first50 {statistics.median(ts[:50]):.4f} ms  last100 {statistics.median(ts[-100:]):.4f} ms  "
          f"energy {(e1 - e0) / 300:.1f} mJ/call  avg power {(e1 - e0) / sum(ts):.0f} W", flush=True)
