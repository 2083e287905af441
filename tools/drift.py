"""Dev tool: per-launch times of nrmf_d over many back-to-back launches, with
NVML clock / power / throttle reasons, to see sustained-load drift."""
import statistics
import sys
import time

import pynvml as nv
import torch

sys.path.insert(0, ".")
import paper_2509_06220_b200 as nrmf  # noqa: E402

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
dt = torch.float64 if (sys.argv[1] if len(sys.argv) > 1 else "d") == "d" else torch.float32
x = torch.randn(1 << 30, dtype=dt, device="cuda")
out = torch.empty((), dtype=dt, device="cuda")
for _ in range(3):
    nrmf.norm(x, out=out)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(300)]
t0 = time.time()
for a, b in ev:
    a.record(); nrmf.norm(x, out=out); b.record()
    if len(ev) and (ev.index((a, b)) % 25 == 0):
        pass
torch.cuda.synchronize()
ts = [a.elapsed_time(b) for a, b in ev]
for i in range(0, 300, 25):
    print(f"launch {i:3d}-{i+24:3d}: median {statistics.median(ts[i:i+25]):.4f} ms  min {min(ts[i:i+25]):.4f}")
print("clock now", nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), "MHz power", nv.nvmlDeviceGetPowerUsage(h) / 1000, "W",
      "reasons", hex(nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
# with gaps between launches
ts2 = []
for i in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); nrmf.norm(x, out=out); b.record(); torch.cuda.synchronize(); ts2.append(a.elapsed_time(b))
    time.sleep(0.05)
print(f"with 50 ms gaps: median {statistics.median(ts2):.4f} min {min(ts2):.4f}")
