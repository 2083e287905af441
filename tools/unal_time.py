"""Dev tool: time the unaligned-vector paths against the aligned one.

    python tools/unal_time.py [--lg 28] [--reps 30]

For fp64 and fp32 at n = 2^lg: the 16-byte aligned base, a base 1 element off
on the stream kernel (StreamLoader UNAL), and the same base on the
element-load kernel (hook off).  Median of per-call CUDA-event times, all
results checked for equal bits."""
import argparse
import statistics

import torch

import paper_2509_06220_b200 as nrmf


def timed(x, reps):
    out = torch.empty((), dtype=x.dtype, device="cuda")
    for _ in range(3):
        nrmf.norm(x, out=out)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nrmf.norm(x, out=out)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out.item()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lg", type=int, default=28)
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    n = 1 << a.lg
    for dt in (torch.float64, torch.float32):
        g = torch.Generator(device="cuda").manual_seed(1)
        buf = torch.randn(n + 8, dtype=dt, device="cuda", generator=g)
        al, un = buf[:n], buf[1:n + 1]
        ref_u = nrmf.norm(un.clone()).item()
        t_a, r_a = timed(al, a.reps)
        t_u, r_u = timed(un, a.reps)
        nrmf._debug_set_unal_stream(False)
        t_e, r_e = timed(un, a.reps)
        nrmf._debug_set_unal_stream(True)
        gbs = lambda t: n * buf.element_size() / (t * 1e-3) / 1e9
        print(f"{dt} n=2^{a.lg}: aligned {t_a:.4f} ms ({gbs(t_a):.0f} GB/s) | unaligned stream {t_u:.4f} ms "
              f"({gbs(t_u):.0f} GB/s, {t_a / t_u:.3f} x aligned) | unaligned element loads {t_e:.4f} ms "
              f"({gbs(t_e):.0f} GB/s) | same bits {r_u == ref_u == r_e}")


if __name__ == "__main__":
    main()
