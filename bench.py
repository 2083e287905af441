#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the B200 xNRMF path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c2|c4|c1] [--no-extras]

Default workload (BASELINE.json metric "DNRMF/SNRMF GB/s and % of binding
roofline at n=2^30; max error (ulp) vs exact", config C3): DNRMF of one fp64
array of n = 2^30 N(0,1) elements (8 GiB, host Box-Muller, seed 1), sharded
contiguously over N GPUs (nrmf_dist_d; nrmf_d at N=1).  One step = one full
xNRMF evaluation of the whole array (all tree levels: loads, lane trees,
cross-lane, group, grid and rank combine).  Inputs (8 GiB, 1 GiB per GPU at
N=8) are larger than the 126 MB L2, so no L2 flush is needed.  Timed with
CUDA events on the launching stream, max over ranks.

Rank 0 prints ONE JSON line.  Extras on the line: roofline (dominant kernel,
HBM bytes vs MEASURED_PEAKS.json), cpu_baseline (the C oracle on one host
core, full workload), e2e (host-resident input through nrmf.norm / the
nrmf_host_d C-ABI call, H2D inside the timed region), accuracy (relerr and
ulp vs the exact norm, bit-equality with the oracle), the SNRMF n=2^30 point
the metric also names, clocks sampled with NVML during the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DNRMF/SNRMF GB/s and % of binding roofline at n=2^30; max error (ulp) vs exact"
N_C3 = 1 << 30


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int, period: float = 0.01):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv = None
            self.err = str(e)
            return self
        try:   # board energy counter (mJ): average power over the timed region
            self.e0 = self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h)
        except Exception:  # noqa: BLE001
            self.e0 = None
        self.t0 = time.perf_counter()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self.t1 = time.perf_counter()
        self.e1 = None
        if getattr(self, "e0", None) is not None:
            try:
                self.e1 = self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h)
            except Exception:  # noqa: BLE001
                self.e1 = None
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        d = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
             "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if getattr(self, "e1", None) is not None and self.t1 > self.t0:
            d["board_power_w"] = round((self.e1 - self.e0) * 1e-3 / (self.t1 - self.t0), 1)
        return d


# ------------------------------------------------------------------ helpers
def ulp_distance(a: float, b: float, dt) -> int | None:
    if not (math.isfinite(a) and math.isfinite(b)):
        return None if a != b else 0
    ia = np.asarray(a, dtype=dt).view(np.int64 if dt == np.float64 else np.int32).item()
    ib = np.asarray(b, dtype=dt).view(np.int64 if dt == np.float64 else np.int32).item()
    return abs(ia - ib)


def make_input(config: str, n: int, off: int, dt):
    import nrmf_inputs as gen
    if config in ("c3",):
        return gen.normal(1, n, off, dtype=dt)
    if config == "c2":
        return gen.sme(1, n, off, dtype=dt)
    if config == "c1":
        return gen.uniform_pm1(1, n, off, dtype=dt)
    raise ValueError(config)


def _nvtx(name):
    """NVTX range around a bench phase (visible in nsys / ncu --nvtx; host-side
    push/pop outside the event-timed regions, no cost to the device times)."""
    def deco(fn):
        def wrapped(*a, **k):
            import torch
            try:
                torch.cuda.nvtx.range_push(name)
                pushed = True
            except Exception:  # no NVTX in this build of torch: time without the range
                pushed = False
            try:
                return fn(*a, **k)
            finally:
                if pushed:
                    torch.cuda.nvtx.range_pop()
        wrapped.__name__, wrapped.__doc__ = fn.__name__, fn.__doc__
        return wrapped
    return deco


@_nvtx("nrmf.bench.burst")
def burst_point(step, stream, total_bytes, hbm_peak, local, flush=None):
    import torch
    ts = []
    with ClockSampler(local) as clk:
        for _ in range(10):
            if flush is not None:
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    gbs = total_bytes / (ms * 1e-3) / 1e9
    clocks = clk.summary()
    clocks.pop("board_power_w", None)  # NVML's power average lags; meaningless over ~20 ms
    return {"ms_per_step": round(ms, 4), "min_ms": round(min(ts), 4), "steps": 10, "value": round(gbs, 2),
            "unit": "GB/s", "frac_hbm": round(gbs / hbm_peak, 4), "clocks": clocks,
            "note": "after ~15 s idle (CPU oracle); context only, not the line's value"}


@_nvtx("nrmf.bench.sustained")
def sustained_point(step, stream, total_bytes, hbm_peak, local, flush=None, launches=300):
    """Context: the step launched `launches` times back to back
    right after the burst point, each launch timed by its own events; the
    median of the last 100 is the power-capped steady state.  Energy per call
    from the NVML total-energy counter over all launches."""
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(launches)]
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for e0, e1 in evs:
            if flush is not None:
                flush.zero_()
            e0.record(stream)
            step()
            e1.record(stream)
        torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for a, b in evs]
    last = statistics.median(ts[-100:])
    first = statistics.median(ts[:50])
    clocks = clk.summary()
    d = {"launches": launches, "first50_median_ms": round(first, 4), "last100_median_ms": round(last, 4),
         "value": round(total_bytes / (last * 1e-3) / 1e9, 2), "unit": "GB/s",
         "frac_hbm": round(total_bytes / (last * 1e-3) / 1e9 / hbm_peak, 4), "clocks": clocks}
    if getattr(clk, "e1", None) is not None and flush is None:
        d["energy_j_per_call"] = round((clk.e1 - clk.e0) * 1e-3 / launches, 3)
        d["avg_power_w"] = round((clk.e1 - clk.e0) * 1e-3 / (sum(ts) * 1e-3), 1)
    return d


def golden_hex(config):
    """The oracle's value of this workload (tests/golden/oracle_bench_values.txt)."""
    p = os.path.join(ROOT, "tests", "golden", "oracle_bench_values.txt")
    try:
        with open(p) as f:
            for ln in f:
                parts = ln.split()
                if len(parts) == 5 and parts[0] == config:
                    return parts[3]
    except OSError:
        pass
    return None


def seq_us(body, stream, k=200):
    """Device time per iteration of k back-to-back calls of body() (each may
    include an L2 flush), one event pair around the whole sequence: used by
    difference, seq(flush; call) - seq(flush), for small calls."""
    import torch
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        body()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / k


@_nvtx("nrmf.bench.timed_steps")
def time_loop(fn, steps: int, stream, flush=None):
    import torch
    if flush is not None:
        # inputs that fit in L2: overwrite a buffer larger than L2 before every
        # step, outside the events; the steps' device times are summed
        # (no host sync inside the loop: each step is already queued behind
        # its flush when its start event fires, so no launch gap is timed)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        for e0, e1 in ev:
            flush.zero_()
            e0.record(stream)
            fn()
            e1.record(stream)
        torch.cuda.synchronize()
        return sum(e0.elapsed_time(e1) for e0, e1 in ev) / steps
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps  # ms per step


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The oracle (plain C, one host core) on the same workload: each step is a
    bounded contiguous sample of 2^26 elements of the C3 array (~1 s of CPU;
    the offset varies per step), so the run ends within a minute or two."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    dt = np.float64 if args.config in ("c3", "c1", "c4") else np.float32
    sample = 1 << 26
    esz = np.dtype(dt).itemsize
    ts = []
    with one_core() as core:
        for s in range(args.warmup + args.steps):
            x = make_input(args.config, sample, (s * sample) % N_C3, dt)
            t0 = time.perf_counter()
            oracle.nrmf(x)
            t1 = time.perf_counter()
            if s >= args.warmup:
                ts.append(t1 - t0)
    ms = 1e3 * sum(ts) / len(ts)
    gbs = sample * esz / (ms * 1e-3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if dt == np.float64 else "f32", "data": "synthetic",
        "config": {"workload": cfg_name(args.config), "n": N_C3, "sample_per_step": sample},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"2^26 contiguous elements of the {args.config.upper()} array per step",
                         "core": core, "nproc": os.cpu_count()},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class one_core:
    """Pin this process to one host core while the oracle is timed (SURVEY
    §8(d): single-threaded oracle on one core); restores the old mask."""

    def __enter__(self):
        self.old = None
        try:
            self.old = os.sched_getaffinity(0)
            core = max(self.old)
            os.sched_setaffinity(0, {core})
            return core
        except (AttributeError, OSError):
            return None

    def __exit__(self, *a):
        if self.old is not None:
            try:
                os.sched_setaffinity(0, self.old)
            except OSError:
                pass


def cfg_name(c):
    return {"c3": "C3 DNRMF fp64 n=2^30 N(0,1) (nrmf_d / nrmf_dist_d)",
            "c2": "SNRMF fp32 n=2^30 s*m*2^e e in [-20,20] (nrmf_s)",
            "c1": "C1 DNRMF fp64 n=2^20 U[-1,1)"}.get(c, c)


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as td

    import paper_2509_06220_b200 as nrmf
    from paper_2509_06220_b200 import _build
    _build.build()
    nrmf.lib()

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    # the distributed step (shard, tree kernel, NCCL allgather, rank tree) for
    # N > 1; NRMF_BENCH_DIST=1 runs it on a 1-rank group (under torchrun) to
    # exercise that path on one GPU
    dist = world > 1 or os.environ.get("NRMF_BENCH_DIST", "0") == "1"
    local = env_int("LOCAL_RANK", 0)
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if dist:
        td.init_process_group("nccl", device_id=device)

    config = args.config
    dt = np.float64 if config in ("c3", "c1") else np.float32
    tdt = torch.float64 if dt == np.float64 else torch.float32
    esz = np.dtype(dt).itemsize
    n = N_C3 if config in ("c3", "c2") else (1 << 20)
    off, cnt = nrmf.shard(n, world, rank) if dist else (0, n)

    t0 = time.time()
    x_host = torch.empty(cnt, dtype=tdt).pin_memory()
    import nrmf_inputs as gen
    xh = x_host.numpy()
    if config == "c3":
        gen.normal(1, cnt, off, dtype=dt, out=xh)
    elif config == "c2":
        gen.sme(1, cnt, off, dtype=dt, out=xh)
    else:
        gen.uniform_pm1(1, cnt, off, dtype=dt, out=xh)
    x = x_host.to(device)
    torch.cuda.synchronize()
    t_gen = time.time() - t0

    stream = torch.cuda.current_stream(device)
    out = torch.empty((), dtype=tdt, device=device)
    comm = nrmf.comm_for(None) if dist else None

    # rank exchange of the N > 1 step: the peer-memory exchange fused into the
    # tree kernel (nrmf_dist_p2p_d; default) or NCCL
    # (NRMF_BENCH_P2P=0: ncclAllGather of one scalar + the rank-tree kernel);
    # if the peer buffers cannot be mapped, NCCL, and the line says so
    p2p = dist and os.environ.get("NRMF_BENCH_P2P", "1") == "1"
    pgroup, p2p_note = None, None
    if p2p:
        try:
            pgroup = nrmf.P2PGroup()      # raises on every rank if any rank cannot map a peer
        except Exception as e:  # noqa: BLE001
            p2p, p2p_note = False, f"P2P setup failed ({e}); NCCL exchange"
    if dist:
        # one CUDA graph per step: counter memset + tile-tree kernel with the
        # peer exchange at its root (p2p), or counter memset, tile-tree kernel,
        # ncclAllGather of one scalar and the rank-tree kernel
        if p2p:
            call = lambda: nrmf.dist_p2p(x, n, pgroup, out=out)  # noqa: E731
            launches_per_step = 1  # the tile-tree kernel (exchange and rank tree inside)
        else:
            call = lambda: nrmf.dist(x, n, comm=comm, out=out)  # noqa: E731
            launches_per_step = 2  # tile-tree kernel + rank-tree kernel (the NCCL allgather is NCCL's)
    else:
        # the step (counter memset + tree kernel) replayed from a CUDA graph:
        # device time without the Python/ctypes launch overhead (matters at C1)
        call = lambda: nrmf.norm(x, out=out)  # noqa: E731
        launches_per_step = 1
    use_graph = os.environ.get("NRMF_BENCH_GRAPH", "1") == "1"
    graph = None
    if use_graph:
        try:
            graph = nrmf.capture(call)
        except Exception as e:  # noqa: BLE001 -- fall back to direct launches, say so in the line
            print(f"bench: CUDA graph capture failed ({e}); timing direct launches", file=sys.stderr)
            graph = None

    def step():
        if graph is not None:
            graph.replay()
        else:
            call()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist and p2p:
        # the fused peer exchange has only ever run on a 1-rank group: check it
        # on this box before timing it -- no rank timed out and every rank holds
        # the same bits -- and otherwise time the NCCL exchange and say so
        hx = torch.tensor([np.asarray(out.cpu().item(), dtype=dt).view(np.int64 if esz == 8 else np.int32).item(),
                           int(pgroup.err.item())], dtype=torch.int64, device=device)
        allh = torch.zeros(2 * world, dtype=torch.int64, device=device)
        td.all_gather_into_tensor(allh, hx)
        vals = allh.view(world, 2).tolist()
        if any(e != 0 for _, e in vals) or len({v for v, _ in vals}) != 1:
            p2p, p2p_note = False, f"P2P exchange check failed on this box ({vals}); NCCL exchange"
            call = lambda: nrmf.dist(x, n, comm=comm, out=out)  # noqa: E731
            launches_per_step = 2
            graph = nrmf.capture(call) if use_graph else None
            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize()
    if dist:
        td.barrier()
    # inputs below 4x the 126 MB L2 (C1: 8 MiB): flush L2 before every timed step
    small = cnt * esz < 4 * 126 * 2**20
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=device) if small else None
    with ClockSampler(local) as clk:
        ms = time_loop(step, args.steps, stream, flush)
    by_diff = None
    if small:
        # context for small calls (other_configs C1 note): the same
        # step by difference of two long flushed sequences, one event pair each
        if dist:
            td.barrier()
        d = []
        for _ in range(3):
            t_f = seq_us(flush.zero_, stream)
            d.append(seq_us(lambda: (flush.zero_(), step()), stream) - t_f)
        by_diff = float(np.median(d))
        if dist:
            tt = torch.tensor([by_diff], dtype=torch.float64, device=device)
            allt = torch.zeros(world, dtype=torch.float64, device=device)
            td.all_gather_into_tensor(allt, tt)
            by_diff = max(allt.tolist())
    per_rank_ms = [ms]
    if dist:
        tt = torch.tensor([ms], dtype=torch.float64, device=device)
        allt = torch.zeros(world, dtype=torch.float64, device=device)
        td.all_gather_into_tensor(allt, tt)
        per_rank_ms = [round(v, 4) for v in allt.tolist()]
        ms = max(allt.tolist())
        td.barrier()
    result = out.cpu().item()
    result_hex = np.asarray(result, dtype=dt).tobytes()[::-1].hex()
    if dist:
        # every rank must hold the same bits
        hx = torch.tensor([int(result_hex, 16)], dtype=torch.int64, device=device)
        allh = torch.zeros(world, dtype=torch.int64, device=device)
        td.all_gather_into_tensor(allh, hx)
        ranks_agree = len(set(allh.tolist())) == 1
    else:
        ranks_agree = True

    # dominant kernel alone (the local tile-tree kernel), same stream, same data;
    # and the 8-byte allgather alone (torch's NCCL, same ranks)
    allgather_us = None
    if dist:
        kern_ms = time_loop(lambda: nrmf.norm(x, out=out), args.steps, stream)
        one = torch.zeros(1, dtype=tdt, device=device)
        allv = torch.zeros(world, dtype=tdt, device=device)
        for _ in range(5):
            td.all_gather_into_tensor(allv, one)
        td.barrier()
        ag = time_loop(lambda: td.all_gather_into_tensor(allv, one), 100, stream)
        tt = torch.tensor([ag], dtype=torch.float64, device=device)
        td.all_reduce(tt, op=td.ReduceOp.MAX)
        allgather_us = round(tt.item() * 1e3, 2)
    else:
        kern_ms = ms
    total_bytes = n * esz
    gbs = total_bytes / (ms * 1e-3) / 1e9

    peaks, peak_src = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    kern_gbs = cnt * esz / (kern_ms * 1e-3) / 1e9
    clocks = clk.summary()

    f_ghz = (clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)) / 1000.0
    line = {
        "metric": METRIC, "value": round(gbs, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if dt == np.float64 else "f32",
        "data": "synthetic",
        "config": {"workload": cfg_name(config), "n": n, "global_batch": n, "elem_bytes": esz,
                   "parallelism": f"shard{world}",
                   "l2": ("L2 flushed before every timed step (256 MiB write, untimed)" if small
                          else "input > 126 MB L2 (no flush needed)"),
                   "tree_version": nrmf.tree_version(), "seed": 1},
        "gpu_launches": launches_per_step * args.steps,
        "us_per_step_by_difference": None if by_diff is None else round(by_diff, 2),
        "graph": graph is not None,
        "rank_exchange": ("p2p" if p2p else "nccl_allgather") if dist else None,
        "clocks": clocks,
        "elements_per_s": round(n / (ms * 1e-3), 1),
        "roofline": {"bound": "hbm", "achieved": round(kern_gbs, 2), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(kern_gbs / hbm_peak, 4), "traffic": None,
                     "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs (copy)",
                     "kernel": "nrmf_tree_kernel<%s,TMA=1>" % ("double" if esz == 8 else "float"),
                     "algorithmic_bytes_per_launch": cnt * esz},
        "roofline_compute": compute_roofline(esz, cnt, kern_ms, f_ghz, hbm_peak),
    }
    if clocks.get("board_power_w"):
        # the FP64 kernel runs at the 1 kW board limit when sustained: its energy
        # per step, not the clock it starts at, decides the sustained rate
        line["energy_j_per_step"] = round(clocks["board_power_w"] * ms * 1e-3, 3)
        line["energy_note"] = ("NVML total-energy counter over the timed region (~0.2 s at the default "
                               "steps): coarse, +-15 %; tools/energy.py measures over 300 launches")
    if allgather_us is not None:
        line["allgather_8B_us"] = allgather_us
    if p2p_note:
        line["rank_exchange_note"] = p2p_note
    tr = load_traffic(esz)
    if tr is not None:
        line["roofline"]["traffic"] = tr
    line["per_rank_ms"] = per_rank_ms
    line["result_hex"] = result_hex
    line["ranks_same_bits"] = ranks_agree
    # the N = 1 tree's bits: the oracle's value of this workload (golden file
    # written by tools/make_golden_bench.py from oracle/ only)
    want = golden_hex(config)
    line["same_bits_as_1gpu_tree"] = (result_hex == want) if want is not None else None

    # ---------------- e2e: host-resident input through the public API
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    if not dist:
        host_out = torch.empty((), dtype=tdt).pin_memory()

        def e2e_step():
            nrmf.norm(x_host, out=host_out)          # nrmf_host_d: H2D ring + kernels + D2H
        e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        e2e_ok = host_out.item() == result or (math.isnan(result) and math.isnan(host_out.item()))
    else:
        xdev = torch.empty_like(x)

        def e2e_step():
            xdev.copy_(x_host, non_blocking=True)
            if p2p:
                nrmf.dist_p2p(xdev, n, pgroup, out=out)
            else:
                nrmf.dist(xdev, n, comm=comm, out=out)
            return out.cpu()
        e2e_step()
        td.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=device)
        td.all_reduce(tt, op=td.ReduceOp.MAX)
        e2e_ms = tt.item()
        v = out.cpu().item()
        e2e_ok = v == result or (math.isnan(result) and math.isnan(v))
    line["e2e"] = {"value": round(total_bytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                   "h2d_bytes_per_step": total_bytes, "d2h_bytes_per_step": esz,
                   "ms_per_step": round(e2e_ms, 3), "steps": e2e_steps, "same_bits": bool(e2e_ok),
                   "api": "nrmf.norm(pinned host tensor) -> nrmf_host_d" if not dist else
                          ("pinned H2D copy + nrmf.dist_p2p -> nrmf_dist_p2p_d" if p2p else
                           "pinned H2D copy + nrmf.dist -> nrmf_dist_d")}

    # ---------------- extras (rank 0, N=1): accuracy, oracle CPU baseline, SNRMF point
    if rank == 0 and world == 1 and not args.no_extras:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        ex = float(oracle.exact(xh))
        t_exact = time.perf_counter() - t0
        acc = {"relerr_eps": oracle.relerr(result, ex, dt), "ulp": ulp_distance(result, ex, dt),
               "exact_hex": np.asarray(ex, dtype=dt).tobytes()[::-1].hex(),
               "bound_thm3_eps": round(oracle.ub_relerr_H(12 + int(math.log2(max(1, n // 4096))), dt), 3)}
        with one_core() as core:
            t0 = time.perf_counter()
            o = oracle.nrmf(xh)
            t_or = time.perf_counter() - t0
        acc["bit_exact_vs_oracle"] = bool(np.asarray(o, dtype=dt).tobytes() == np.asarray(result, dtype=dt).tobytes())
        line["accuracy"] = acc
        line["cpu_baseline"] = {"value": round(total_bytes / t_or / 1e9, 4), "unit": "GB/s", "cores": 1,
                                "kind": "oracle", "seconds": round(t_or, 3),
                                "sample": f"full workload ({n} elements), single-threaded C oracle",
                                "cpu": cpu_model(), "core": core, "nproc": os.cpu_count()}
        line["timing_s"] = {"gen": round(t_gen, 2), "exact": round(t_exact, 2), "oracle": round(t_or, 2)}
        # context: the same step right after the GPU idled through the CPU
        # oracle (not power-capped yet), 10 steps timed one by one; the line's
        # value stays the sustained K-step number above
        line["burst"] = burst_point(step, stream, total_bytes, hbm_peak, local, flush)
        line["sustained"] = sustained_point(step, stream, total_bytes, hbm_peak, local, flush)
        line["context_sumsq"] = sumsq_context(x, ex, dt, ms, args, stream)
        if config == "c3" and not args.no_snrmf:
            line["snrmf"] = snrmf_point(nrmf, device, stream, args, hbm_peak)
        if config == "c3" and not args.no_other:
            del x
            torch.cuda.empty_cache()
            line["other_configs"] = other_configs(nrmf, device, stream, hbm_peak)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        if pgroup is not None:
            pgroup.close()
        comm.close()
        td.destroy_process_group()
    return 0


# Compute term of the roofline, from the
# instruction counts the shipped kernel EXECUTES per warp-node (ncu on this
# build, profiles/instr_per_node.json): the FP64 pipe takes 2 cycles per warp
# instruction per SM sub-partition (16 lanes/clk), the issue stage 1; 148 SMs
# x 4 sub-partitions, at the SM clock sampled during the run.  The binding
# term is the larger of these floors and the HBM time.
N_SM = 148


def load_instr(esz):
    p = os.path.join(ROOT, "profiles", "instr_per_node.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f).get("fp64" if esz == 8 else "fp32")


def compute_roofline(esz, n, ms, f_ghz, hbm_peak):
    t = ms * 1e-3
    warp_nodes = max(n - 1, 1) / 32
    t_hbm = n * esz / (hbm_peak * 1e9)
    c = load_instr(esz)
    if c is None:
        return {"bound": "alu", "unmeasured": "profiles/instr_per_node.json missing", "t_hbm_ms": round(t_hbm * 1e3, 4)}
    slots = N_SM * 4 * f_ghz * 1e9                      # warp-instruction issue slots per second
    t_issue = warp_nodes * c["warp_instr_per_warp_node"] / slots
    d = {"bound": "alu", "sm_ghz": f_ghz, "source": c.get("source"),
         "warp_instr_per_warp_node": c["warp_instr_per_warp_node"], "t_issue_ms": round(t_issue * 1e3, 4),
         "t_hbm_ms": round(t_hbm * 1e3, 4)}
    if esz == 8:
        t_fp64 = warp_nodes * c["fp64_instr_per_warp_node"] * 2 / slots
        d.update({"pipe": "FP64 (2 cycles per warp-instruction per SMSP)",
                  "fp64_instr_per_warp_node": c["fp64_instr_per_warp_node"],
                  "achieved": round(warp_nodes * 32 * c["fp64_instr_per_warp_node"] / t / 1e12, 4),
                  "peak": round(N_SM * 64 * f_ghz * 1e9 / 1e12, 4), "unit": "T FP64 lane-instr/s",
                  "t_fp64_ms": round(t_fp64 * 1e3, 4)})
        t_comp = max(t_fp64, t_issue)
    else:
        d.update({"pipe": "issue (1 warp-instruction per cycle per SMSP)",
                  "achieved": round(warp_nodes * c["warp_instr_per_warp_node"] / t / 1e12, 4),
                  "peak": round(slots / 1e12, 4), "unit": "T warp-instr/s"})
        t_comp = t_issue
    d["frac"] = round(t_comp / t, 4)
    d["t_compute_ms"] = round(t_comp * 1e3, 4)
    if c.get("rf_read_cycles_per_warp_node"):
        # a model, not a hardware peak: register-file read cycles per warp
        # instruction from the bank model of DESIGN.md §8, summed over the
        # executed instructions (ncu source page) -- it predicts the kernel's
        # time (the instructions do not overlap each other's operand reads)
        t_rf = warp_nodes * c["rf_read_cycles_per_warp_node"] / slots
        d["rf_model"] = {"read_cycles_per_warp_node": c["rf_read_cycles_per_warp_node"],
                         "t_ms": round(t_rf * 1e3, 4), "ratio_to_kernel": round(t_rf / t, 4)}
    d["binding"] = "hbm" if t_hbm >= t_comp else "alu"
    d["binding_frac"] = round(max(t_hbm, t_comp) / t, 4)
    return d


def load_traffic(esz):
    """dram bytes read+written per launch of the dominant kernel, from the
    committed ncu --set full capture of this build (profiles/)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get("fp64" if esz == 8 else "fp32")


def snrmf_point(nrmf, device, stream, args, hbm_peak):
    """The SNRMF half of the metric: fp32 n = 2^30, C2 recipe (s*m*2^e)."""
    import torch

    import nrmf_inputs as gen
    import oracle
    n = N_C3
    xh = torch.empty(n, dtype=torch.float32).pin_memory()
    gen.sme(1, n, 0, dtype=np.float32, out=xh.numpy())
    x = xh.to(device)
    out = torch.empty((), dtype=torch.float32, device=device)
    for _ in range(args.warmup):
        nrmf.norm(x, out=out)
    with ClockSampler(device.index) as clk:
        ms = time_loop(lambda: nrmf.norm(x, out=out), args.steps, stream)
    r = out.cpu().item()
    ex = float(oracle.exact(xh.numpy()))
    gbs = n * 4 / (ms * 1e-3) / 1e9
    ctx = sumsq_context(x, ex, np.float32, ms, args, stream)
    del x
    return {"workload": "SNRMF fp32 n=2^30 s*m*2^e, e in [-20,20] (C2 recipe)", "value": round(gbs, 2),
            "context_sumsq": ctx,
            "unit": "GB/s", "ms_per_step": round(ms, 4),
            "roofline": {"bound": "hbm", "achieved": round(gbs, 2), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(gbs / hbm_peak, 4), "traffic": load_traffic(4)},
            "roofline_compute": compute_roofline(4, n, ms, (clk.summary().get("sm_mhz") or 1965.0) / 1000.0,
                                                 hbm_peak),
            "relerr_eps": oracle.relerr(r, ex, np.float32), "ulp": ulp_distance(r, ex, np.float32),
            "clocks": clk.summary()}


def sumsq_context(x, ex, dt, ms_nrmf, args, stream):
    """Context only (the paper's e:speed analog, against a GPU
    library norm instead of L): torch.linalg.vector_norm -- the unscaled
    sqrt(sum of squares) reduction of torch's CUDA library on the same device
    data, timed the same way -- with its error against the exact norm.  NRMF's
    slowdown = its time / this time.  Not a baseline of the metric."""
    import torch
    r = torch.empty((), dtype=x.dtype, device=x.device)

    def step():
        torch.linalg.vector_norm(x, out=r)
    for _ in range(max(3, args.warmup)):
        step()
    ms = time_loop(step, min(args.steps, 50), stream)
    v = r.cpu().item()
    import oracle
    return {"impl": "torch.linalg.vector_norm (library, context)", "ms_per_step": round(ms, 4),
            "value": round(x.numel() * x.element_size() / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "nrmf_slowdown": round(ms_nrmf / ms, 3), "relerr_eps": oracle.relerr(v, ex, dt),
            "ulp": ulp_distance(v, ex, dt)}


@_nvtx("nrmf.bench.other_configs")
def other_configs(nrmf, device, stream, hbm_peak):
    """The other BASELINE configs, reported beside the metric (parity-test
    cases, not bench lines): C1 DNRMF n=2^20 (cold and L2-resident), C2 SNRMF
    n=2^28, C4 column norms 4096 x 65536, C5 extreme range n=2^27 (three
    readings, R9) and its complex view, and the unaligned-base path.  Inputs
    device-resident, each timed as graph replays after warm-up; bits checked
    against the oracle."""
    import torch

    import nrmf_inputs as gen
    import oracle

    def timed(fn, reps=20):
        g = nrmf.capture(fn)
        for _ in range(3):
            g.replay()
        return time_loop(g.replay, reps, stream)

    res = {}
    # C1: DNRMF n = 2^20 U[-1,1) (BASELINE configs[0]) -- 8 MiB fits in L2, so
    # L2 is flushed (256 MiB write, outside the events) before every step; the
    # captured call is one kernel node (NRMF_WS_CLEAN)
    n1 = 1 << 20
    x1h = gen.uniform_pm1(1, n1)
    x1 = torch.from_numpy(x1h).to(device)
    o1 = torch.empty((), dtype=torch.float64, device=device)
    g1 = nrmf.capture(lambda: nrmf.norm(x1, out=o1))
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=device)
    for _ in range(3):
        g1.replay()
    ms_cold = time_loop(g1.replay, 50, stream, flush)
    ms_warm = time_loop(g1.replay, 50, stream)

    # Per-call event pairs behind a 256 MiB flush carry a fixed overhead and
    # move in ~2.05 us steps on this pool (a 1 us globaltimer spin kernel
    # timed the same way reads 6.1 us; tools/timer_probe.py).  So also: the
    # call's cost inside a stream, by difference of two long sequences timed
    # with one event pair each, K x [flush; call] - K x [flush], and the same
    # for an empty kernel (the launch gap every kernel pays).
    tiny = torch.zeros(1, device=device)
    d_call, d_empty = [], []
    for _ in range(3):
        t_f = seq_us(flush.zero_, stream)
        d_call.append(seq_us(lambda: (flush.zero_(), g1.replay()), stream) - t_f)
        d_empty.append(seq_us(lambda: (flush.zero_(), tiny.add_(0)), stream) - t_f)
    floor = time_loop(lambda: tiny.add_(0), 50, stream, flush)
    res["C1"] = {"workload": "DNRMF fp64 n=2^20 U[-1,1)", "us_cold_l2_flushed": round(ms_cold * 1e3, 2),
                 "us_cold_by_difference": round(float(np.median(d_call)), 2),
                 "us_empty_kernel_by_difference": round(float(np.median(d_empty)), 2),
                 "us_empty_kernel_per_call_events": round(floor * 1e3, 2),
                 "note": "us_cold_l2_flushed: one event pair per call behind the flush (includes the event "
                         "floor us_empty_kernel_per_call_events); us_cold_by_difference: median over 3 of "
                         "(200 x [flush; call] - 200 x [flush]) / 200, one event pair per sequence",
                 "us_warm_l2_resident": round(ms_warm * 1e3, 2), "graph_nodes": 1,
                 "bit_exact_vs_oracle": bool(o1.cpu().numpy().tobytes() == np.float64(oracle.nrmf(x1h)).tobytes())}
    del tiny
    del x1, flush
    # the paper's unaligned case (aligned vs unaligned loads): a base
    # 8 bytes past a 16-byte boundary runs the stream kernel on shifted spans
    # (StreamLoader UNAL; same bits); the element-load kernel beside it
    nu = 1 << 28
    xuh = gen.normal(2, nu + 1)
    xu = torch.from_numpy(xuh).to(device)
    ou = torch.empty((), dtype=torch.float64, device=device)
    xa, xm = xu[:nu], xu[1:]
    msa = timed(lambda: nrmf.norm(xa, out=ou))
    try:
        nrmf._debug_set_unal_stream(False)
        mse = timed(lambda: nrmf.norm(xm, out=ou))
    finally:
        nrmf._debug_set_unal_stream(True)
    msu = timed(lambda: nrmf.norm(xm, out=ou))
    res["unaligned"] = {"workload": "DNRMF fp64 n=2^28 N(0,1), base 16-byte aligned vs 8 bytes off",
                        "ms_aligned": round(msa, 4), "ms_unaligned": round(msu, 4),
                        "unaligned_frac_of_aligned": round(msa / msu, 3),
                        "ms_unaligned_element_loads": round(mse, 4),
                        "GB/s_aligned": round(nu * 8 / (msa * 1e-3) / 1e9, 1),
                        "GB/s_unaligned": round(nu * 8 / (msu * 1e-3) / 1e9, 1),
                        "bit_exact_vs_oracle": bool(ou.cpu().numpy().tobytes() ==
                                                    np.float64(oracle.nrmf(xuh[1:])).tobytes())}
    del xu, xa, xm, xuh
    n2 = 1 << 28
    x2h = gen.sme(1, n2)
    x2 = torch.from_numpy(x2h).to(device)
    o2 = torch.empty((), dtype=torch.float32, device=device)
    ms = timed(lambda: nrmf.norm(x2, out=o2))
    res["C2"] = {"workload": "SNRMF fp32 n=2^28 s*m*2^e", "ms": round(ms, 4),
                 "GB/s": round(n2 * 4 / (ms * 1e-3) / 1e9, 1), "hbm_frac": round(n2 * 4 / (ms * 1e-3) / 1e9 / hbm_peak, 4),
                 "bit_exact_vs_oracle": bool(o2.cpu().numpy().tobytes() == np.float32(oracle.nrmf(x2h)).tobytes())}
    del x2, x2h
    r, c = 4096, 65536
    Ah = gen.colscaled_normal(1, r, c)
    A = torch.from_numpy(Ah).to(device).as_strided((r, c), (1, r))
    col = torch.empty(c, dtype=torch.float64, device=device)
    fr = torch.empty((), dtype=torch.float64, device=device)

    def colsc():
        cc, ff = nrmf.cols(A)
        col.copy_(cc)
        fr.copy_(ff)
    ms = timed(colsc)
    ecol, efr = oracle.cols(Ah, r, c, r)
    res["C4"] = {"workload": "nrmf_cols_d 4096 x 65536 N(0,1)*2^k_j", "ms": round(ms, 4),
                 "GB/s": round(r * c * 8 / (ms * 1e-3) / 1e9, 1),
                 "hbm_frac": round(r * c * 8 / (ms * 1e-3) / 1e9 / hbm_peak, 4),
                 "bit_exact_vs_oracle": bool(col.cpu().numpy().tobytes() == ecol.tobytes()
                                             and fr.cpu().numpy().tobytes() == np.float64(efr).tobytes())}
    del A, Ah
    n5 = 1 << 27
    for variant in ("lit", "fin", "fin2"):
        xh = gen.extreme(1, n5, variant)
        xd = torch.from_numpy(xh).to(device)
        o = torch.empty((), dtype=torch.float64, device=device)
        ms = timed(lambda: nrmf.norm(xd, out=o))
        oz = nrmf.norm_complex(xd.view(torch.complex128)).cpu().numpy()
        exp = np.float64(oracle.nrmf(xh))
        res["C5_" + variant] = {"workload": f"DNRMF fp64 n=2^27 extreme range ({variant})", "ms": round(ms, 4),
                                "GB/s": round(n5 * 8 / (ms * 1e-3) / 1e9, 1),
                                "bit_exact_vs_oracle": bool(o.cpu().numpy().tobytes() == exp.tobytes()),
                                "complex_view_same_bits": bool(oz.tobytes() == exp.tobytes())}
        del xd, xh
    return res


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} cpus)"
    except OSError:
        pass
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c3", "c2", "c1"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-snrmf", action="store_true")
    ap.add_argument("--no-other", action="store_true", help="skip the C2/C4/C5 report (other_configs)")
    ap.add_argument("--launcher", default="auto", choices=["auto", "torchrun"],
                    help="torchrun: re-exec under torch.distributed.run even for --gpus 1")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and (args.gpus > 1 or args.launcher == "torchrun"):
        return reexec_torchrun(args)
    world = env_int("WORLD_SIZE", 1)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    return run_ours(args)


def reexec_torchrun(args):
    """--gpus N without a torchrun environment: run this script under
    torch.distributed.run with N ranks (one per GPU), as the driver would."""
    import socket
    import subprocess
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        have = 0
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, {have} visible", file=sys.stderr)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    argv = [a for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
