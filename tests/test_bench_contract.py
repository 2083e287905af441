"""The bench contract's reference arm runs on CPU (the oracle on host cores):
one JSON line with the keys the driver reads.  The GPU arm's line is checked
on the box by running bench.py itself."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    env = dict(os.environ)
    env.pop("RANK", None)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert not [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]



def test_gpus_beyond_the_visible_devices_fail_fast():
    """--gpus N without a torchrun environment re-execs under torch.distributed.run;
    with fewer than N visible GPUs it exits non-zero at once (never silently
    one GPU under an N-GPU label)."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode != 0
    assert "needs 2 GPUs" in p.stderr
    assert not [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode != 0 and "WORLD_SIZE=1" in p.stderr


@pytest.mark.gpu
def test_gpu_arm_reexec_under_torchrun():
    """The re-exec branch: bench.py launches itself under
    torch.distributed.run (forced with --launcher torchrun at --gpus 1 on this
    one-GPU box); the line's n_gpus equals --gpus and its result is the N = 1
    tree's bits (the oracle's value of the workload)."""
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--launcher", "torchrun",
                        "--steps", "3", "--warmup", "3", "--no-extras", "--e2e-steps", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["ranks_same_bits"] and d["same_bits_as_1gpu_tree"] is True
    assert d["result_hex"] == _c3_oracle_hex() and len(d["per_rank_ms"]) == 1


@pytest.mark.gpu
def test_gpu_arm_prints_one_contract_line():
    """bench.py's own arm on the GPU (short run): one JSON line carrying the
    contract keys, a roofline and cpu_baseline object, e2e with its copy
    bytes, clocks, launches, and a result bit-exact with the oracle."""
    env = dict(os.environ)
    env.pop("RANK", None)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-other", "--no-snrmf", "--e2e-steps", "1"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0 and d["gpu_launches"] >= 3
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == d["config"]["n"] * d["config"]["elem_bytes"] and e["same_bits"]
    assert d["accuracy"]["bit_exact_vs_oracle"]
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k


@pytest.mark.gpu
@pytest.mark.parametrize("p2p", ["0", "1"])
def test_gpu_arm_distributed_step_on_one_rank(p2p):
    """The N > 1 step (shard, tree kernel, NCCL allgather or the P2P
    exchange, rank tree; one CUDA graph) run on a 1-rank group under torchrun
    (NRMF_BENCH_DIST=1): the line is produced, the graph captured, e2e bits
    equal the device bits, and the result equals the single-GPU tree's."""
    env = dict(os.environ, NRMF_BENCH_DIST="1", NRMF_BENCH_P2P=p2p)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    port = str(29650 + int(p2p))
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", port, os.path.join(ROOT, "bench.py"),
                        "--gpus", "1", "--steps", "3", "--warmup", "3", "--no-extras", "--e2e-steps", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["rank_exchange"] == ("p2p" if p2p == "1" else "nccl_allgather")
    assert d["graph"] and d["e2e"]["same_bits"] and d["allgather_8B_us"] > 0
    assert d["result_hex"] == _c3_oracle_hex() and d["same_bits_as_1gpu_tree"] is True
    assert d["gpu_launches"] == d["steps"] * (1 if p2p == "1" else 2)


_C3_HEX = []


def _c3_oracle_hex():
    """The oracle's value of bench.py's C3 workload (n = 2^30 N(0,1), seed 1),
    big-endian hex as bench.py prints it (computed once, ~15 s on one core);
    it must equal the golden file bench.py reads (tools/make_golden_bench.py)."""
    if not _C3_HEX:
        import numpy as np

        import golden_values
        import nrmf_inputs as gen
        import oracle
        x = gen.normal(1, 1 << 30, 0, dtype=np.float64)
        _C3_HEX.append(np.asarray(oracle.nrmf(x), dtype=np.float64).tobytes()[::-1].hex())
        assert golden_values.hex_of("c3") == _C3_HEX[0]
    return _C3_HEX[0]
