"""Bitwise identity across 1/2/4/8 GPUs, through the real kernels (north star:
"bitwise identical across runs and GPU counts", and
P:1077-1084: contiguous chunks per worker, combined in a fixed order).

A G-rank run of nrmf_dist_[ds] is: every rank r runs the local step on its
canonical shard (nrmf_dist_local_[ds] -- the tree kernel over the rank's
aligned subtree), the G values are gathered in rank order (ncclAllGather),
and every rank evaluates the rank tree (nrmf_rank_combine_[ds]).  One GPU
runs every rank's local step in turn, the gathered vector is assembled on the
device, and the GPU rank tree combines it: the bits must equal nrmf_[ds] on
the whole array and the oracle (per rank, oracle.shard_norms; overall,
oracle.nrmf).  Only the transport -- one scalar per rank -- is not exercised
here (world-1 NCCL and P2P runs cover it, tests/test_gpu_p2p.py)."""
import numpy as np
import pytest
import torch

import nrmf_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
T = 4096
NP2T = {np.float64: torch.float64, np.float32: torch.float32}


@pytest.fixture(scope="module")
def nrmf():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2509_06220_b200 import _build
    _build.build()
    import paper_2509_06220_b200 as m
    m.lib()
    torch.cuda.set_device(0)
    return m


def bits(v, dt):
    return np.asarray(v, dtype=dt).tobytes()


def run_ranks(nrmf, xd, n, G, top="v1"):
    """Every rank's local step, the gathered vector, the GPU rank tree."""
    vals = torch.empty(G, dtype=xd.dtype, device=xd.device)
    for r in range(G):
        off, cnt = nrmf.shard(n, G, r)
        nrmf.dist_local(xd[off:off + cnt], n, G, r, out=vals[r], top=top)
    return vals, nrmf.rank_combine(vals, n, G, top=top)


CASES = [(4 * T * 8 + 5, np.float64), (1000 * T + 777, np.float64), (3 * T, np.float32),
         (2049 * T + 1, np.float32), (5, np.float64), (T * 17, np.float32)]


@pytest.mark.parametrize("top", ["v1", "cr"])
@pytest.mark.parametrize("n,dt", CASES)
@pytest.mark.parametrize("G", [1, 2, 4, 8, 16])
def test_ranks_combine_to_the_one_gpu_bits(nrmf, n, dt, G, top):
    x = gen.normal(n + G, n, dtype=dt)
    xd = torch.from_numpy(x).cuda()
    vals, out = run_ranks(nrmf, xd, n, G, top)
    one = nrmf.norm(xd, top=top)
    want = oracle.shard_norms(x, G, top=top)
    got = vals.cpu().numpy()
    for r, w in enumerate(want):           # ranks beyond P2 own nothing (+0)
        assert bits(got[r], dt) == bits(dt(0) if w is None else w, dt), (r, got[r], w)
    assert bits(out.cpu().numpy(), dt) == bits(one.cpu().numpy(), dt)
    assert bits(out.cpu().numpy(), dt) == bits(oracle.nrmf(x, top=top), dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_nan_shard(nrmf, dt, G):
    """A NaN in one rank's shard: the rank trees still agree with the
    one-GPU tree (Listing 2 ignores one NaN operand, R4)."""
    n = 64 * T + 9
    x = gen.sme(3, n, dtype=dt)
    x[n // G + 5] = np.nan
    xd = torch.from_numpy(x).cuda()
    _, out = run_ranks(nrmf, xd, n, G)
    assert bits(out.cpu().numpy(), dt) == bits(nrmf.norm(xd).cpu().numpy(), dt) == bits(oracle.nrmf(x), dt)


@pytest.mark.slow
@pytest.mark.parametrize("G", [2, 4, 8])
def test_c3_full_size_across_gpu_counts(nrmf, G):
    """C3 at its full size (n = 2^30 N(0,1), seed 1, bench.py's workload): every
    rank's shard (2^29 .. 2^27 elements: the persistent stream kernel with its
    CTA combine step) through the local step, then the rank tree: the bits of
    the 1-GPU call and of the oracle (golden file)."""
    import golden_values
    n = 1 << 30
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    gen.normal(1, n, 0, dtype=np.float64, out=xh.numpy())
    xd = xh.cuda()
    del xh
    _, out = run_ranks(nrmf, xd, n, G)
    one = nrmf.norm(xd)
    assert bits(out.cpu().numpy(), np.float64) == bits(one.cpu().numpy(), np.float64)
    assert out.cpu().numpy().tobytes()[::-1].hex() == golden_values.hex_of("c3")


def test_ranks_sequence_of_calls_is_reproducible(nrmf):
    """Runs are bitwise reproducible: 20 repetitions at G = 8, fresh workspaces each time."""
    n = 3000 * T + 123
    x = gen.normal(5, n, dtype=np.float64)
    xd = torch.from_numpy(x).cuda()
    ref = None
    for i in range(20):
        nrmf.clear_workspaces()
        _, out = run_ranks(nrmf, xd, n, 8)
        b = bits(out.cpu().numpy(), np.float64)
        ref = ref or b
        assert b == ref
    assert ref == bits(oracle.nrmf(x), np.float64)
