"""The rank level through peer memory (nrmf_p2p.cuh).

With one GPU per call, ranks that wait on one another cannot be separate
launches (B200_PROFILING: no guarantee they are co-resident).  So the exchange
protocol -- P2P value stores, release flags, parity halves per epoch, the rank
tree -- is run with `world` ranks emulated as the CTAs of ONE cooperative
launch, each rank with its own buffer; every rank's result must equal the
oracle's rank tree bit for bit, over several epochs without resetting the
buffers.  The full dist_p2p call (the tree kernel with the exchange at its
root, IPC setup) is run on a 1-rank group against the oracle."""
import os

import numpy as np
import pytest
import torch

import nrmf_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
T = 4096


@pytest.fixture(scope="module")
def nrmf():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2509_06220_b200 import _build
    _build.build()
    import paper_2509_06220_b200 as m
    m.lib()
    torch.cuda.set_device(0)
    return m


def _bufs(nrmf, world):
    import ctypes
    L = nrmf.lib()
    ptrs = []
    for _ in range(world):
        p = ctypes.c_void_p()
        assert L.nrmf_p2p_alloc(ctypes.byref(p)) == 0
        ptrs.append(p.value)
    return ptrs, torch.tensor(ptrs, dtype=torch.int64, device="cuda")


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("world", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("top", ["v1", "cr"])
def test_exchange_protocol_emulated_ranks(nrmf, dt, world, top):
    ptrs, bufs = _bufs(nrmf, world)
    try:
        for epoch in range(1, 6):                     # call counter in the buffers, halves reused
            vals = np.abs(gen.normal(100 * world + epoch, world, dtype=dt)) * dt(2.0 ** (epoch * 7 - 20))
            if epoch == 4:
                vals[world // 2] = 0                   # a rank that owns only padding
            got = nrmf._debug_p2p_emulate(torch.from_numpy(vals).cuda(), bufs, top=top).cpu().numpy()
            exp = np.asarray(oracle.combine(vals, top=top), dtype=dt)
            for r in range(world):
                assert got[r].tobytes() == exp.tobytes(), (epoch, r)
    finally:
        for p in ptrs:
            nrmf.lib().nrmf_p2p_free(p)


@pytest.mark.parametrize("grid", [0, 1, 2, 5])
def test_dist_p2p_world1(nrmf, grid):
    """dist_p2p on a 1-rank group (IPC handle, peer array, the exchange fused
    into the tree kernel's root writer with the rank's own buffer) equals the
    oracle, over calls.  Every place the root can be written: the split
    kernel's climb (grid 0, small n) and its single group (n <= T), the
    persistent kernel's single group (forced grid 1, n = 8T), its climbs and
    CTA combine step (forced grids 1/2/5, and grid 0 at 2^26 + 5), and a rank
    without data (n = 0: +0 through the separate exchange kernel)."""
    import torch.distributed as td
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29547")
    created = False
    if not td.is_initialized():
        td.init_process_group("gloo", rank=0, world_size=1)
        created = True
    pg = None
    nrmf._debug_set_grid(grid)
    try:
        pg = nrmf.P2PGroup()
        sizes = [0, 1, 4097, 8 * T, 300 * T + 5, (1 << 22) + 3] + ([(1 << 26) + 5] if grid == 0 else [])
        for dt in (np.float64, np.float32):
            for n in sizes:
                x = gen.normal(n + 1, n, dtype=dt)
                for _ in range(2):
                    r = nrmf.dist_p2p(torch.from_numpy(x).cuda(), n, pg).cpu().numpy()
                    assert np.asarray(r, dtype=dt).tobytes() == np.asarray(oracle.nrmf(x), dtype=dt).tobytes(), n
                rc = nrmf.dist_p2p(torch.from_numpy(x).cuda(), n, pg, top="cr").cpu().numpy()
                assert np.asarray(rc, dtype=dt).tobytes() == np.asarray(oracle.nrmf(x, top="cr"),
                                                                         dtype=dt).tobytes(), n
        assert int(pg.err.item()) == 0
    finally:
        nrmf._debug_set_grid(0)
        if pg is not None:
            pg.close()
        if created:
            td.destroy_process_group()


def test_dist_p2p_graph_replay_world1(nrmf):
    """The exchange keeps its call counter in device memory: a captured
    dist_p2p call is one kernel node and replays correctly (here on a 1-rank
    group)."""
    import torch.distributed as td
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29549")
    created = False
    if not td.is_initialized():
        td.init_process_group("gloo", rank=0, world_size=1)
        created = True
    pg = None
    try:
        pg = nrmf.P2PGroup()
        n = 100 * T + 3
        xh = gen.normal(5, n, dtype=np.float64)
        x = torch.from_numpy(xh).cuda()
        out = torch.empty((), dtype=torch.float64, device="cuda")
        g = torch.cuda.CUDAGraph(keep_graph=True)
        nrmf.capture(lambda: nrmf.dist_p2p(x, n, pg, out=out), graph=g)
        # the whole distributed step is ONE kernel: no counter memset
        # (NRMF_WS_CLEAN in capture), the exchange inside the tree kernel
        from test_gpu_graph import _graph_node_types
        assert _graph_node_types(g) == ["cudaGraphNodeTypeKernel"]
        g.instantiate()
        for _ in range(4):
            g.replay()
            torch.cuda.synchronize()
            assert out.cpu().numpy().tobytes() == np.float64(oracle.nrmf(xh)).tobytes()
        assert int(pg.err.item()) == 0
    finally:
        if pg is not None:
            pg.close()
        if created:
            td.destroy_process_group()
