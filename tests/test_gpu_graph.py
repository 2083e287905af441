"""CUDA-graph capture of nrmf calls (kernel, allgather and rank
tree captured once, replayed with one launch): replays give the oracle's bits,
including after the input changes in place between replays."""
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


def bits(v, dt):
    return np.asarray(v, dtype=dt).tobytes()


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", [5, 3 * T + 7, 300 * T + 11])
def test_norm_graph_replay(nrmf, dt, n):
    x1 = gen.normal(7, n, dtype=dt)
    x2 = gen.sme(8, n, dtype=dt)
    x = torch.from_numpy(x1).cuda()
    out = torch.empty((), dtype=x.dtype, device="cuda")
    g = nrmf.capture(lambda: nrmf.norm(x, out=out))
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert bits(out.cpu().numpy(), dt) == bits(oracle.nrmf(x1), dt)
    x.copy_(torch.from_numpy(x2))          # same buffer, new contents
    g.replay()
    torch.cuda.synchronize()
    assert bits(out.cpu().numpy(), dt) == bits(oracle.nrmf(x2), dt)


def test_cols_graph_replay(nrmf):
    r, c = 4096 + 5, 37
    A = gen.normal(9, r * c, dtype=np.float64).reshape(c, r)    # column j = row j of this array
    At = torch.from_numpy(A).cuda().t()                           # column-major view
    col = torch.empty(c, dtype=torch.float64, device="cuda")
    fr = torch.empty((), dtype=torch.float64, device="cuda")

    def call():
        cc, ff = nrmf.cols(At)
        col.copy_(cc)
        fr.copy_(ff)
    g = nrmf.capture(call)
    g.replay()
    torch.cuda.synchronize()
    got = col.cpu().numpy()
    for j in range(c):
        assert bits(got[j], np.float64) == bits(oracle.nrmf(A[j]), np.float64)


def test_dist_graph_replay_world1(nrmf):
    """nrmf.dist (tree kernel + ncclAllGather + rank tree) captured on a
    1-rank NCCL communicator: replays equal the oracle bitwise."""
    import torch.distributed as td
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    created = False
    if not td.is_initialized():
        td.init_process_group("gloo", rank=0, world_size=1)
        created = True
    try:
        for dt in (np.float64, np.float32):
            n = 100 * T + 5
            xh = gen.normal(3, n, dtype=dt)
            x = torch.from_numpy(xh).cuda()
            out = torch.empty((), dtype=x.dtype, device="cuda")
            comm = nrmf.comm_for(None)
            g = nrmf.capture(lambda: nrmf.dist(x, n, comm=comm, out=out))
            for _ in range(2):
                g.replay()
                torch.cuda.synchronize()
                assert bits(out.cpu().numpy(), dt) == bits(oracle.nrmf(xh), dt)
    finally:
        for c in list(nrmf._comms.values()):
            c.close()
        nrmf._comms.clear()
        if created:
            td.destroy_process_group()


def test_graphs_own_their_workspaces(nrmf):
    """each captured graph owns its workspace (g._nrmf_ws), so two
    graphs never share arrival counters, a later capture that needs more space
    cannot free an earlier graph's, and clear_workspaces() leaves them alive."""
    xs = [gen.normal(11 + i, n, dtype=np.float64) for i, n in enumerate((300 * T + 11, 3000 * T + 5))]
    xd = [torch.from_numpy(x).cuda() for x in xs]
    outs = [torch.empty((), dtype=torch.float64, device="cuda") for _ in xs]
    gs = [nrmf.capture(lambda x=x, o=o: nrmf.norm(x, out=o)) for x, o in zip(xd, outs)]
    ptrs = [{t.data_ptr() for t in g._nrmf_ws} for g in gs]
    assert ptrs[0] and ptrs[1] and not (ptrs[0] & ptrs[1])
    nrmf.clear_workspaces()
    torch.cuda.empty_cache()
    junk = torch.full((1 << 26,), 0xAB, dtype=torch.uint8, device="cuda")  # reuse freed blocks, if any
    side = torch.cuda.Stream()
    for _ in range(3):
        gs[0].replay()
        with torch.cuda.stream(side):
            gs[1].replay()                   # concurrently on another stream
        torch.cuda.synchronize()
        for o, x in zip(outs, xs):
            assert bits(o.cpu().numpy(), np.float64) == bits(oracle.nrmf(x), np.float64)
    del junk


def _graph_node_types(g):
    """Node types of a captured graph (cuda-python on the raw cudaGraph_t)."""
    from cuda.bindings import runtime as rt
    graph = rt.cudaGraph_t(init_value=g.raw_cuda_graph())
    err, nodes, num = rt.cudaGraphGetNodes(graph, 0)
    assert err == rt.cudaError_t.cudaSuccess
    err, nodes, num = rt.cudaGraphGetNodes(graph, num)
    assert err == rt.cudaError_t.cudaSuccess
    kinds = []
    for nd in nodes[:num]:
        err, t = rt.cudaGraphNodeGetType(nd)
        assert err == rt.cudaError_t.cudaSuccess
        kinds.append(t.name)
    return kinds


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", [3 * T + 7, 256 * T, (1 << 24) + 5])
def test_captured_call_is_one_kernel(nrmf, dt, n):
    """VERDICT r1 (C1, one graph node per call): a captured norm uses its own
    zero-filled arena workspace with NRMF_WS_CLEAN, so the graph holds the
    tree kernel alone -- no counter memset -- and replays stay bit-exact
    (every completed call leaves the counters zero for the next replay)."""
    x1 = gen.uniform_pm1(17, n, dtype=dt)
    x = torch.from_numpy(x1).cuda()
    out = torch.empty((), dtype=x.dtype, device="cuda")
    g = torch.cuda.CUDAGraph(keep_graph=True)
    nrmf.capture(lambda: nrmf.norm(x, out=out), graph=g)
    kinds = _graph_node_types(g)
    assert kinds == ["cudaGraphNodeTypeKernel"], kinds
    g.instantiate()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    assert bits(out.cpu().numpy(), dt) == bits(oracle.nrmf(x1), dt)


def test_ws_clean_direct_calls(nrmf):
    """NRMF_WS_CLEAN through the C ABI on a zero-filled workspace dedicated to
    one call shape: 50 calls back to back, every one bit-exact (the last
    arrivers leave the counters zero); and the same bits as the default."""
    import ctypes
    L = nrmf.lib()
    for dt, f, esz in ((np.float64, L.nrmf_ex_d, 8), (np.float32, L.nrmf_ex_s, 4)):
        for n in (1000, 300 * T + 1, (1 << 23) + 3):
            xh = gen.normal(n, n, dtype=dt)
            x = torch.from_numpy(xh).cuda()
            out = torch.empty(50, dtype=x.dtype, device="cuda")
            nb = L.nrmf_workspace_bytes(n, esz)
            ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
            s = torch.cuda.current_stream().cuda_stream
            for i in range(50):
                assert f(n, x.data_ptr(), out[i:].data_ptr(), nrmf.NRMF_WS_CLEAN, ws.data_ptr(), nb, s) == 0
            torch.cuda.synchronize()
            want = bits(oracle.nrmf(xh), dt)
            got = out.cpu().numpy()
            assert all(bits(v, dt) == want for v in got), n
