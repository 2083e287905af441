"""The split kernel's last combine step by flag-in-data slots (nrmf.cu,
ll_*): the same tree as the counter-based step, so the same bits as the
oracle; garbage workspaces, back-to-back calls on one workspace (the epoch
advances, nothing is cleared), CUDA-graph replays and the one- and two-step
plans (<= 256 and up to 592 warp groups)."""
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


SIZES = [T + 1, 2 * T, 3 * T + 5, 33 * T, 256 * T, 256 * T + 1, 300 * T + 7, 591 * T, 592 * T + 3, 1100 * T + 9]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("top", ["v1", "cr"])
def test_ll_last_step_equals_counter_step_and_oracle(nrmf, dt, top):
    for n in SIZES:
        x = gen.normal(n + 11, n, dtype=dt)
        xd = torch.from_numpy(x).cuda()
        want = bits(oracle.nrmf(x, top=top), dt)
        try:
            nrmf._debug_set_split_ll(False)
            a = nrmf.norm(xd, top=top).cpu().numpy()
        finally:
            nrmf._debug_set_split_ll(True)
        b = nrmf.norm(xd, top=top).cpu().numpy()
        assert bits(a, dt) == want and bits(b, dt) == want, n


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_ll_garbage_workspace_and_many_calls(nrmf, dt):
    """Workspaces full of random bytes (incl. a copy of a used one) and 200
    calls back to back on one workspace (the epoch word advances by one per
    call, the slots keep the previous call's values): always the oracle's bits."""
    import ctypes
    L = nrmf.lib()
    f, esz = (L.nrmf_d, 8) if dt == np.float64 else (L.nrmf_s, 4)
    s = torch.cuda.current_stream().cuda_stream
    for n in (100 * T + 3, 256 * T, 500 * T + 1):
        x = gen.sme(n, n, dtype=dt)
        xd = torch.from_numpy(x).cuda()
        want = bits(oracle.nrmf(x), dt)
        nb = L.nrmf_workspace_bytes(n, esz)
        g = torch.Generator(device="cuda").manual_seed(n)
        for trial in range(5):
            ws = torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda", generator=g)
            outs = torch.empty(40, dtype=xd.dtype, device="cuda")
            for i in range(40):
                assert f(n, xd.data_ptr(), outs[i:].data_ptr(), ws.data_ptr(), nb, s) == 0
            torch.cuda.synchronize()
            assert all(bits(v, dt) == want for v in outs.cpu().numpy()), (n, trial)
        used = ws.clone()                              # a copy of a used workspace
        outs = torch.empty(1, dtype=xd.dtype, device="cuda")
        assert f(n, xd.data_ptr(), outs.data_ptr(), used.data_ptr(), nb, s) == 0
        torch.cuda.synchronize()
        assert bits(outs.cpu().numpy()[0], dt) == want


def test_ll_graph_replay(nrmf):
    n = 256 * T
    x1 = gen.uniform_pm1(1, n)
    x = torch.from_numpy(x1).cuda()
    out = torch.empty((), dtype=torch.float64, device="cuda")
    g = nrmf.capture(lambda: nrmf.norm(x, out=out))
    for _ in range(50):
        g.replay()
    torch.cuda.synchronize()
    assert bits(out.cpu().numpy(), np.float64) == bits(oracle.nrmf(x1), np.float64)


@pytest.mark.parametrize("seed", [1, 2])
def test_ll_one_workspace_shared_by_many_shapes(nrmf, seed):
    """One workspace shared by calls of many sizes and both precisions in a
    random order (the Python binding caches one workspace per stream and kind,
    so a test suite does exactly this): the layouts overlap -- one shape's
    slots and counters sit on another's header -- and no call may pick up a
    stale slot.  300 calls, each checked against the oracle."""
    import ctypes
    L = nrmf.lib()
    rng = np.random.default_rng(seed)
    shapes = [(n, dt) for n in (3 * T + 5, 33 * T, 64 * T + 1, 100 * T + 3, 256 * T, 300 * T + 7, 591 * T, 1000 * T)
              for dt in (np.float64, np.float32)]
    data = {}
    for n, dt in shapes:
        x = gen.normal(n + (dt == np.float32), n, dtype=dt)
        data[(n, dt)] = (torch.from_numpy(x).cuda(), bits(oracle.nrmf(x), dt))
    nb = max(L.nrmf_workspace_bytes(n, 8) for n, _ in shapes)
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    outs = {k: torch.empty((), dtype=v[0].dtype, device="cuda") for k, v in data.items()}
    for i in range(300):
        k = shapes[int(rng.integers(len(shapes)))]
        xd, want = data[k]
        f = L.nrmf_d if k[1] == np.float64 else L.nrmf_s
        assert f(k[0], xd.data_ptr(), outs[k].data_ptr(), ws.data_ptr(), nb, s) == 0
        torch.cuda.synchronize()
        assert bits(outs[k].cpu().numpy(), k[1]) == want, (i, k)
        if i % 50 == 49:
            ws[: 4096].zero_()      # another user of the memory resets a prefix (headers of small layouts)
