"""GPU parity of the unaligned-vector stream kernel (StreamLoader UNAL).

A vector whose base is a multiple of its element size but not of 16 bytes is
the paper's unaligned case (head / body / tail: the body is loaded
with aligned vector loads, the unaligned head and the masked tail by element).
Here the stream kernel fetches each batch as the aligned 16-byte span around
it and the lanes read their rows from the shifted stage; the group whose span
would start before x (group 0) and a last full group without 16 bytes of the
array after it go through element loads.  The tree does not depend on the
base, so every result must equal the oracle on the same values, the aligned
copy and the element-load kernel, bit for bit."""
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


def shifted(x, shift):
    """x on the device at `shift` elements past a 256-byte aligned base."""
    t = NP2T[x.dtype.type]
    buf = torch.empty(x.size + shift + 64, dtype=t, device="cuda")
    buf.fill_(float("nan"))  # the bytes around the view must not matter
    buf[shift:shift + x.size] = torch.from_numpy(x).cuda()
    v = buf[shift:shift + x.size]
    assert (v.data_ptr() % 16 != 0) == (shift * x.itemsize % 16 != 0)
    return v


def norm_three_ways(nrmf, x, shift):
    """(unaligned on the stream kernel, unaligned on the element-load kernel,
    16-byte aligned copy)."""
    v = shifted(x, shift)
    r_u = nrmf.norm(v).cpu().numpy()
    try:
        nrmf._debug_set_unal_stream(False)
        r_e = nrmf.norm(v).cpu().numpy()
    finally:
        nrmf._debug_set_unal_stream(True)
    r_a = nrmf.norm(torch.from_numpy(x).cuda()).cpu().numpy()
    return r_u, r_e, r_a


CASES = [
    # (dtype, shift in elements, tiles, extra elements)
    (np.float64, 1, 3000, 11),      # ragged tail of >= 16 bytes: every full group streamed but group 0
    (np.float64, 1, 4096, 0),       # no tail: the last full group by element loads
    (np.float64, 1, 2047, 1),       # an 8-byte tail (< 16): the last full group by element loads
    (np.float64, 3, 1500, 4095),
    (np.float32, 1, 3000, 3),       # 12-byte tail
    (np.float32, 2, 3000, 4),       # 16-byte tail: streamed
    (np.float32, 3, 4096, 0),
    (np.float32, 1, 1999, 777),
]


@pytest.mark.parametrize("dt,shift,tiles,extra", CASES)
def test_unaligned_stream_same_bits(nrmf, dt, shift, tiles, extra):
    n = tiles * T + extra
    x = gen.normal(21 + tiles, n, dtype=dt)
    r_u, r_e, r_a = norm_three_ways(nrmf, x, shift)
    want = bits(oracle.nrmf(x), dt)
    assert bits(r_u, dt) == want
    assert bits(r_e, dt) == want
    assert bits(r_a, dt) == want


@pytest.mark.parametrize("dt,shift", [(np.float64, 1), (np.float32, 1), (np.float32, 3)])
@pytest.mark.parametrize("grid", [1, 7, 148, 300])
def test_unaligned_stream_forced_grids(nrmf, dt, shift, grid):
    """Warps with many groups each, warp 0 starting at group W (group 0 by
    element loads), CTA step on and off."""
    n = 900 * T + 5
    x = gen.uniform_pm1(77, n, dtype=dt)
    want = bits(oracle.nrmf(x), dt)
    v = shifted(x, shift)
    try:
        nrmf._debug_set_grid(grid)
        for step in (True, False):
            nrmf._debug_set_cta_step(step)
            assert bits(nrmf.norm(v).cpu().numpy(), dt) == want
    finally:
        nrmf._debug_set_grid(0)
        nrmf._debug_set_cta_step(True)


@pytest.mark.parametrize("variant", ["fin2", "lit"])
def test_unaligned_stream_extreme_range(nrmf, variant):
    """Flagged groups (out-of-domain leaves, subnormals, inf) on the UNAL
    kernel take the exact path with element loads: same bits."""
    n = 1200 * T + 3
    x = gen.extreme(5, n, variant=variant)
    want = bits(oracle.nrmf(x), np.float64)
    r_u, r_e, r_a = norm_three_ways(nrmf, x, 1)
    assert bits(r_u, np.float64) == want
    assert bits(r_e, np.float64) == want
    assert bits(r_a, np.float64) == want


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_unaligned_stream_specials(nrmf, dt):
    """NaN and +-inf inside streamed groups and in group 0 (a NaN leaf is
    dropped by fmin/fmax, Listing 2; two NaNs meeting give NaN)."""
    n = 1000 * T + 9
    x = gen.normal(8, n, dtype=dt)
    for pos in ((5,), (3 * T * 8 + 100,), (700 * T + 3,), (700 * T + 2, 700 * T + 3), (4, 5)):
        for val in (np.inf, -np.inf, np.nan):
            y = x.copy()
            y[list(pos)] = val
            r_u, r_e, r_a = norm_three_ways(nrmf, y, 1)
            want = bits(oracle.nrmf(y), dt)
            assert bits(r_u, dt) == want and bits(r_e, dt) == want and bits(r_a, dt) == want


def test_unaligned_stream_graph_replay(nrmf):
    """Captured unaligned call: replays give the oracle's bits."""
    n = 2000 * T + 1
    x = gen.normal(4, n)
    v = shifted(x, 1)
    want = bits(oracle.nrmf(x), np.float64)
    out = torch.empty((), dtype=torch.float64, device="cuda")
    g = nrmf.capture(lambda: nrmf.norm(v, out=out))
    for _ in range(5):
        g.replay()
        torch.cuda.synchronize()
        assert bits(out.cpu().numpy(), np.float64) == want


@pytest.mark.slow
def test_unaligned_c3_size(nrmf):
    """2^28 fp64 at an 8-byte offset (the bench's unaligned line): the oracle's bits."""
    n = 1 << 28
    x = gen.normal(1, n)
    v = shifted(x, 1)
    assert bits(nrmf.norm(v).cpu().numpy(), np.float64) == bits(oracle.nrmf(x), np.float64)
