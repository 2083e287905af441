"""GPU parity of the stream kernel's safe mode (fp64).

After a warp group that needed the exact path (a leaf outside the fast
domain), the warp evaluates its next groups with the safe node
(Listing 2 for every operand) straight from the shared-memory ring
and returns to the fast path after a group whose leaves all lie in the fast
domain.  The mode only changes who evaluates a node how fast, never the tree
or the node's bits, so every result must be the oracle's -- whatever mix of
flagged and clean groups a warp sees, entering and leaving the mode many
times, with tile values written (column blocks), both tops, forced grids."""
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


def bits(v):
    return np.asarray(v, dtype=np.float64).tobytes()


def planted(seed, n, density, kinds=("huge", "tiny", "sub", "inf")):
    """N(0,1) with a fraction `density` of elements replaced by values that
    flag their leaf: huge (>= 2^1012), tiny pairs' partners, subnormals, inf."""
    rng = np.random.default_rng(seed)
    x = gen.normal(seed, n)
    k = max(1, int(n * density))
    pos = rng.choice(n, size=k, replace=False)
    vals = []
    for i in range(k):
        kind = kinds[i % len(kinds)]
        if kind == "huge":
            vals.append(np.ldexp(1.0 + rng.random(), int(rng.integers(1012, 1014))))
        elif kind == "tiny":
            vals.append(np.ldexp(1.0 + rng.random(), int(rng.integers(-1020, -901))))
        elif kind == "sub":
            vals.append(np.ldexp(1.0, -1074) * int(rng.integers(1, 1 << 40)))
        else:
            vals.append(np.inf)
    x[pos] = np.array(vals) * np.where(rng.random(k) < 0.5, -1.0, 1.0)
    return x


def tiny_blocks(seed, n, every):
    """Whole groups of subnormal/tiny data (every leaf flagged) every
    `every`-th 8-tile block, N(0,1) elsewhere: long runs in and out of safe mode."""
    x = gen.normal(seed, n)
    blk = 8 * T
    for b in range(0, n // blk, every):
        x[b * blk:(b + 1) * blk] *= 2.0 ** -1030
    return x


@pytest.mark.parametrize("density", [1e-7, 1e-6, 1e-5, 1e-4, 1e-3])
@pytest.mark.parametrize("grid", [0, 1, 7, 148])
def test_safe_mode_planted(nrmf, density, grid):
    n = 3000 * T + 17
    x = planted(int(density * 1e7) + grid, n, density, kinds=("huge", "tiny", "sub"))
    want = bits(oracle.nrmf(x))
    xd = torch.from_numpy(x).cuda()
    try:
        nrmf._debug_set_grid(grid)
        assert bits(nrmf.norm(xd).cpu().numpy()) == want
    finally:
        nrmf._debug_set_grid(0)


@pytest.mark.parametrize("every", [2, 3, 5])
@pytest.mark.parametrize("grid", [1, 2, 148])
def test_safe_mode_runs(nrmf, every, grid):
    """Runs of flagged groups between clean ones on every warp."""
    n = 2048 * T
    x = tiny_blocks(every, n, every)
    want = bits(oracle.nrmf(x))
    xd = torch.from_numpy(x).cuda()
    try:
        nrmf._debug_set_grid(grid)
        for step in (True, False):
            nrmf._debug_set_cta_step(step)
            assert bits(nrmf.norm(xd).cpu().numpy()) == want
    finally:
        nrmf._debug_set_grid(0)
        nrmf._debug_set_cta_step(True)


def test_safe_mode_inf_and_nan(nrmf):
    n = 2500 * T + 3
    x = planted(5, n, 1e-5, kinds=("huge", "inf"))
    assert bits(nrmf.norm(torch.from_numpy(x).cuda()).cpu().numpy()) == bits(oracle.nrmf(x))
    y = x.copy()
    y[1000 * T:1000 * T + 2] = np.nan  # two NaN leaves meet: the tile is NaN
    r = nrmf.norm(torch.from_numpy(y).cuda()).cpu().numpy()
    assert bits(r) == bits(oracle.nrmf(y))


def test_safe_mode_top_cr(nrmf):
    n = 2000 * T + 5
    x = tiny_blocks(9, n, 3)
    x[::100003] = 2.0 ** 1015
    r = nrmf.norm(torch.from_numpy(x).cuda(), top="cr").cpu().numpy()
    assert bits(r) == bits(oracle.nrmf(x, top="cr"))


@pytest.mark.parametrize("grid", [0, 2, 9])
def test_safe_mode_column_blocks(nrmf, grid):
    """Back-to-back columns of T rows (stream kernel, tile values = column
    norms): columns scaled by 2^k with k over the whole range, so flagged and
    clean groups alternate; every column norm and the Frobenius norm equal the
    oracle's."""
    rows, c = T, 4096 + 8 * 37 + 3
    rng = np.random.default_rng(grid + 1)
    A = gen.normal(grid + 3, rows * c).reshape(c, rows)
    k = rng.integers(-1070, 1015, size=c)
    k[rng.random(c) < 0.7] = 0  # mostly clean columns
    A = np.ldexp(A, k[:, None]).reshape(-1)
    At = torch.from_numpy(A).cuda().as_strided((rows, c), (1, rows))
    ecol, efr = oracle.cols(A, rows, c, rows)
    try:
        nrmf._debug_set_grid(grid)
        col, fr = nrmf.cols(At)
        assert col.cpu().numpy().tobytes() == np.asarray(ecol).tobytes()
        assert bits(fr.cpu().numpy()) == bits(efr)
    finally:
        nrmf._debug_set_grid(0)


def test_safe_mode_unaligned(nrmf):
    """The unaligned stream kernel's safe mode (element-aligned base)."""
    n = 2200 * T + 9
    x = tiny_blocks(4, n, 2)
    buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(x).cuda()
    assert bits(nrmf.norm(buf[1:]).cpu().numpy()) == bits(oracle.nrmf(x))


@pytest.mark.parametrize("variant", ["lit", "fin", "fin2"])
def test_safe_mode_c5_graph_replays(nrmf, variant):
    """C5 recipe at 2^24 as graph replays (every warp in safe mode after its
    first group): the oracle's bits on every replay."""
    n = 1 << 24
    x = gen.extreme(3, n, variant)
    want = bits(oracle.nrmf(x))
    xd = torch.from_numpy(x).cuda()
    out = torch.empty((), dtype=torch.float64, device="cuda")
    g = nrmf.capture(lambda: nrmf.norm(xd, out=out))
    for _ in range(5):
        g.replay()
        torch.cuda.synchronize()
        assert bits(out.cpu().numpy()) == want
