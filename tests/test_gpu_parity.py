"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit for bit.

Every expected value comes from ``oracle`` (plain C, same tree) on the same
seeded inputs; accuracy is checked against the exact reference.  Sizes span
several tiles/groups and ragged tails; full BASELINE sizes are in the `slow`
tests at the bottom (same launch configuration bench.py times)."""
import math
import os

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


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def bits(v, dt):
    return np.asarray(v, dtype=dt).tobytes()


def gpu_norm(nrmf, x):
    r = nrmf.norm(dev(x))
    return r.cpu().numpy()


DISTS = {
    "uniform": lambda s, n, dt: gen.uniform_pm1(s, n, dtype=dt),
    "normal": lambda s, n, dt: gen.normal(s, n, dtype=dt),
    "sme": lambda s, n, dt: gen.sme(s, n, dtype=dt),
}

SIZES = [0, 1, 2, 3, 31, 64, 65, 127, 128, 129, 4095, 4096, 4097, 8191, 2 * T + 3,
         8 * T - 1, 8 * T, 8 * T + 1, 9 * T + 17, 17 * T, 64 * T + 1, 100 * T + 999, 257 * T + 5]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", SIZES)
def test_parity_sizes(nrmf, dt, n):
    x = gen.normal(n + 1, n, dtype=dt)
    assert bits(gpu_norm(nrmf, x), dt) == bits(oracle.nrmf(x), dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("dist", list(DISTS))
def test_parity_random_sizes(nrmf, dt, dist):
    rng = np.random.default_rng(12345)
    for n in rng.integers(1, 1 << 20, 6):
        x = DISTS[dist](int(n), int(n), dt)
        assert bits(gpu_norm(nrmf, x), dt) == bits(oracle.nrmf(x), dt), n


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("shift", [1, 2, 3])
def test_unaligned_base_same_bits(nrmf, dt, shift):
    """16-byte vector loads vs element loads give identical bits."""
    n = 37 * T + 11
    x = gen.uniform_pm1(9, n, dtype=dt)
    buf = torch.zeros(n + 8, dtype=NP2T[dt], device="cuda")
    buf[shift:shift + n] = dev(x)
    view = buf[shift:shift + n]
    assert view.data_ptr() % 16 != 0 or shift * np.dtype(dt).itemsize % 16 == 0
    r = nrmf.norm(view).cpu().numpy()
    assert bits(r, dt) == bits(oracle.nrmf(x), dt)


def test_c1_dnrmf_2p20_uniform(nrmf):
    """BASELINE config C1: DNRMF fp64, n = 2^20, U[-1,1)."""
    for seed in range(1, 6):
        x = gen.uniform_pm1(seed, 1 << 20)
        r = gpu_norm(nrmf, x)
        assert bits(r, np.float64) == bits(oracle.nrmf(x), np.float64)
        assert oracle.relerr(r, oracle.exact(x)) < 3


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_reproducible_across_runs_and_grids(nrmf, dt):
    n = 300 * T + 77
    x = dev(gen.normal(3, n, dtype=dt))
    ref = nrmf.norm(x).cpu().numpy()
    for _ in range(100):
        assert bits(nrmf.norm(x).cpu().numpy(), dt) == bits(ref, dt)
    try:
        for g in (1, 7, 148, 296, 592):
            nrmf._debug_set_grid(g)
            assert bits(nrmf.norm(x).cpu().numpy(), dt) == bits(ref, dt), g
    finally:
        nrmf._debug_set_grid(0)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", [8 * T * 3000 + 5, 2400 * T + 1, (1 << 24) + 3])
def test_same_bits_for_every_group_size_and_grid(nrmf, dt, n):
    """The tree does not depend on how tiles are batched into warp groups
    (g0 = 0..4, i.e. 1..16 tiles; 16 on the fp32 stream kernel, clamped to 8
    for fp64) nor on the persistent grid: every
    combination gives the oracle's bits (stream kernel with full groups, a
    partial last group and a ragged tail)."""
    xh = gen.sme(n % 1000, n, dtype=dt)
    x = dev(xh)
    exp = bits(oracle.nrmf(xh), dt)
    try:
        for g0 in (0, 1, 2, 3, 4):
            nrmf._debug_set_g0(g0)
            for grid in (0, 37, 148):
                nrmf._debug_set_grid(grid)
                assert bits(nrmf.norm(x).cpu().numpy(), dt) == exp, (g0, grid)
    finally:
        nrmf._debug_set_g0(-1)
        nrmf._debug_set_grid(0)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("grid", [1, 2, 5])
@pytest.mark.parametrize("case", ["normal", "nan_group", "zero_run", "huge_tiny", "cr"])
def test_cta_combine_step(nrmf, dt, grid, case):
    """The stream kernel's first combine step in shared memory (16 warp groups
    of a round per CTA, claimed by the first warp to finish its next round):
    small grids give many rounds per CTA (slot reuse beyond the 4 slots),
    partial last blocks and a ragged tail; a NaN group, runs of +0 groups and
    out-of-fast-domain group values take the exact fallback of that step;
    top="cr" evaluates it with cr_hypot.  Same bits as the oracle, and as
    with the step disabled (global fan-in-64 climbs only)."""
    G = 16 if dt == np.float32 else 8
    n = grid * 16 * G * T * 9 + 5 * G * T + 3 * T + 17      # 9 full rounds, a partial one, ragged tail
    xh = gen.normal(grid * 7 + len(case), n, dtype=dt)
    if case == "nan_group":
        xh[3 * G * T + 5] = np.nan
    elif case == "zero_run":
        xh[: 40 * G * T] = 0
    elif case == "huge_tiny":
        # group values above / below the fast node's domain of M
        # ([2^-900, 2^1012) fp64, [2^-80, 2^116) fp32): one large group, 16 tiny
        big, tiny = (2.0 ** 1010, 2.0 ** -950) if dt == np.float64 else (2.0 ** 110, 2.0 ** -100)
        xh[G * T * 17: G * T * 18] *= dt(big)
        xh[G * T * 40: G * T * 56] *= dt(tiny)
    top = "cr" if case == "cr" else "v1"
    exp = bits(oracle.nrmf(xh, top=top), dt)
    x = dev(xh)
    try:
        nrmf._debug_set_grid(grid)
        for on in (True, False):
            nrmf._debug_set_cta_step(on)
            assert bits(nrmf.norm(x, top=top).cpu().numpy(), dt) == exp, on
    finally:
        nrmf._debug_set_cta_step(True)
        nrmf._debug_set_grid(0)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("top", ["v1", "cr"])
@pytest.mark.parametrize("extra", [0, 5])
def test_cta_combine_step_is_root(nrmf, dt, top, extra):
    """One CTA (grid 1) and exactly 16 warp groups (+ a few elements of a 17th
    group when extra > 0, which adds a global step): the CTA step writes the
    root itself, or feeds the global step."""
    G = 16 if dt == np.float32 else 8
    n = 16 * G * T + extra
    xh = gen.uniform_pm1(n, n, dtype=dt)
    exp = bits(oracle.nrmf(xh, top=top), dt)
    x = dev(xh)
    try:
        nrmf._debug_set_grid(1)
        for on in (True, False):
            nrmf._debug_set_cta_step(on)
            assert bits(nrmf.norm(x, top=top).cpu().numpy(), dt) == exp, on
    finally:
        nrmf._debug_set_cta_step(True)
        nrmf._debug_set_grid(0)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("rows", [T, 2 * T])
def test_cta_combine_step_columns(nrmf, dt, rows):
    """Back-to-back columns of a multiple of T rows take the stream kernel
    (tile values = column norms written by the group step): with a grid of 2
    CTAs it runs many rounds through the CTA combine step.  Column norms and
    the Frobenius norm equal the oracle's, with the step on and off."""
    G = 16 if dt == np.float32 else 8
    c = (2 * 16 * G * 5 + 3 * G + 1) * T // rows
    A = gen.colscaled_normal(11, rows, c, ld=rows, dtype=dt)
    At = dev(A).as_strided((rows, c), (1, rows))
    ecol, efr = oracle.cols(A, rows, c, rows)
    try:
        nrmf._debug_set_grid(2)
        for on in (True, False):
            nrmf._debug_set_cta_step(on)
            col, fr = nrmf.cols(At)
            assert col.cpu().numpy().tobytes() == ecol.tobytes(), on
            assert bits(fr.cpu().numpy(), dt) == bits(efr, dt), on
    finally:
        nrmf._debug_set_cta_step(True)
        nrmf._debug_set_grid(0)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("rows,cols,gap", [(T, 6000, 64), (3 * T, 2001, 64), (2 * T, 3500, 4096 + 32),
                                           (5 * T, 1300, 16)])
@pytest.mark.parametrize("grid", [0, 2, 37])
def test_cols_gapped_stream(nrmf, dt, rows, cols, gap, grid):
    """Column blocks with a gap between columns (ld = rows + gap, rows a
    multiple of T; ld 16-byte aligned for both precisions): the stream
    kernel's walk skips the gaps and seeks every new group from its tile
    index (tiles per column 1, 2, 3, 5 -- groups span columns when tpc < G).
    Column norms and frob equal the oracle's, with the gapped stream path and
    with the general kernel."""
    ld = rows + gap
    A = gen.colscaled_normal(rows + cols, rows, cols, ld=ld, dtype=dt)
    A.reshape(cols, ld)[:, rows:] = np.nan                # the gaps must never be read
    At = dev(A).as_strided((rows, cols), (1, ld))
    ecol, efr = oracle.cols(A, rows, cols, ld)
    try:
        nrmf._debug_set_grid(grid)
        for on in (True, False):
            nrmf._debug_set_gap_stream(on)
            col, fr = nrmf.cols(At)
            assert col.cpu().numpy().tobytes() == ecol.tobytes(), on
            assert bits(fr.cpu().numpy(), dt) == bits(efr, dt), on
    finally:
        nrmf._debug_set_gap_stream(True)
        nrmf._debug_set_grid(0)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("groups_lg", [7, 8])
@pytest.mark.parametrize("case", ["normal", "nan", "huge", "zero_run", "cr"])
def test_split_kernel_wide_last_step(nrmf, dt, groups_lg, case):
    """Small calls (split kernel) finish with one climb of up to 8 levels
    (fan-in 128 / 256): its fast path, and its exact fallback (a NaN tile, an
    out-of-fast-domain tile value, +0 tiles, the cr top), against the oracle."""
    G = 1 if dt == np.float64 else 2                       # split-kernel tiles per group
    n = (1 << groups_lg) * G * T - 3 * T // 2             # ragged last tile
    xh = gen.normal(groups_lg * 10 + len(case), n, dtype=dt)
    if case == "nan":
        xh[5 * T + 7] = np.nan
    elif case == "huge":
        xh[9 * T: 10 * T] *= dt(2.0 ** 1010) if dt == np.float64 else dt(2.0 ** 110)
    elif case == "zero_run":
        xh[: 40 * T] = 0
    top = "cr" if case == "cr" else "v1"
    exp = bits(oracle.nrmf(xh, top=top), dt)
    assert bits(nrmf.norm(dev(xh), top=top).cpu().numpy(), dt) == exp


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_special_values(nrmf, dt):
    """Non-finite inputs follow Listing 2 literally on both sides (reading R4):
    inf anywhere -> inf; a NaN collapses to +0 when it meets a +0 leaf."""
    n = 20 * T + 5
    rng = np.random.default_rng(4)
    cases = []
    x = gen.uniform_pm1(1, n, dtype=dt); x[rng.integers(0, n)] = np.inf; cases.append(x)
    x = gen.uniform_pm1(2, n, dtype=dt); x[rng.integers(0, n, 5)] = np.nan; cases.append(x)
    x = gen.uniform_pm1(3, n, dtype=dt); x[-1] = np.nan; cases.append(x)     # NaN in the tail tile
    x = np.full(n, np.nan, dtype=dt); cases.append(x)
    x = np.zeros(n, dtype=dt); x[::7] = -0.0; cases.append(x)
    x = np.zeros(n, dtype=dt); x[rng.integers(0, n, 3)] = [np.inf, -np.inf, np.nan]; cases.append(x)
    info = np.finfo(dt)
    x = np.full(n, info.tiny, dtype=dt) * dt(0.5); cases.append(x)            # subnormals
    x = np.full(n, info.max / 4, dtype=dt); cases.append(x)                   # overflows to inf
    x = np.zeros(n, dtype=dt); x[0] = info.max; cases.append(x)
    for x in cases:
        g, o = gpu_norm(nrmf, x), oracle.nrmf(x)
        if np.isnan(o):
            assert np.isnan(g)
        else:
            assert bits(g, dt) == bits(o, dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_hypot_many_pairs_via_columns(nrmf, dt):
    """rows = 2 columns: col_norms[j] = v1_hypot(A[0,j], A[1,j]) (the lane tree
    pads with exact v1(a,0) = a nodes).  10^6 pairs over the full exponent
    range, subnormals and exact ties, GPU == oracle bit for bit."""
    m = 1 << 20
    rng = np.random.default_rng(5)
    info = np.finfo(dt)
    emin, emax = (-1074, 1023) if dt == np.float64 else (-149, 127)
    a = np.ldexp(rng.uniform(1, 2, m), rng.integers(emin, emax, m)).astype(dt)
    b = np.ldexp(rng.uniform(1, 2, m), rng.integers(emin, emax, m)).astype(dt)
    k = m // 4
    # q near 1 (rounding-sensitive S = fma(q,q,1)): |b| in [|a|/2, |a|), never
    # beyond |a|, so nothing overflows near the top of the range
    b[:k] = (a[:k].astype(np.float64) * rng.uniform(0.5, 1.0, k)).astype(dt)
    a[k:2 * k] = np.ldexp(rng.integers(0, 1 << 20, k), emin).astype(dt)   # subnormals
    A = np.empty(2 * m, dtype=dt)
    A[0::2], A[1::2] = a, b
    col = nrmf.cols(dev(A).as_strided((2, m), (1, 2)), frob=False).cpu().numpy()
    # a 2-element column is one v1_hypot (two-hot pin of the tree, tests/test_oracle_tree.py)
    assert col.tobytes() == oracle.v1_hypot_array(a, b).tobytes()
    sub = 512
    exp, _ = oracle.cols(A[:2 * sub], 2, sub, 2)
    assert col[:sub].tobytes() == exp.tobytes()
    assert math.isfinite(info.max)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("r,c,ld", [(4096, 1000, 4096), (4096, 37, 4100), (1000, 333, 1000),
                                    (1, 5, 1), (4097, 20, 4097), (9000, 33, 9003), (3 * 4096, 8, 3 * 4096),
                                    (4096, 1, 4096), (7, 300, 9)])
def test_cols_parity(nrmf, dt, r, c, ld):
    A = gen.colscaled_normal(7, r, c, ld=ld, dtype=dt)
    At = dev(A).as_strided((r, c), (1, ld))
    col, fr = nrmf.cols(At)
    ecol, efr = oracle.cols(A, r, c, ld)
    assert col.cpu().numpy().tobytes() == ecol.tobytes()
    assert bits(fr.cpu().numpy(), dt) == bits(efr, dt)
    if r == ld == T:
        assert bits(fr.cpu().numpy(), dt) == bits(oracle.nrmf(A), dt)


def test_cols_empty_shapes(nrmf):
    for r, c in ((0, 5), (5, 0), (0, 0)):
        A = torch.zeros(max(r, 1) * max(c, 1), dtype=torch.float64, device="cuda").as_strided((r, c), (1, max(r, 1)))
        col, fr = nrmf.cols(A)
        assert col.numel() == c and torch.all(col == 0) and fr.item() == 0


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_complex_view(nrmf, dt):
    n = 50 * T + 3
    x = gen.normal(8, 2 * n, dtype=dt)
    z = dev(x).view(torch.complex128 if dt == np.float64 else torch.complex64)
    assert bits(nrmf.norm_complex(z).cpu().numpy(), dt) == bits(oracle.nrmf(x), dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", [0, 5, 4096 * 512, 4096 * 512 * 3 + 17, (1 << 24) + 5])
def test_host_streaming_same_bits(nrmf, dt, n):
    x = gen.normal(21, n, dtype=dt)
    h = torch.from_numpy(x).pin_memory()
    r = nrmf.norm(h).numpy()
    assert bits(r, dt) == bits(oracle.nrmf(x), dt)


def test_dist_world1(nrmf):
    """nrmf_dist_d on a 1-rank NCCL communicator equals nrmf_d bitwise."""
    import torch.distributed as td
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    created = False
    if not td.is_initialized():
        td.init_process_group("gloo", rank=0, world_size=1)
        created = True
    try:
        for dt in (np.float64, np.float32):
            for n in (1, 4097, 100 * T + 5):
                x = gen.normal(2, n, dtype=dt)
                r = nrmf.dist(dev(x), n).cpu().numpy()
                assert bits(r, dt) == bits(oracle.nrmf(x), dt)
    finally:
        for c in list(nrmf._comms.values()):
            c.close()
        nrmf._comms.clear()
        if created:
            td.destroy_process_group()


def test_workspace_contents_do_not_matter(nrmf):
    """A workspace full of garbage (0xFF), and one reused across calls of
    different shapes and functions, gives the same bits."""
    L = nrmf.lib()
    x = gen.normal(4, 300 * T + 7)
    xd = dev(x)
    out = torch.empty((), dtype=torch.float64, device="cuda")
    nb = L.nrmf_workspace_bytes(x.size, 8)
    ws = torch.full((nb + 4096,), 0xFF, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    exp = bits(oracle.nrmf(x), np.float64)
    for _ in range(3):
        assert L.nrmf_d(x.size, xd.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s) == 0
        assert bits(out.cpu().numpy(), np.float64) == exp
        ws.fill_(0xAB)
    # interleave column calls of different layouts on one cached workspace
    for (r, c) in [(9000, 33), (4096, 20000), (9000, 5), (4096, 70000)]:
        A = gen.colscaled_normal(3, r, c)
        col, fr = nrmf.cols(dev(A).as_strided((r, c), (1, r)))
        ecol, efr = oracle.cols(A, r, c, r)
        assert col.cpu().numpy().tobytes() == ecol.tobytes()
        assert bits(fr.cpu().numpy(), np.float64) == bits(efr, np.float64)


def test_errors_raise(nrmf):
    with pytest.raises(ValueError):
        nrmf.norm(torch.zeros(10, dtype=torch.float16, device="cuda"))
    with pytest.raises(ValueError):
        nrmf.norm(torch.zeros(10, 10, dtype=torch.float64, device="cuda").t())


# ------------------------------------------------------------ full sizes
@pytest.mark.slow
def test_c2_snrmf_2p28(nrmf):
    n = 1 << 28
    x = gen.sme(1, n)
    r = gpu_norm(nrmf, x)
    assert bits(r, np.float32) == bits(oracle.nrmf(x), np.float32)
    assert oracle.relerr(r, oracle.exact(x), np.float32) <= 64


@pytest.mark.slow
def test_c3_dnrmf_2p30_normal(nrmf):
    n = 1 << 30
    x = gen.normal(1, n)
    r = gpu_norm(nrmf, x)
    o = oracle.nrmf(x)
    assert bits(r, np.float64) == bits(o, np.float64)
    assert oracle.relerr(r, oracle.exact(x)) <= 64


@pytest.mark.slow
def test_c4_cols_4096x65536(nrmf):
    r, c = 4096, 65536
    A = gen.colscaled_normal(1, r, c)
    col, fr = nrmf.cols(dev(A).as_strided((r, c), (1, r)))
    ecol, efr = oracle.cols(A, r, c, r)
    assert col.cpu().numpy().tobytes() == ecol.tobytes()
    assert bits(fr.cpu().numpy(), np.float64) == bits(efr, np.float64)
    assert oracle.relerr(fr.cpu().numpy(), oracle.exact(A)) <= 64


@pytest.mark.slow
@pytest.mark.parametrize("variant", ["lit", "fin", "fin2"])
def test_c5_extreme_2p27(nrmf, variant):
    n = 1 << 27
    x = gen.extreme(1, n, variant)
    r = gpu_norm(nrmf, x)
    o = oracle.nrmf(x)
    assert bits(r, np.float64) == bits(o, np.float64)
    z = dev(x).view(torch.complex128)
    assert bits(nrmf.norm_complex(z).cpu().numpy(), np.float64) == bits(o, np.float64)
    ex = oracle.exact(x)
    if variant == "lit":
        assert ex == np.inf and r == np.inf
    else:
        assert math.isfinite(ex) and oracle.relerr(r, ex) <= 64


@pytest.mark.slow
def test_max_size_beyond_2p31_elements(nrmf):
    """Maximum-size edge case: n = 2^31 + 3*4096 + 5 fp32 elements (8 GiB): element
    indices beyond 2^31 and a ragged tail in a 2^20-tile tree (P2 = 2^20 with
    2^19 + 4 real tiles); bit-exact with the oracle over the whole array."""
    n = (1 << 31) + 3 * T + 5
    x = gen.sme(3, n)
    r = gpu_norm(nrmf, x)
    assert bits(r, np.float32) == bits(oracle.nrmf(x), np.float32)
    torch.cuda.empty_cache()


PARTIAL = [1, 2, 3, 63, 64, 65, 127, 128, 129, 255, 1000, 2047, 2049, 4031, 4095]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("valid", PARTIAL)
def test_partial_tile_padded_fast_path(nrmf, dt, valid):
    """Partial last tile (valid < T): the padded fast path (padding forced to
    +0 subtree by subtree) is bit-exact with the oracle -- as the last tile of
    a vector, and as every column of a ragged column set (rows = valid)."""
    n = 3 * T + valid
    x = gen.normal(valid, n, dtype=dt)
    assert bits(gpu_norm(nrmf, x), dt) == bits(oracle.nrmf(x), dt)
    c = 6
    A = gen.sme(valid + 1, valid * c, dtype=dt)
    col, fr = nrmf.cols(dev(A).as_strided((valid, c), (1, valid)))
    ecol, efr = oracle.cols(A, valid, c, valid)
    assert col.cpu().numpy().tobytes() == ecol.tobytes()
    assert bits(fr.cpu().numpy(), dt) == bits(efr, dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("special", ["nan", "inf", "zero", "subnormal", "huge"])
@pytest.mark.parametrize("where", ["mixed_pair", "full_pair", "first"])
def test_partial_tile_specials(nrmf, dt, special, where):
    """Specials inside a partial tile send it to the exact path, which keeps
    Listing 2's semantics (e.g. v1(NaN, +0) = +0 next to padding)."""
    valid = 700                      # lanes 0..699 valid; rows 0..ceil((700-l)/p)-1
    n = 2 * T + valid
    x = gen.normal(3, n, dtype=dt)
    fi = np.finfo(dt)
    val = {"nan": np.nan, "inf": np.inf, "zero": 0.0, "subnormal": fi.tiny / 4, "huge": fi.max / 4}[special]
    p = 64 if dt == np.float64 else 128
    # element of the partial tile: row j of lane l is index 2T + j*p + l
    if where == "mixed_pair":        # lane 699's last valid row is paired with padding
        rows = (valid - 699 + p - 1) // p
        idx = 2 * T + (rows - 1) * p + 699
    elif where == "full_pair":
        idx = 2 * T + 0 * p + 5
    else:
        idx = 2 * T
    x[idx] = val
    r = gpu_norm(nrmf, x)
    assert bits(r, dt) == bits(oracle.nrmf(x), dt)


def test_cols_dist_world1(nrmf):
    """nrmf_cols_dist_[ds] on a 1-rank NCCL communicator: column norms and the
    Frobenius norm equal nrmf_cols bitwise (and the oracle)."""
    import torch.distributed as td
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29537")
    created = False
    if not td.is_initialized():
        td.init_process_group("gloo", rank=0, world_size=1)
        created = True
    try:
        for dt in (np.float64, np.float32):
            for (r, c) in ((4096, 33), (5000, 7), (100, 65)):
                A = gen.normal(r + c, r * c, dtype=dt)
                At = dev(A).as_strided((r, c), (1, r))
                col, fr = nrmf.cols_dist(At, c)
                ecol, efr = oracle.cols(A, r, c, r)
                assert col.cpu().numpy().tobytes() == ecol.tobytes()
                assert bits(fr.cpu().numpy(), dt) == bits(efr, dt)
                assert nrmf.cols_dist(At, c, frob=False).cpu().numpy().tobytes() == ecol.tobytes()
    finally:
        for cm in list(nrmf._comms.values()):
            cm.close()
        nrmf._comms.clear()
        if created:
            td.destroy_process_group()
