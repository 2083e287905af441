"""Short columns (rows <= 2 batches of rows: 1024 fp64 / 2048 fp32, 16-byte
aligned columns) evaluated two per warp (warp_tiles_short2): the same tree as
one column at a time, so
the oracle's bits for every column norm and the Frobenius norm -- on the
persistent kernel (many columns), with forced small grids, odd column counts
(a last unpaired column), zero / NaN / inf / huge / subnormal columns (the
exact fallback of a pair), leading dimensions > rows, both tops."""
import numpy as np
import pytest
import torch

import nrmf_inputs as gen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nrmf():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2509_06220_b200 import _build
    _build.build()
    import paper_2509_06220_b200 as m
    m.lib()
    torch.cuda.set_device(0)
    return m


def run(nrmf, r, c, ld, dt, top="v1", specials=False, seed=1):
    A = gen.colscaled_normal(seed, r, c, ld=ld, dtype=dt)
    if specials:
        rng = np.random.default_rng(seed)
        cols = rng.choice(c, 12, replace=False)
        A[cols[0] * ld: cols[0] * ld + r] = 0
        A[cols[1] * ld + r // 2] = np.nan
        A[cols[2] * ld] = np.inf
        A[cols[3] * ld: cols[3] * ld + r] = np.finfo(dt).max / 4
        A[cols[4] * ld: cols[4] * ld + r] = np.finfo(dt).tiny / 8
        A[cols[5] * ld + r - 1] = -np.finfo(dt).max
    T = torch.from_numpy(A).cuda().as_strided((r, c), (1, ld))
    col, fr = nrmf.cols(T, top=top)
    ecol, efr = oracle.cols(A, r, c, ld, top=top)
    got, want = col.cpu().numpy(), ecol
    same = (got.tobytes() == want.tobytes()) or np.array_equal(got, want, equal_nan=True)
    assert same, (r, c, ld, np.nonzero(~((got == want) | (np.isnan(got) & np.isnan(want))))[0][:5])
    f = fr.cpu().numpy()
    assert f.tobytes() == np.asarray(efr, dtype=dt).tobytes() or (np.isnan(f) and np.isnan(efr))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("r", [1, 5, 64, 127, 500, 600, 900, 1000, 1024, 1500, 2048])
def test_short_columns_parity(nrmf, dt, r):
    if dt == np.float64 and r > 1024:
        r = 1023
    a = 2 if dt == np.float64 else 4           # 16-byte aligned columns: the paired path
    lda = -(-r // a) * a
    for c, ld in ((5001, lda), (7777, lda + a), (4099, r + 3)):   # the last: element loads, one at a time
        run(nrmf, r, c, ld, dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_short_columns_specials_and_tops(nrmf, dt):
    a = 2 if dt == np.float64 else 4
    for r in (7, 300, 1000):
        lda = -(-r // a) * a
        run(nrmf, r, 6001, lda, dt, specials=True, seed=r)
        run(nrmf, r, 6001, lda + a, dt, top="cr", seed=r + 1)


@pytest.mark.parametrize("grid", [1, 3, 7])
def test_short_columns_forced_grids(nrmf, grid):
    nrmf._debug_set_grid(grid)
    try:
        for dt in (np.float64, np.float32):
            run(nrmf, 333, 999, 336, dt, seed=grid)
            run(nrmf, 1000, 64, 1000, dt, specials=True, seed=grid + 10)
            run(nrmf, 333, 99, 333, dt, seed=grid + 20)
    finally:
        nrmf._debug_set_grid(0)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_short_columns_identity_skip_edges(nrmf, dt):
    """Columns of at most one batch of rows skip the nodes whose right subtree
    is padding in every lane (v1(L, +0) = L); longer ones (to 15 rows of lane
    0) run the plain path with the same plants.  Plant out-of-domain values and
    NaN in the leaves those skipped nodes pass through (the last valid row of
    lane 0, whose row partner is padding in every lane), one special per
    column, and compare with the oracle: the skipped leaf must keep the fast
    node's leaf check, and a NaN must still reach the exact path."""
    p = 64 if dt == np.float64 else 128
    a = 2 if dt == np.float64 else 4
    fi = np.finfo(dt)
    specials = [0.0, -0.0, np.nan, np.inf, -np.inf, fi.max, -fi.max / 3, fi.tiny / 8, fi.smallest_subnormal,
                fi.tiny * 2, 1.0, -2.5]
    for r in (1, 2, p - 1, p, p + 1, 2 * p + 1, 3 * p - 5, 4 * p + 2, 5 * p, 6 * p + 3, 7 * p + 1, 8 * p,
              8 * p + 1, 9 * p + 1, 10 * p, 11 * p + 7, 13 * p + 2, 14 * p + 1, 15 * p - 1, 15 * p):
        lda = -(-r // a) * a
        c = 2 * len(specials) + 1
        A = gen.colscaled_normal(r, r, c, ld=lda, dtype=dt)
        jmax = -(-r // p)
        row_last = jmax - 1                       # lane 0's last valid row
        for k, sv in enumerate(specials):
            A[k * lda + row_last * p] = sv        # lane 0, last valid row
            A[(len(specials) + k) * lda + r - 1] = sv   # the column's last element
        T = torch.from_numpy(A).cuda().as_strided((r, c), (1, lda))
        col, fr = nrmf.cols(T)
        ecol, efr = oracle.cols(A, r, c, lda)
        got = col.cpu().numpy()
        same = (got.tobytes() == ecol.tobytes()) or np.array_equal(got, ecol, equal_nan=True)
        assert same, (r, np.nonzero(~((got == ecol) | (np.isnan(got) & np.isnan(ecol))))[0][:5])
