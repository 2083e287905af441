"""The seeded generators: deterministic, index-addressable (shards and chunks
reproduce the whole array bitwise), and of the configured distributions."""
import numpy as np
import pytest

import nrmf_inputs as gen


@pytest.mark.parametrize("make", [
    lambda n, off: gen.uniform_pm1(4, n, off),
    lambda n, off: gen.uniform_pm1(4, n, off, dtype=np.float32),
    lambda n, off: gen.sme(4, n, off),
    lambda n, off: gen.normal(4, n, off),
    lambda n, off: gen.normal(4, n, off, dtype=np.float32),
    lambda n, off: gen.extreme(4, n, "fin2", off),
])
def test_index_addressable(make):
    whole = make(10000, 0)
    parts = np.concatenate([make(3000, 0), make(4567, 3000), make(10000 - 7567, 7567)])
    assert whole.tobytes() == parts.tobytes()
    assert whole.tobytes() == make(10000, 0).tobytes()


def test_distributions():
    u = gen.uniform_pm1(1, 1 << 20)
    assert u.min() >= -1 and u.max() < 1 and abs(u.mean()) < 0.005
    z = gen.normal(1, 1 << 20)
    assert abs(z.mean()) < 0.005 and abs(z.var() - 1) < 0.01
    s = gen.sme(1, 1 << 20)
    assert s.dtype == np.float32
    m, e = np.frexp(np.abs(s))
    assert (e - 1).min() == -20 and (e - 1).max() == 20
    assert abs((s > 0).mean() - 0.5) < 0.005
    A = gen.colscaled_normal(3, 64, 100)
    k = np.log2(np.abs(A.reshape(100, 64)).max(axis=1))
    assert k.min() > -32 and k.max() < 33
    x = gen.extreme(1, 1 << 16, "lit")
    assert np.all(np.isfinite(x)) and np.abs(x).max() <= 0.99 * np.finfo(np.float64).max
    assert (np.abs(x) < np.finfo(np.float64).tiny).mean() > 0.01   # subnormals present


def test_column_generator_matches_linear_index():
    """Column j of C4 uses normals at linear index j*r + i; any column block
    generated alone equals the same block of the whole matrix."""
    r, c = 100, 12
    A = gen.colscaled_normal(9, r, c)
    B = gen.colscaled_normal(9, r, c, c0=5, cc=4)
    assert A[5 * r:9 * r].tobytes() == B.tobytes()
    A2 = gen.colscaled_normal(9, r, c, ld=103)
    for j in range(c):
        assert A2[j * 103:j * 103 + r].tobytes() == A[j * r:(j + 1) * r].tobytes()
