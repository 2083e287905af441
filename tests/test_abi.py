"""The C-ABI library loads and exports every symbol include/nrmf.h declares;
host-only entry points (no GPU needed) behave as documented."""
import os
import re

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nrmf.h")


@pytest.fixture(scope="module")
def L():
    from paper_2509_06220_b200 import _build
    _build.build()
    import paper_2509_06220_b200 as nrmf
    return nrmf.lib()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:char\s*\*|int|size_t|void)\s+\**\s*(nrmf_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = declared_symbols()
    for n in ("nrmf_s", "nrmf_d", "nrmf_cols_s", "nrmf_cols_d", "nrmf_dist_d"):
        assert n in names
    assert len(names) >= 20


def test_every_declared_symbol_is_exported(L):
    for name in declared_symbols():
        assert hasattr(L, name), name


def test_status_strings_and_version(L):
    assert L.nrmf_tree_version() == 1
    for s in range(7):
        assert L.nrmf_status_str(s).startswith(b"NRMF_")


def test_tree_params_match_design(L):
    import paper_2509_06220_b200 as nrmf
    import torch
    assert nrmf.tree_params(torch.float64) == (64, 64, 4096)
    assert nrmf.tree_params(torch.float32) == (128, 32, 4096)
    # the oracle restates the same constants independently
    import numpy as np
    assert oracle.TREE[np.dtype(np.float64)] == (64, 64)
    assert oracle.TREE[np.dtype(np.float32)] == (128, 32)


def test_workspace_sizes(L):
    assert L.nrmf_workspace_bytes(0, 8) >= 256
    assert L.nrmf_workspace_bytes(-1, 8) == 0
    assert L.nrmf_workspace_bytes(1 << 30, 8) >= (1 << 30) // 4096 // 8 * 8
    assert L.nrmf_cols_workspace_bytes(4096, 65536, 8) >= 65536 // 8 * 8
    assert L.nrmf_dist_workspace_bytes(1 << 30, 8, 8) > 0
    assert L.nrmf_host_workspace_bytes(1 << 20, 8) > (1 << 20) * 8 // 2


def test_argument_errors_without_gpu(L):
    # invalid arguments are rejected at enqueue time, before touching the device
    assert L.nrmf_d(-1, None, None, None, 0, None) == 1          # EINVAL
    assert L.nrmf_d(10, 12, 16, 1024, 4096, None) == 2            # EALIGN (12 % 8)
    assert L.nrmf_s(10, 6, 16, 1024, 4096, None) == 2             # EALIGN (6 % 4)
    assert L.nrmf_d(10, 16, 16, 1024, 0, None) == 3               # EWORKSPACE
    assert L.nrmf_cols_d(10, 2, 5, 16, 16, None, 1024, 1 << 20, None) == 1   # ld < rows


def test_workspace_alignment_is_checked_at_enqueue(L):
    # a workspace not 16-byte aligned is NRMF_EALIGN (nrmf.h), not an
    # asynchronous fault; checked before any device work
    big = 1 << 20
    assert L.nrmf_d(10, 16, 16, 1024 + 8, big, None) == 2
    assert L.nrmf_s(10, 16, 16, 1024 + 4, big, None) == 2
    assert L.nrmf_cols_d(10, 2, 10, 16, 16, None, 1024 + 8, big, None) == 2
    assert L.nrmf_host_d(10, 16, 16, 1024 + 8, 1 << 30, None) == 2
    assert L.nrmf_dist_local_d(10, 1, 0, 0, 10, 16, 16, 0, 1024 + 8, big, None) == 2
    assert L.nrmf_dist_local_d(10, 2, 2, 0, 10, 16, 16, 0, 1024, big, None) == 1      # rank >= world
    assert L.nrmf_dist_local_d(10, 2, 0, 0, 9, 16, 16, 0, 1024, big, None) == 4       # not the canonical shard
    assert L.nrmf_dist_local_d(10, 3, 0, 0, 10, 16, 16, 0, 1024, big, None) == 4      # world not a power of two
    assert L.nrmf_rank_combine_d(10, 2, 12, 16, 0, None) == 2                          # values misaligned
    assert L.nrmf_rank_combine_d(10, 2, 16, 16, 4, None) == 1                          # unknown flag


@pytest.mark.parametrize("n,G", [(1 << 30, 1), (1 << 30, 2), (1 << 30, 8), (5, 8), (4097, 4),
                                 (17 * 4096 - 3, 8), (0, 2)])
def test_shard_partition_matches_oracle_reading(n, G):
    """nrmf_dist_shard (C, host-only) == the oracle's restatement of the
    canonical partition; shards tile [0, n) contiguously."""
    import paper_2509_06220_b200 as nrmf
    exp = oracle.shard_ranges(n, G)
    got = [nrmf.shard(n, G, g) for g in range(G)]
    assert got == [(a, c) for a, c, _ in exp]
    pos = 0
    for a, c in got:
        assert a == pos or c == 0
        pos = a + c if c else pos
    assert sum(c for _, c in got) == n


def test_shard_rejects_non_power_of_two(L):
    import paper_2509_06220_b200 as nrmf
    with pytest.raises(RuntimeError):
        nrmf.shard(1000, 3, 0)


@pytest.mark.parametrize("c,G", [(65536, 1), (65536, 8), (5, 8), (7, 4), (1, 2), (0, 4), (100, 2)])
def test_cols_shard_partition_matches_oracle_reading(c, G):
    """nrmf_cols_dist_shard (C, host-only) == the oracle's restatement of the
    canonical column blocks; blocks cover [0, c) contiguously."""
    import paper_2509_06220_b200 as nrmf
    exp = oracle.cols_shard_ranges(c, G)
    got = [nrmf.cols_shard(c, G, g) for g in range(G)]
    assert got == [(a, n) for a, n, _ in exp]
    assert sum(n for _, n in got) == c
