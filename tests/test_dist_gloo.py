"""The N>1 (sharded) path's host logic on CPU, with real processes and the gloo
backend: the canonical shard partition (nrmf_dist_shard from libnrmf.so), each
rank generating its own shard with the index-addressable generator, the
per-rank aligned subtree (oracle), the one-scalar exchange, the rank tree, and
the NCCL unique-id bootstrap through torch.distributed.  The combined value must
equal the single-process oracle bit for bit at every world size (the GPU path
runs exactly this partition + combine with NCCL instead of gloo)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as td
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes

        import nrmf_inputs as gen
        import oracle
        import paper_2509_06220_b200 as nrmf
        res = []
        for (n, dt_name, nan_last) in cases:
            dt = np.float64 if dt_name == "f64" else np.float32
            off, cnt = nrmf.shard(n, world, rank)
            x = gen.normal(7, cnt, off, dtype=dt)
            if nan_last and off + cnt == n and cnt > 0:
                x[-1] = np.nan
            ranges = oracle.shard_ranges(n, world)
            p2l = ranges[rank][2]
            local = oracle.nrmf(x, p2_min=p2l) if p2l > 0 else None
            vals = [None] * world
            td.all_gather_object(vals, None if local is None else float(local))
            comb = oracle.combine_ranks([None if v is None else dt(v) for v in vals])
            res.append(np.asarray(comb, dtype=dt).tobytes())
        # NCCL unique-id bootstrap: rank 0 creates, everyone receives the same bytes
        idbuf = ctypes.create_string_buffer(128)
        if rank == 0:
            assert nrmf.lib().nrmf_nccl_unique_id(idbuf) == 0
        obj = [bytes(idbuf.raw)]
        td.broadcast_object_list(obj, src=0)
        ids = [None] * world
        td.all_gather_object(ids, obj[0])
        q.put((rank, res, len(set(ids)) == 1 and len(ids[0]) == 128))
    finally:
        td.destroy_process_group()


CASES = [(1, "f64", False), (4097, "f64", False), (5 * 4096 + 3, "f32", False), (40000, "f64", True),
         (17 * 4096 - 3, "f32", True), (300 * 4096 + 11, "f64", False)]


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_combine_equals_global(world):
    import nrmf_inputs as gen
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for (n, dt_name, nan_last), k in zip(CASES, range(len(CASES))):
        dt = np.float64 if dt_name == "f64" else np.float32
        x = gen.normal(7, n, 0, dtype=dt)
        if nan_last:
            x[-1] = np.nan
        exp = np.asarray(oracle.nrmf(x), dtype=dt).tobytes()
        got = {o[1][k] for o in out}
        assert got == {exp}, (n, dt_name)
    assert all(o[2] for o in out)


def _cols_worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import nrmf_inputs as gen
        import oracle
        import paper_2509_06220_b200 as nrmf
        res = []
        for (r, c, dt_name) in cases:
            dt = np.float64 if dt_name == "f64" else np.float32
            off, cnt = nrmf.cols_shard(c, world, rank)      # C partition (libnrmf.so)
            # each rank generates its own block (index-addressable generator)
            A = gen.normal(11, r * cnt, r * off, dtype=dt)
            ranges = oracle.cols_shard_ranges(c, world)
            p2l = ranges[rank][2]
            local = None
            if p2l > 0:
                col, _ = oracle.cols(A, r, cnt, r) if cnt > 0 else (np.zeros(0, dtype=dt), None)
                pad = np.zeros(p2l, dtype=dt)
                pad[:cnt] = col
                local = float(oracle.combine(pad))
            vals = [None] * world
            td.all_gather_object(vals, local)
            comb = oracle.combine_ranks([None if v is None else dt(v) for v in vals])
            res.append(np.asarray(comb, dtype=dt).tobytes())
        q.put((rank, res))
    finally:
        td.destroy_process_group()


COLS_CASES = [(4096, 9, "f64"), (100, 5, "f32"), (5000, 3, "f64"), (7, 64, "f32")]


@pytest.mark.parametrize("world", [2, 4])
def test_cols_block_sharding_combine_equals_global(world):
    """Column blocks over real processes (gloo): per-rank Frobenius subtrees of
    the canonical blocks, one scalar each, the rank tree == the one-process
    Frobenius norm bitwise."""
    import nrmf_inputs as gen
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cols_worker, args=(r, world, port, COLS_CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, (r, c, dt_name) in enumerate(COLS_CASES):
        dt = np.float64 if dt_name == "f64" else np.float32
        A = gen.normal(11, r * c, 0, dtype=dt)
        _, efr = oracle.cols(A, r, c, r)
        exp = np.asarray(efr, dtype=dt).tobytes()
        assert {o[1][k] for o in out} == {exp}, (r, c, dt_name)
