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
import torch
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
