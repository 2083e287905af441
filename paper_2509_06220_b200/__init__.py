"""paper_2509_06220_b200 -- B200-native xNRMF (arXiv 2509.06220).

Thin Python binding over the C ABI in ``include/nrmf.h`` (``libnrmf.so``,
hand-written sm_100a CUDA).  This module only marshals arguments: every step
of the norm runs in the library's kernels.  PyTorch provides device memory,
streams and process groups.  There is no CPU fallback: if ``libnrmf.so`` is
missing or a call fails, an exception is raised.

    norm(x)                 ||x||_F of a contiguous fp32/fp64 tensor (CUDA, or
                            host memory streamed through the GPU)
    norm_complex(z)         ||z||_F of a complex64/complex128 tensor
    cols(A)                 (column norms, Frobenius norm) of a column-major matrix
    dist(x_local, n_global) ||x||_F of an array sharded over torch.distributed ranks
    dist_p2p(x_local, n_global, pg)  the same, rank exchange fused into the tree kernel
    dist_local / rank_combine  the two halves of dist (no communication)
    shard(n_global, world, rank) -> (offset, count) canonical shard
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnrmf.so")

NRMF_OK = 0
NRMF_TOP_CR = 1   # include/nrmf.h: cr_hypot above the tile level (A-style final reduction)
NRMF_WS_CLEAN = 2  # include/nrmf.h: the workspace's counters are known to be zero (no memset)
_lib = None
_lock = threading.Lock()


def _load():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libnrmf.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
        L.nrmf_status_str.argtypes = [i32]; L.nrmf_status_str.restype = ctypes.c_char_p
        L.nrmf_tree_version.argtypes = []; L.nrmf_tree_version.restype = i32
        L.nrmf_tree_params.argtypes = [i32, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.nrmf_workspace_bytes.argtypes = [i64, i32]; L.nrmf_workspace_bytes.restype = sz
        L.nrmf_cols_workspace_bytes.argtypes = [i64, i64, i32]; L.nrmf_cols_workspace_bytes.restype = sz
        L.nrmf_host_workspace_bytes.argtypes = [i64, i32]; L.nrmf_host_workspace_bytes.restype = sz
        L.nrmf_dist_workspace_bytes.argtypes = [i64, i32, i32]; L.nrmf_dist_workspace_bytes.restype = sz
        for f in ("nrmf_d", "nrmf_s", "nrmf_z_d", "nrmf_z_s", "nrmf_host_d", "nrmf_host_s"):
            getattr(L, f).argtypes = [i64, vp, vp, vp, sz, vp]
            getattr(L, f).restype = i32
        for f in ("nrmf_ex_d", "nrmf_ex_s", "nrmf_host_ex_d", "nrmf_host_ex_s"):
            getattr(L, f).argtypes = [i64, vp, vp, i32, vp, sz, vp]
            getattr(L, f).restype = i32
        for f in ("nrmf_cols_ex_d", "nrmf_cols_ex_s"):
            getattr(L, f).argtypes = [i64, i64, i64, vp, vp, vp, i32, vp, sz, vp]
            getattr(L, f).restype = i32
        for f in ("nrmf_dist_ex_d", "nrmf_dist_ex_s"):
            getattr(L, f).argtypes = [i64, i64, i64, vp, vp, i32, vp, sz, vp, vp]
            getattr(L, f).restype = i32
        for f in ("nrmf_cols_d", "nrmf_cols_s"):
            getattr(L, f).argtypes = [i64, i64, i64, vp, vp, vp, vp, sz, vp]
            getattr(L, f).restype = i32
        for f in ("nrmf_dist_d", "nrmf_dist_s"):
            getattr(L, f).argtypes = [i64, i64, i64, vp, vp, vp, sz, vp, vp]
            getattr(L, f).restype = i32
        for f in ("nrmf_dist_local_d", "nrmf_dist_local_s"):
            getattr(L, f).argtypes = [i64, i32, i32, i64, i64, vp, vp, i32, vp, sz, vp]
            getattr(L, f).restype = i32
        for f in ("nrmf_rank_combine_d", "nrmf_rank_combine_s"):
            getattr(L, f).argtypes = [i64, i32, vp, vp, i32, vp]
            getattr(L, f).restype = i32
        L.nrmf_dist_shard.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.nrmf_dist_shard.restype = i32
        L.nrmf_p2p_buffer_bytes.argtypes = []; L.nrmf_p2p_buffer_bytes.restype = sz
        L.nrmf_p2p_alloc.argtypes = [ctypes.POINTER(vp)]; L.nrmf_p2p_alloc.restype = i32
        L.nrmf_p2p_free.argtypes = [vp]; L.nrmf_p2p_free.restype = i32
        L.nrmf_p2p_ipc_handle.argtypes = [vp, ctypes.c_char_p]; L.nrmf_p2p_ipc_handle.restype = i32
        L.nrmf_p2p_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]; L.nrmf_p2p_open.restype = i32
        L.nrmf_p2p_close.argtypes = [vp]; L.nrmf_p2p_close.restype = i32
        for f in ("nrmf_dist_p2p_d", "nrmf_dist_p2p_s"):
            getattr(L, f).argtypes = [i64, i64, i64, vp, vp, i32, vp, sz, vp, i32, i32, vp, vp]
            getattr(L, f).restype = i32
        for f in ("nrmf_debug_p2p_emulate_d", "nrmf_debug_p2p_emulate_s"):
            getattr(L, f).argtypes = [i32, vp, vp, i32, vp, vp]
            getattr(L, f).restype = i32
        L.nrmf_cols_dist_shard.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.nrmf_cols_dist_shard.restype = i32
        L.nrmf_cols_dist_workspace_bytes.argtypes = [i64, i64, i32, i32]
        L.nrmf_cols_dist_workspace_bytes.restype = sz
        for f in ("nrmf_cols_dist_d", "nrmf_cols_dist_s"):
            getattr(L, f).argtypes = [i64, i64, i64, i64, i64, vp, vp, vp, i32, vp, sz, vp, vp]
            getattr(L, f).restype = i32
        L.nrmf_nccl_unique_id.argtypes = [ctypes.c_char_p]; L.nrmf_nccl_unique_id.restype = i32
        L.nrmf_nccl_comm_init.argtypes = [i32, i32, ctypes.c_char_p, ctypes.POINTER(vp)]
        L.nrmf_nccl_comm_init.restype = i32
        L.nrmf_nccl_comm_destroy.argtypes = [vp]; L.nrmf_nccl_comm_destroy.restype = i32
        L.nrmf_debug_set_grid.argtypes = [i32]; L.nrmf_debug_set_grid.restype = i32
        _lib = L
    return _lib


def lib():
    """The loaded ctypes library (raises if it is not built)."""
    return _load()


def _check(status: int, what: str):
    if status != NRMF_OK:
        raise RuntimeError(f"{what}: {_load().nrmf_status_str(status).decode()}")


def tree_version() -> int:
    return _load().nrmf_tree_version()


def tree_params(dtype) -> tuple[int, int, int]:
    esz = torch.empty(0, dtype=dtype).element_size()
    a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(_load().nrmf_tree_params(esz, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "tree_params")
    return a.value, b.value, c.value


# --------------------------------------------------------------- workspaces
# Cached per (device, stream, kind).  The library clears the arrival counters
# it uses on every call, so the initial contents do not matter.  While
# capture() records a graph, calls draw from that capture's own arena instead:
# the graph keeps its workspaces alive (g._nrmf_ws) and shares them with no
# other graph or direct call.
_ws_cache: dict = {}
_arena = threading.local()


def _workspace(nbytes: int, device: torch.device, stream: torch.cuda.Stream, kind: str) -> torch.Tensor:
    arena = getattr(_arena, "tensors", None)
    if arena is not None:
        # the n-th workspace of this kind requested by the captured call (the
        # warm-up runs and the captured run make the same requests in order)
        i = _arena.counts.get((device.index, kind), 0)
        _arena.counts[(device.index, kind)] = i + 1
        key = (device.index, kind, i)
        t = arena.get(key)
        if t is None or t.numel() < nbytes:
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError("nrmf.capture: the captured call requested a workspace its warm-up did not")
            t = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
            arena[key] = t
        return t
    key = (device.index, stream.cuda_stream, kind)
    t = _ws_cache.get(key)
    if t is None or t.numel() < nbytes:
        t = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def clear_workspaces():
    """Drop the cached workspaces of direct calls (captured graphs own theirs)."""
    _ws_cache.clear()


def _flags(top: str) -> int:
    """Flags of a call: the top-level hypot, and NRMF_WS_CLEAN inside capture():
    a captured call's arena workspaces are zero-filled once and used only by
    that call (its warm-up runs and the graph's replays), so the library may
    skip the per-call counter memset -- the captured call is one kernel."""
    if top == "v1":
        f = 0
    elif top == "cr":
        f = NRMF_TOP_CR
    else:
        raise ValueError(f"nrmf: top must be 'v1' or 'cr', got {top!r}")
    if getattr(_arena, "tensors", None) is not None:
        f |= NRMF_WS_CLEAN
    return f


def _elem(dtype) -> tuple[int, str]:
    if dtype == torch.float64:
        return 8, "d"
    if dtype == torch.float32:
        return 4, "s"
    raise ValueError(f"nrmf: unsupported dtype {dtype} (float32/float64 only)")


# --------------------------------------------------------------- public API
def norm(x: torch.Tensor, out: torch.Tensor | None = None, top: str = "v1") -> torch.Tensor:
    """||x||_F by the xNRMF tree (bitwise reproducible).

    CUDA tensor: enqueued on the current stream, returns a 0-d CUDA tensor.
    CPU tensor (pin it for copy/compute overlap): streamed through the current
    CUDA device; synchronizes and returns a 0-d CPU tensor.
    top="cr": correctly rounded hypot above the tile level (NRMF_TOP_CR)."""
    fl = _flags(top)
    if not x.is_contiguous():
        raise ValueError("nrmf.norm: tensor must be contiguous")
    esz, c = _elem(x.dtype)
    L = _load()
    n = x.numel()
    if x.is_cuda:
        dev = x.device
        with torch.cuda.device(dev):
            s = torch.cuda.current_stream(dev)
            if out is None:
                out = torch.empty((), dtype=x.dtype, device=dev)
            ws = _workspace(L.nrmf_workspace_bytes(n, esz), dev, s, "vec")
            f = L.nrmf_ex_d if c == "d" else L.nrmf_ex_s
            _check(f(n, x.data_ptr() if n else None, out.data_ptr(), fl, ws.data_ptr(), ws.numel(),
                     s.cuda_stream), "nrmf.norm")
        return out
    # host input
    dev = torch.device("cuda", torch.cuda.current_device())
    s = torch.cuda.current_stream(dev)
    if out is None:
        out = torch.empty((), dtype=x.dtype).pin_memory()
    ws = _workspace(L.nrmf_host_workspace_bytes(n, esz), dev, s, "host")
    f = L.nrmf_host_ex_d if c == "d" else L.nrmf_host_ex_s
    _check(f(n, x.data_ptr() if n else None, out.data_ptr(), fl, ws.data_ptr(), ws.numel(), s.cuda_stream),
           "nrmf.norm(host)")
    s.synchronize()
    return out


def norm_complex(z: torch.Tensor) -> torch.Tensor:
    """||z||_F of a complex tensor = the real norm of its 2*numel interleaved
    parts (e:F); bitwise equal to norm(torch.view_as_real(z))."""
    if not z.is_complex():
        raise ValueError("nrmf.norm_complex: complex tensor expected")
    if not z.is_contiguous():
        raise ValueError("nrmf.norm_complex: tensor must be contiguous")
    zr = torch.view_as_real(z)
    if not z.is_cuda:
        return norm(zr.reshape(-1))
    esz, c = _elem(zr.dtype)
    L = _load()
    dev = z.device
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev)
        out = torch.empty((), dtype=zr.dtype, device=dev)
        ws = _workspace(L.nrmf_workspace_bytes(2 * z.numel(), esz), dev, s, "vec")
        f = L.nrmf_z_d if c == "d" else L.nrmf_z_s
        _check(f(z.numel(), zr.data_ptr() if z.numel() else None, out.data_ptr(), ws.data_ptr(),
                 ws.numel(), s.cuda_stream), "nrmf.norm_complex")
    return out


def cols(A: torch.Tensor, frob: bool = True, top: str = "v1"):
    """Column norms and Frobenius norm of a column-major CUDA matrix
    (A.stride(0) == 1, ld = A.stride(1)); e.g. ``B.t()`` of a row-major B."""
    fl = _flags(top)
    if A.dim() != 2:
        raise ValueError("nrmf.cols: 2-D tensor expected")
    r, c = A.shape
    if not A.is_cuda:
        raise ValueError("nrmf.cols: CUDA tensor expected")
    if r > 1 and A.stride(0) != 1:
        raise ValueError("nrmf.cols: column-major storage expected (stride(0) == 1)")
    ld = A.stride(1) if c > 1 else max(r, 1)
    if c > 1 and ld < r:
        raise ValueError("nrmf.cols: leading dimension smaller than rows")
    esz, ch = _elem(A.dtype)
    L = _load()
    dev = A.device
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev)
        col = torch.empty(c, dtype=A.dtype, device=dev)
        fr = torch.empty((), dtype=A.dtype, device=dev) if frob else None
        ws = _workspace(L.nrmf_cols_workspace_bytes(r, c, esz), dev, s, "cols")
        f = L.nrmf_cols_ex_d if ch == "d" else L.nrmf_cols_ex_s
        _check(f(r, c, ld, A.data_ptr() if A.numel() else None, col.data_ptr() if c else None,
                 fr.data_ptr() if fr is not None else None, fl, ws.data_ptr(), ws.numel(), s.cuda_stream),
               "nrmf.cols")
    return (col, fr) if frob else col


def shard(n_global: int, world: int, rank: int) -> tuple[int, int]:
    """Canonical contiguous shard (offset, count) of `rank` (nrmf_dist_shard)."""
    off, cnt = ctypes.c_int64(), ctypes.c_int64()
    _check(_load().nrmf_dist_shard(n_global, world, rank, ctypes.byref(off), ctypes.byref(cnt)),
           "nrmf.shard")
    return off.value, cnt.value


class Comm:
    """An NCCL communicator owned by the library, bootstrapped through a
    torch.distributed process group (the 128-byte unique id is broadcast with
    the group's own backend)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        L = _load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        idbuf = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(L.nrmf_nccl_unique_id(idbuf), "nccl unique id")
        obj = [bytes(idbuf.raw)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        h = ctypes.c_void_p()
        _check(L.nrmf_nccl_comm_init(self.world, self.rank, ctypes.c_char_p(obj[0]), ctypes.byref(h)),
               "nccl comm init")
        self.handle = h

    def close(self):
        if self.handle:
            _load().nrmf_nccl_comm_destroy(self.handle)
            self.handle = None
        for k, v in list(_comms.items()):
            if v is self:
                del _comms[k]


_comms: dict = {}


def comm_for(group=None) -> Comm:
    key = (id(group), torch.cuda.current_device())
    c = _comms.get(key)
    if c is None or not c.handle:
        c = Comm(group)
        _comms[key] = c
    return c


def dist(x_local: torch.Tensor, n_global: int, group=None, comm: Comm | None = None,
         out: torch.Tensor | None = None, top: str = "v1") -> torch.Tensor:
    """||x||_F of an array of n_global elements sharded canonically over the
    ranks of `group` (x_local = this rank's shard, see shard()).  Collective;
    returns the same 0-d CUDA tensor bits on every rank."""
    if not x_local.is_cuda or not x_local.is_contiguous():
        raise ValueError("nrmf.dist: contiguous CUDA tensor expected")
    esz, c = _elem(x_local.dtype)
    fl = _flags(top)
    comm = comm or comm_for(group)
    off, cnt = shard(n_global, comm.world, comm.rank)
    if x_local.numel() != cnt:
        raise ValueError(f"nrmf.dist: rank {comm.rank} expects {cnt} elements, got {x_local.numel()}")
    L = _load()
    dev = x_local.device
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev)
        if out is None:
            out = torch.empty((), dtype=x_local.dtype, device=dev)
        ws = _workspace(L.nrmf_dist_workspace_bytes(n_global, comm.world, esz), dev, s, "dist")
        f = L.nrmf_dist_ex_d if c == "d" else L.nrmf_dist_ex_s
        _check(f(n_global, off, cnt, x_local.data_ptr() if cnt else None, out.data_ptr(), fl, ws.data_ptr(),
                 ws.numel(), comm.handle, s.cuda_stream), "nrmf.dist")
    return out


def dist_local(x_local: torch.Tensor, n_global: int, world: int, rank: int, out: torch.Tensor | None = None,
               top: str = "v1") -> torch.Tensor:
    """The value of `rank`'s aligned subtree of the n_global-element tree
    (x_local = its canonical shard, see shard()): the local half of dist(),
    nrmf_dist_local_[ds].  No communication."""
    if not x_local.is_cuda or not x_local.is_contiguous():
        raise ValueError("nrmf.dist_local: contiguous CUDA tensor expected")
    esz, c = _elem(x_local.dtype)
    fl = _flags(top)
    off, cnt = shard(n_global, world, rank)
    if x_local.numel() != cnt:
        raise ValueError(f"nrmf.dist_local: rank {rank} expects {cnt} elements, got {x_local.numel()}")
    L = _load()
    dev = x_local.device
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev)
        if out is None:
            out = torch.empty((), dtype=x_local.dtype, device=dev)
        ws = _workspace(L.nrmf_dist_workspace_bytes(n_global, world, esz), dev, s, "dist")
        f = L.nrmf_dist_local_d if c == "d" else L.nrmf_dist_local_s
        _check(f(n_global, world, rank, off, cnt, x_local.data_ptr() if cnt else None, out.data_ptr(), fl,
                 ws.data_ptr(), ws.numel(), s.cuda_stream), "nrmf.dist_local")
    return out


def rank_combine(values: torch.Tensor, n_global: int, world: int, out: torch.Tensor | None = None,
                 top: str = "v1") -> torch.Tensor:
    """The rank tree over the ranks' dist_local values (a CUDA vector in rank
    order, at least min(world, P2) entries): nrmf_rank_combine_[ds]."""
    if not values.is_cuda or not values.is_contiguous():
        raise ValueError("nrmf.rank_combine: contiguous CUDA tensor expected")
    esz, c = _elem(values.dtype)
    fl = _flags(top)
    L = _load()
    dev = values.device
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev)
        if out is None:
            out = torch.empty((), dtype=values.dtype, device=dev)
        f = L.nrmf_rank_combine_d if c == "d" else L.nrmf_rank_combine_s
        _check(f(n_global, world, values.data_ptr(), out.data_ptr(), fl, s.cuda_stream), "nrmf.rank_combine")
    return out


class P2PGroup:
    """Peer-memory rank exchange for dist_p2p: allocates this rank's
    exchange buffer, all-gathers the CUDA IPC handles through the
    torch.distributed group, maps every peer's buffer and keeps the device
    array of peer pointers.  One per (group, device); every rank must make the
    same sequence of dist_p2p calls on it (the call counter lives in the
    buffer, so calls may be captured in CUDA graphs)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        L = _load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > 32:
            raise ValueError("nrmf.P2PGroup: at most 32 ranks")
        dev = torch.device("cuda", torch.cuda.current_device())
        buf = ctypes.c_void_p()
        _check(L.nrmf_p2p_alloc(ctypes.byref(buf)), "nrmf_p2p_alloc")
        self.buf = buf
        h = ctypes.create_string_buffer(64)
        _check(L.nrmf_p2p_ipc_handle(buf, h), "nrmf_p2p_ipc_handle")
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        self._opened = []
        ptrs = []
        failed = None
        for r in range(self.world):
            if r == self.rank:
                ptrs.append(buf.value)
                continue
            p = ctypes.c_void_p()
            st = L.nrmf_p2p_open(ctypes.c_char_p(handles[r]), ctypes.byref(p))
            if st != NRMF_OK:
                failed = f"rank {self.rank} cannot map rank {r}'s buffer: {L.nrmf_status_str(st).decode()}"
                break
            self._opened.append(p)
            ptrs.append(p.value)
        # every rank learns whether every rank mapped every peer (this is also
        # the barrier: every buffer is mapped before the first exchange)
        status = [None] * self.world
        dist.all_gather_object(status, failed, group=group)
        bad = [m for m in status if m]
        if bad:
            self.close()
            raise RuntimeError("nrmf.P2PGroup: " + "; ".join(bad))
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)

    def close(self):
        L = _load()
        for p in self._opened:
            L.nrmf_p2p_close(p)
        self._opened = []
        if self.buf:
            L.nrmf_p2p_free(self.buf)
            self.buf = None


def dist_p2p(x_local: torch.Tensor, n_global: int, pg: P2PGroup, out: torch.Tensor | None = None,
             top: str = "v1") -> torch.Tensor:
    """As dist(), with the rank values exchanged through peer memory (one
    kernel, no NCCL).  Collective over pg's ranks; same bits on every rank and
    as norm() of the whole array on one GPU.  pg.err turns 1 if an exchange
    timed out (the result is then NaN)."""
    if not x_local.is_cuda or not x_local.is_contiguous():
        raise ValueError("nrmf.dist_p2p: contiguous CUDA tensor expected")
    esz, c = _elem(x_local.dtype)
    fl = _flags(top)
    off, cnt = shard(n_global, pg.world, pg.rank)
    if x_local.numel() != cnt:
        raise ValueError(f"nrmf.dist_p2p: rank {pg.rank} expects {cnt} elements, got {x_local.numel()}")
    L = _load()
    dev = x_local.device
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev)
        if out is None:
            out = torch.empty((), dtype=x_local.dtype, device=dev)
        ws = _workspace(L.nrmf_dist_workspace_bytes(n_global, pg.world, esz), dev, s, "dist")
        f = L.nrmf_dist_p2p_d if c == "d" else L.nrmf_dist_p2p_s
        _check(f(n_global, off, cnt, x_local.data_ptr() if cnt else None, out.data_ptr(), fl, ws.data_ptr(),
                 ws.numel(), pg.peers.data_ptr(), pg.world, pg.rank, pg.err.data_ptr(),
                 s.cuda_stream), "nrmf.dist_p2p")
    return out


def _debug_p2p_emulate(values: torch.Tensor, bufs: torch.Tensor, top: str = "v1") -> torch.Tensor:
    """Test hook: len(values) ranks emulated as the CTAs of one cooperative
    launch on this GPU (bufs: device int64 array of their zeroed buffers)."""
    esz, c = _elem(values.dtype)
    outs = torch.empty_like(values)
    f = _load().nrmf_debug_p2p_emulate_d if c == "d" else _load().nrmf_debug_p2p_emulate_s
    _check(f(values.numel(), values.data_ptr(), bufs.data_ptr(), _flags(top), outs.data_ptr(),
             torch.cuda.current_stream().cuda_stream), "nrmf p2p emulate")
    return outs


def cols_shard(cols_global: int, world: int, rank: int) -> tuple[int, int]:
    """Canonical column block (col_offset, col_count) of `rank` (nrmf_cols_dist_shard)."""
    off, cnt = ctypes.c_int64(), ctypes.c_int64()
    _check(_load().nrmf_cols_dist_shard(cols_global, world, rank, ctypes.byref(off), ctypes.byref(cnt)),
           "nrmf.cols_shard")
    return off.value, cnt.value


def cols_dist(A_local: torch.Tensor, cols_global: int, group=None, comm: Comm | None = None,
              frob: bool = True, top: str = "v1"):
    """Column norms of this rank's canonical column block (A_local: rows x
    col_count, column-major, see cols_shard) and -- collectively, when frob --
    the Frobenius norm of the whole sharded matrix, the same bits on every rank
    and as cols() on one GPU."""
    if A_local.dim() != 2 or not A_local.is_cuda:
        raise ValueError("nrmf.cols_dist: 2-D CUDA tensor expected")
    r, c = A_local.shape
    if r > 1 and c > 0 and A_local.stride(0) != 1:
        raise ValueError("nrmf.cols_dist: column-major storage expected (stride(0) == 1)")
    ld = A_local.stride(1) if c > 1 else max(r, 1)
    esz, ch = _elem(A_local.dtype)
    fl = _flags(top)
    comm = comm or comm_for(group)
    off, cnt = cols_shard(cols_global, comm.world, comm.rank)
    if c != cnt:
        raise ValueError(f"nrmf.cols_dist: rank {comm.rank} expects {cnt} columns, got {c}")
    L = _load()
    dev = A_local.device
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev)
        col = torch.empty(c, dtype=A_local.dtype, device=dev)
        fr = torch.empty((), dtype=A_local.dtype, device=dev) if frob else None
        ws = _workspace(L.nrmf_cols_dist_workspace_bytes(r, cols_global, comm.world, esz), dev, s, "colsdist")
        f = L.nrmf_cols_dist_d if ch == "d" else L.nrmf_cols_dist_s
        _check(f(r, cols_global, ld, off, cnt, A_local.data_ptr() if A_local.numel() else None,
                 col.data_ptr() if c else None, fr.data_ptr() if fr is not None else None, fl, ws.data_ptr(),
                 ws.numel(), comm.handle, s.cuda_stream), "nrmf.cols_dist")
    return (col, fr) if frob else col


def capture(fn, warmup: int = 1, graph: "torch.cuda.CUDAGraph | None" = None) -> "torch.cuda.CUDAGraph":
    """Capture one stream-ordered nrmf call (``norm`` / ``cols`` / ``dist`` on
    fixed tensors, e.g. ``lambda: nrmf.dist(x, n, comm=c, out=o)``) in a CUDA
    graph; ``g.replay()`` then re-runs its launches -- counter memset, tree
    kernel, and for ``dist`` the NCCL allgather and the rank-tree kernel --
    with one launch.  The call is first run ``warmup`` times on
    the capture stream with workspaces from an arena of its own, which the
    capture reuses and the returned graph keeps alive (``g._nrmf_ws``): no
    other graph or direct call shares them, and clear_workspaces() does not
    free them.  Captured calls pass NRMF_WS_CLEAN (the arena is zero-filled
    and dedicated), so a captured norm/cols/dist_p2p call is ONE kernel node.
    Replays give the same bits as direct calls (tested); replays of one graph
    must not overlap each other.  `graph`: a CUDAGraph to capture into (e.g.
    with debug mode enabled)."""
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    arena: dict = {}
    prev = getattr(_arena, "tensors", None), getattr(_arena, "counts", None)
    try:
        _arena.tensors = arena
        with torch.cuda.stream(cs):
            for _ in range(max(1, warmup)):
                _arena.counts = {}
                fn()
        torch.cuda.current_stream().wait_stream(cs)
        g = graph if graph is not None else torch.cuda.CUDAGraph()
        _arena.counts = {}
        with torch.cuda.graph(g, stream=cs):
            fn()
    finally:
        _arena.tensors, _arena.counts = prev
    g._nrmf_ws = list(arena.values())
    return g


def _debug_set_grid(grid: int):
    """Test hook: force the persistent grid size (0 = automatic)."""
    _load().nrmf_debug_set_grid(grid)


def _debug_set_g0(g0: int):
    """Test hook: force the warp-group level count g0 in 0..3 (-1 = automatic)."""
    L = _load()
    L.nrmf_debug_set_g0.argtypes = [ctypes.c_int]
    L.nrmf_debug_set_g0(g0)


def _debug_set_gap_stream(on: bool):
    """Test hook: gapped column blocks (ld > rows, rows % 4096 == 0) on the stream kernel (default on)."""
    L = _load()
    L.nrmf_debug_set_gap_stream.argtypes = [ctypes.c_int]
    L.nrmf_debug_set_gap_stream(1 if on else 0)


def _debug_set_unal_stream(on: bool):
    """Test hook: unaligned vectors on the stream kernel (default on) or the element-load kernel."""
    L = _load()
    L.nrmf_debug_set_unal_stream.argtypes = [ctypes.c_int]
    L.nrmf_debug_set_unal_stream(1 if on else 0)


def _debug_set_split_ll(on: bool):
    """Test hook: the split kernel's last combine step by flag-in-data slots (default on) or a counter."""
    L = _load()
    L.nrmf_debug_set_split_ll.argtypes = [ctypes.c_int]
    L.nrmf_debug_set_split_ll(1 if on else 0)


def _debug_set_cta_step(on: bool):
    """Test hook: the stream kernel's first combine step in shared memory (default on)."""
    L = _load()
    L.nrmf_debug_set_cta_step.argtypes = [ctypes.c_int]
    L.nrmf_debug_set_cta_step(1 if on else 0)


def build(force: bool = False) -> str:
    return _build.build(force=force)
