// nrmf_dist.cu -- the rank level of the tree (a6 of DESIGN.md §8).
//
// e:hr: the norms of two disjoint parts combine by one hypot; the
// paper's §5 suggests contiguous chunks per worker with hypot as
// the reduction but warns that an unspecified reduction order breaks
// reproducibility.  Here the order is fixed: every rank owns an aligned
// subtree of the one global tile tree, reduces it locally (the same kernel as
// nrmf_d), exchanges ONE scalar with ncclAllGather (NCCL has no user-defined
// reduction and summing squares would reintroduce the overflow the method
// avoids), and evaluates the top lg(world) levels itself.  Every rank gets the
// same bits, equal to the 1-GPU result.
//
// NCCL is loaded with dlopen("libnccl.so.2") so that the process uses the
// NCCL it already has (torch's) and libnrmf.so has no link-time dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/nrmf.h"
#include "nrmf_internal.h"
#include "nrmf_p2p.cuh"

namespace nrmf {
namespace {

constexpr int64_t kTileE = 4096;
constexpr uintptr_t kWsAlign = 16;  // nrmf.h: workspaces are 16-byte aligned

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) =
      nullptr;
  bool ok = false;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi* nccl() {
  std::call_once(g_nccl_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return;
    g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    g_nccl.CommCount = reinterpret_cast<decltype(g_nccl.CommCount)>(dlsym(h, "ncclCommCount"));
    g_nccl.CommUserRank = reinterpret_cast<decltype(g_nccl.CommUserRank)>(dlsym(h, "ncclCommUserRank"));
    g_nccl.AllGather = reinterpret_cast<decltype(g_nccl.AllGather)>(dlsym(h, "ncclAllGather"));
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.CommCount &&
                g_nccl.CommUserRank && g_nccl.AllGather;
  });
  return g_nccl.ok ? &g_nccl : nullptr;
}

int64_t pow2_ceil(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}
bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Canonical shard (nrmf.h): returns local subtree size p2_local (0 = none).
int64_t shard(int64_t n, int world, int rank, int64_t* off, int64_t* cnt) {
  const int64_t nt = (n + kTileE - 1) / kTileE;
  const int64_t P2 = pow2_ceil(std::max<int64_t>(nt, 1));
  int64_t t0, t1, p2l;
  if (world <= P2) {
    const int64_t per = P2 / world;
    t0 = rank * per;
    t1 = t0 + per;
    p2l = per;
  } else if (rank < P2) {
    t0 = rank;
    t1 = rank + 1;
    p2l = 1;
  } else {
    t0 = t1 = P2;
    p2l = 0;
  }
  const int64_t a = std::min(t0 * kTileE, n), b = std::min(t1 * kTileE, n);
  *off = a;
  *cnt = b - a;
  return p2l;
}

// Canonical aligned partition of P2 = pow2 >= units leaves (tiles or columns)
// over world ranks: [t0, t1) and the local subtree size (0 = none).
int64_t shard_units(int64_t units, int world, int rank, int64_t* t0, int64_t* t1) {
  const int64_t P2 = pow2_ceil(std::max<int64_t>(units, 1));
  if (world <= P2) {
    const int64_t per = P2 / world;
    *t0 = rank * per;
    *t1 = *t0 + per;
    return per;
  }
  if (rank < P2) {
    *t0 = rank;
    *t1 = rank + 1;
    return 1;
  }
  *t0 = *t1 = P2;
  return 0;
}

// workspace: [local tree ws][local value (256)][gathered (world entries)]
size_t dist_ws(int64_t n, int world, size_t esz) {
  const int64_t nt = (n + kTileE - 1) / kTileE;
  const int64_t P2 = pow2_ceil(std::max<int64_t>(nt, 1));
  const int64_t p2l = world <= P2 ? P2 / world : 1;
  return tree_workspace(p2l, esz) + 256 + align_up((size_t)world * esz, 256);
}

// The rank's step of the distributed tree (shared by nrmf_dist_local_[ds],
// nrmf_dist_[ds] and nrmf_dist_p2p_[ds], so all of them run the same kernels):
// validate the canonical shard, then reduce the rank's aligned subtree of the
// global tile tree (size p2l, +0 padded) into *local -- the same tree kernel
// as nrmf_[ds].  A rank that owns an all-padding subtree or none contributes +0.
// rx (nullable): the peer exchange fused into the tree kernel's root writer;
// *local then receives the rank tree's root (the global norm).
template <typename F>
__global__ void __launch_bounds__(32) p2p_exchange_kernel(const F* local, PeerArgs a, int nr, int cr, F* out);

template <typename F>
int local_step(int64_t n, int world, int rank, int64_t offset, int64_t count, const F* x, F* local, int flags,
               void* ws, size_t ws_bytes, cudaStream_t s, const RankExchange* rx) {
  if ((flags & ~(NRMF_TOP_CR | NRMF_WS_CLEAN)) != 0) return NRMF_EINVAL;
  const int cr = flags & NRMF_TOP_CR;
  if (local == nullptr || ws == nullptr || n < 0 || world < 1 || rank < 0 || rank >= world) return NRMF_EINVAL;
  if (count > 0 && x == nullptr) return NRMF_EINVAL;
  if (reinterpret_cast<uintptr_t>(x) % sizeof(F) || reinterpret_cast<uintptr_t>(local) % sizeof(F))
    return NRMF_EALIGN;
  if (reinterpret_cast<uintptr_t>(ws) % kWsAlign) return NRMF_EALIGN;
  if (!is_pow2(world)) return NRMF_ESHARD;
  int64_t off = 0, cnt = 0;
  const int64_t p2l = shard(n, world, rank, &off, &cnt);
  if (off != offset || cnt != count) return NRMF_ESHARD;
  if (ws_bytes < dist_ws(n, world, sizeof(F))) return NRMF_EWORKSPACE;
  const int64_t nt = (n + kTileE - 1) / kTileE;
  const int64_t P2 = pow2_ceil(std::max<int64_t>(nt, 1));
  const int64_t p2ws = world <= P2 ? P2 / world : 1;
  const size_t tws = tree_workspace(p2ws, sizeof(F));
  if (p2l > 0 && cnt > 0) return tree_eval<F>(cnt, x, p2l, local, ws, tws, s, flags, rx);
  // no data here: the subtree value is +0
  F* zero = reinterpret_cast<F*>(static_cast<char*>(ws) + tws);
  if (cudaMemsetAsync(rx ? zero : local, 0, sizeof(F), s) != cudaSuccess) return NRMF_ECUDA;
  if (rx == nullptr) return NRMF_OK;
  PeerArgs a{rx->peers, rx->world, rx->rank, rx->err};
  p2p_exchange_kernel<F><<<1, 32, 0, s>>>(zero, a, rx->nr, cr, local);
  return cudaGetLastError() == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
}

// The rank tree: the balanced tree over the values of the min(world, P2)
// ranks that own part of the tile tree, in rank order (e:hr; a FIXED order,
// P:1077-1084).
template <typename F>
int rank_combine(int64_t n, int world, const F* values, F* out, int flags, cudaStream_t s) {
  if ((flags & ~(NRMF_TOP_CR | NRMF_WS_CLEAN)) != 0) return NRMF_EINVAL;
  if (values == nullptr || out == nullptr || n < 0 || world < 1) return NRMF_EINVAL;
  if (reinterpret_cast<uintptr_t>(values) % sizeof(F) || reinterpret_cast<uintptr_t>(out) % sizeof(F))
    return NRMF_EALIGN;
  if (!is_pow2(world)) return NRMF_ESHARD;
  const int64_t nt = (n + kTileE - 1) / kTileE;
  const int64_t P2 = pow2_ceil(std::max<int64_t>(nt, 1));
  const int64_t nr = std::min<int64_t>(world, P2);
  return bal_eval<F>(values, nr, nr, out, s, flags & NRMF_TOP_CR);
}

template <typename F>
int dist_impl(int64_t n, int64_t offset, int64_t count, const F* x, F* out, void* ws,
              size_t ws_bytes, void* comm_v, void* stream, int flags) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const NcclApi* api = nccl();
  if (api == nullptr) return NRMF_ENCCL;
  if (comm_v == nullptr || out == nullptr || ws == nullptr || n < 0) return NRMF_EINVAL;
  ncclComm_t comm = static_cast<ncclComm_t>(comm_v);
  int world = 0, rank = 0;
  if (api->CommCount(comm, &world) != ncclSuccess || api->CommUserRank(comm, &rank) != ncclSuccess)
    return NRMF_ENCCL;
  if (reinterpret_cast<uintptr_t>(out) % sizeof(F)) return NRMF_EALIGN;
  if (!is_pow2(world)) return NRMF_ESHARD;
  const int64_t nt = (n + kTileE - 1) / kTileE;
  const int64_t P2 = pow2_ceil(std::max<int64_t>(nt, 1));
  const size_t tws = tree_workspace(world <= P2 ? P2 / world : 1, sizeof(F));
  char* p = static_cast<char*>(ws);
  F* local = reinterpret_cast<F*>(p + tws);
  F* gathered = reinterpret_cast<F*>(p + tws + 256);
  int st = local_step<F>(n, world, rank, offset, count, x, local, flags, ws, ws_bytes, s, nullptr);
  if (st != NRMF_OK) return st;
  const ncclDataType_t dt = sizeof(F) == 8 ? ncclFloat64 : ncclFloat32;
  if (api->AllGather(local, gathered, 1, dt, comm, s) != ncclSuccess) return NRMF_ENCCL;
  return rank_combine<F>(n, world, gathered, out, flags, s);
}

// ---------------------------------------------------------------- peer memory
// The rank level through peer memory (nrmf_p2p.cuh): one warp per rank.  Used
// on its own only by a rank without data (and by the emulation test); with
// data the exchange runs inside the tree kernel (write_root, nrmf.cu).
template <typename F>
__global__ void __launch_bounds__(32) p2p_exchange_kernel(const F* local, PeerArgs a, int nr, int cr, F* out) {
  const F v = rank_exchange<F>(*local, a, nr, cr);
  if (threadIdx.x == 0) *out = v;
}

// Test emulation of `world` ranks on one GPU as the CTAs of ONE cooperative
// launch (co-resident by construction): CTA r plays rank r with value
// values[r], every rank's buffer lives on this GPU.
template <typename F>
__global__ void __launch_bounds__(32) p2p_emulate_kernel(const F* values, PeerArgs a, int nr, int cr, F* outs) {
  PeerArgs b = a;
  b.rank = (int)blockIdx.x;
  const F v = rank_exchange<F>(values[blockIdx.x], b, nr, cr);
  if (threadIdx.x == 0) outs[blockIdx.x] = v;
}

template <typename F>
int dist_p2p_impl(int64_t n, int64_t offset, int64_t count, const F* x, F* out, int flags, void* ws,
                  size_t ws_bytes, const void* peers, int world, int rank, unsigned* err, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (peers == nullptr || out == nullptr || ws == nullptr || n < 0) return NRMF_EINVAL;
  if (world < 1 || world > kP2PMaxRanks || rank < 0 || rank >= world) return NRMF_EINVAL;
  const int64_t nt = (n + kTileE - 1) / kTileE;
  const int64_t P2 = pow2_ceil(std::max<int64_t>(nt, 1));
  RankExchange rx{static_cast<char* const*>(peers), err, world, rank, (int)std::min<int64_t>(world, P2)};
  return local_step<F>(n, world, rank, offset, count, x, out, flags, ws, ws_bytes, s, &rx);
}

template <typename F>
int p2p_emulate(int world, const F* values, const void* peers, int flags, F* outs, void* stream) {
  if (world < 1 || world > kP2PMaxRanks || !is_pow2(world) || !values || !peers || !outs) return NRMF_EINVAL;
  PeerArgs a{static_cast<char* const*>(peers), world, 0, nullptr};
  int nr = world;
  int cr = flags & NRMF_TOP_CR;
  void* args[] = {(void*)&values, (void*)&a, (void*)&nr, (void*)&cr, (void*)&outs};
  if (cudaLaunchCooperativeKernel((void*)p2p_emulate_kernel<F>, dim3(world), dim3(32), args, 0,
                                  static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return NRMF_ECUDA;
  return NRMF_OK;
}

// ---------------------------------------------------------------- columns
// Column blocks: rank r owns columns [t0, t1) of the canonical partition of
// the P2c = pow2 >= cols column leaves of the Frobenius tree; its column norms
// are local (each column lies on one rank), its block's Frobenius subtree
// (size P2c/world, padded with +0) is exchanged as one scalar, and every rank
// evaluates the top lg min(world, P2c) levels.
// workspace: [local cols ws][local value (256)][gathered (world entries)]
size_t cols_dist_ws(int64_t rows, int64_t cols, int world, size_t esz) {
  int64_t t0, t1;
  const int64_t p2l = std::max<int64_t>(shard_units(cols, world, 0, &t0, &t1), 1);
  const int64_t cl = std::max<int64_t>(std::min(t1, cols) - std::min(t0, cols), 1);
  return align_up(cols_workspace(rows, cl, p2l, esz), 256) + 256 + align_up((size_t)world * esz, 256);
}

template <typename F>
int cols_dist_impl(int64_t rows, int64_t cols, int64_t ld, int64_t col_off, int64_t col_cnt, const F* A,
                   F* col_norms, F* frob, int flags, void* ws, size_t ws_bytes, void* comm_v, void* stream) {
  if ((flags & ~(NRMF_TOP_CR | NRMF_WS_CLEAN)) != 0) return NRMF_EINVAL;
  const int cr = flags & NRMF_TOP_CR;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rows < 0 || cols < 0 || ld < rows || col_off < 0 || col_cnt < 0) return NRMF_EINVAL;
  if (comm_v == nullptr || ws == nullptr) return NRMF_EINVAL;
  const NcclApi* api = nccl();
  if (api == nullptr) return NRMF_ENCCL;
  ncclComm_t comm = static_cast<ncclComm_t>(comm_v);
  int world = 0, rank = 0;
  if (api->CommCount(comm, &world) != ncclSuccess || api->CommUserRank(comm, &rank) != ncclSuccess)
    return NRMF_ENCCL;
  if (!is_pow2(world)) return NRMF_ESHARD;
  int64_t t0, t1;
  const int64_t p2l = shard_units(cols, world, rank, &t0, &t1);
  const int64_t a = std::min(t0, cols), b = std::min(t1, cols);
  if (col_off != a || col_cnt != b - a) return NRMF_ESHARD;
  if (ws_bytes < cols_dist_ws(rows, cols, world, sizeof(F))) return NRMF_EWORKSPACE;
  char* p = static_cast<char*>(ws);
  const size_t lws = align_up(cols_workspace(rows, std::max<int64_t>(col_cnt, 1), std::max<int64_t>(p2l, 1),
                                             sizeof(F)), 256);
  F* local = reinterpret_cast<F*>(p + lws);
  F* gathered = reinterpret_cast<F*>(p + lws + 256);
  int st = NRMF_OK;
  if (col_cnt > 0) {
    st = cols_eval<F>(rows, col_cnt, ld, A, col_norms, frob != nullptr ? local : nullptr, p2l, flags, ws, lws, s);
  } else if (frob != nullptr && cudaMemsetAsync(local, 0, sizeof(F), s) != cudaSuccess) {
    st = NRMF_ECUDA;  // no columns here: an all-padding subtree (value +0)
  }
  if (st != NRMF_OK || frob == nullptr) return st;
  if (reinterpret_cast<uintptr_t>(frob) % sizeof(F)) return NRMF_EALIGN;
  const ncclDataType_t dt = sizeof(F) == 8 ? ncclFloat64 : ncclFloat32;
  if (api->AllGather(local, gathered, 1, dt, comm, s) != ncclSuccess) return NRMF_ENCCL;
  const int64_t P2c = pow2_ceil(std::max<int64_t>(cols, 1));
  const int64_t nr = std::min<int64_t>(world, P2c);
  return bal_eval<F>(gathered, nr, nr, frob, s, cr);
}

}  // namespace
}  // namespace nrmf

using namespace nrmf;

extern "C" {

int nrmf_dist_shard(int64_t n_global, int world, int rank, int64_t* offset, int64_t* count) {
  if (n_global < 0 || world < 1 || rank < 0 || rank >= world || !offset || !count) return NRMF_EINVAL;
  if (!is_pow2(world)) return NRMF_ESHARD;
  shard(n_global, world, rank, offset, count);
  return NRMF_OK;
}

size_t nrmf_dist_workspace_bytes(int64_t n_global, int world, int elem_bytes) {
  if (n_global < 0 || world < 1 || (elem_bytes != 4 && elem_bytes != 8)) return 0;
  return dist_ws(n_global, world, (size_t)elem_bytes);
}

int nrmf_dist_d(int64_t n_global, int64_t offset, int64_t count, const double* x_local, double* out,
                void* ws, size_t ws_bytes, void* nccl_comm, void* stream) {
  return dist_impl<double>(n_global, offset, count, x_local, out, ws, ws_bytes, nccl_comm, stream, 0);
}
int nrmf_dist_s(int64_t n_global, int64_t offset, int64_t count, const float* x_local, float* out,
                void* ws, size_t ws_bytes, void* nccl_comm, void* stream) {
  return dist_impl<float>(n_global, offset, count, x_local, out, ws, ws_bytes, nccl_comm, stream, 0);
}
int nrmf_dist_ex_d(int64_t n_global, int64_t offset, int64_t count, const double* x_local, double* out,
                   int flags, void* ws, size_t ws_bytes, void* nccl_comm, void* stream) {
  return dist_impl<double>(n_global, offset, count, x_local, out, ws, ws_bytes, nccl_comm, stream, flags);
}
int nrmf_dist_ex_s(int64_t n_global, int64_t offset, int64_t count, const float* x_local, float* out,
                   int flags, void* ws, size_t ws_bytes, void* nccl_comm, void* stream) {
  return dist_impl<float>(n_global, offset, count, x_local, out, ws, ws_bytes, nccl_comm, stream, flags);
}

int nrmf_dist_local_d(int64_t n_global, int world, int rank, int64_t offset, int64_t count, const double* x_local,
                      double* local_out, int flags, void* ws, size_t ws_bytes, void* stream) {
  return local_step<double>(n_global, world, rank, offset, count, x_local, local_out, flags, ws, ws_bytes,
                            static_cast<cudaStream_t>(stream), nullptr);
}
int nrmf_dist_local_s(int64_t n_global, int world, int rank, int64_t offset, int64_t count, const float* x_local,
                      float* local_out, int flags, void* ws, size_t ws_bytes, void* stream) {
  return local_step<float>(n_global, world, rank, offset, count, x_local, local_out, flags, ws, ws_bytes,
                           static_cast<cudaStream_t>(stream), nullptr);
}
int nrmf_rank_combine_d(int64_t n_global, int world, const double* values, double* out, int flags, void* stream) {
  return rank_combine<double>(n_global, world, values, out, flags, static_cast<cudaStream_t>(stream));
}
int nrmf_rank_combine_s(int64_t n_global, int world, const float* values, float* out, int flags, void* stream) {
  return rank_combine<float>(n_global, world, values, out, flags, static_cast<cudaStream_t>(stream));
}

int nrmf_cols_dist_shard(int64_t cols_global, int world, int rank, int64_t* col_offset, int64_t* col_count) {
  if (cols_global < 0 || world < 1 || rank < 0 || rank >= world || !col_offset || !col_count) return NRMF_EINVAL;
  if (!is_pow2(world)) return NRMF_ESHARD;
  int64_t t0, t1;
  shard_units(cols_global, world, rank, &t0, &t1);
  *col_offset = std::min(t0, cols_global);
  *col_count = std::min(t1, cols_global) - *col_offset;
  return NRMF_OK;
}

size_t nrmf_cols_dist_workspace_bytes(int64_t rows, int64_t cols_global, int world, int elem_bytes) {
  if (rows < 0 || cols_global < 0 || world < 1 || (elem_bytes != 4 && elem_bytes != 8)) return 0;
  return cols_dist_ws(rows, cols_global, world, (size_t)elem_bytes);
}

int nrmf_cols_dist_d(int64_t rows, int64_t cols_global, int64_t ld, int64_t col_offset, int64_t col_count,
                     const double* A_local, double* col_norms_local, double* frob, int flags, void* ws,
                     size_t ws_bytes, void* nccl_comm, void* stream) {
  return cols_dist_impl<double>(rows, cols_global, ld, col_offset, col_count, A_local, col_norms_local, frob,
                                flags, ws, ws_bytes, nccl_comm, stream);
}
int nrmf_cols_dist_s(int64_t rows, int64_t cols_global, int64_t ld, int64_t col_offset, int64_t col_count,
                     const float* A_local, float* col_norms_local, float* frob, int flags, void* ws,
                     size_t ws_bytes, void* nccl_comm, void* stream) {
  return cols_dist_impl<float>(rows, cols_global, ld, col_offset, col_count, A_local, col_norms_local, frob,
                               flags, ws, ws_bytes, nccl_comm, stream);
}

size_t nrmf_p2p_buffer_bytes(void) { return (size_t)kP2PBytes; }

int nrmf_p2p_alloc(void** buf) {
  if (buf == nullptr) return NRMF_EINVAL;
  void* p = nullptr;
  if (cudaMalloc(&p, kP2PBytes) != cudaSuccess) return NRMF_ECUDA;
  if (cudaMemset(p, 0, kP2PBytes) != cudaSuccess) {
    cudaFree(p);
    return NRMF_ECUDA;
  }
  *buf = p;
  return NRMF_OK;
}
int nrmf_p2p_free(void* buf) { return cudaFree(buf) == cudaSuccess ? NRMF_OK : NRMF_ECUDA; }

int nrmf_p2p_ipc_handle(const void* buf, char* handle64) {
  if (buf == nullptr || handle64 == nullptr) return NRMF_EINVAL;
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(buf)) != cudaSuccess) return NRMF_ECUDA;
  std::memcpy(handle64, &h, sizeof h);
  return NRMF_OK;
}
int nrmf_p2p_open(const char* handle64, void** peer_buf) {
  if (handle64 == nullptr || peer_buf == nullptr) return NRMF_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  if (cudaIpcOpenMemHandle(peer_buf, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return NRMF_ECUDA;
  return NRMF_OK;
}
int nrmf_p2p_close(void* peer_buf) {
  return cudaIpcCloseMemHandle(peer_buf) == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
}

int nrmf_dist_p2p_d(int64_t n_global, int64_t offset, int64_t count, const double* x_local, double* out,
                    int flags, void* ws, size_t ws_bytes, const void* peers, int world, int rank, unsigned* err,
                    void* stream) {
  return dist_p2p_impl<double>(n_global, offset, count, x_local, out, flags, ws, ws_bytes, peers, world, rank,
                               err, stream);
}
int nrmf_dist_p2p_s(int64_t n_global, int64_t offset, int64_t count, const float* x_local, float* out,
                    int flags, void* ws, size_t ws_bytes, const void* peers, int world, int rank, unsigned* err,
                    void* stream) {
  return dist_p2p_impl<float>(n_global, offset, count, x_local, out, flags, ws, ws_bytes, peers, world, rank,
                              err, stream);
}

// test hooks (not in nrmf.h): `world` ranks emulated as CTAs of one cooperative launch
int nrmf_debug_p2p_emulate_d(int world, const double* values, const void* peers, int flags, double* outs,
                             void* stream) {
  return p2p_emulate<double>(world, values, peers, flags, outs, stream);
}
int nrmf_debug_p2p_emulate_s(int world, const float* values, const void* peers, int flags, float* outs,
                             void* stream) {
  return p2p_emulate<float>(world, values, peers, flags, outs, stream);
}

int nrmf_nccl_unique_id(char* id128) {
  const NcclApi* api = nccl();
  if (api == nullptr) return NRMF_ENCCL;
  if (id128 == nullptr) return NRMF_EINVAL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return NRMF_ENCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof id);
  return NRMF_OK;
}

int nrmf_nccl_comm_init(int world, int rank, const char* id128, void** comm) {
  const NcclApi* api = nccl();
  if (api == nullptr) return NRMF_ENCCL;
  if (id128 == nullptr || comm == nullptr || world < 1 || rank < 0 || rank >= world) return NRMF_EINVAL;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  if (api->CommInitRank(&c, world, id, rank) != ncclSuccess) return NRMF_ENCCL;
  *comm = c;
  return NRMF_OK;
}

int nrmf_nccl_comm_destroy(void* comm) {
  const NcclApi* api = nccl();
  if (api == nullptr) return NRMF_ENCCL;
  if (comm == nullptr) return NRMF_EINVAL;
  return api->CommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? NRMF_OK : NRMF_ENCCL;
}

}  // extern "C"
