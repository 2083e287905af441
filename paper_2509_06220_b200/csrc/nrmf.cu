// nrmf.cu -- kernels and C ABI (include/nrmf.h) of the B200 xNRMF path.
//
// One kernel evaluates the whole tree of one call (a1-a5 of DESIGN.md §8):
//   * persistent grid, kWarps warps per CTA, CTA loops over groups g of
//     kWarps consecutive tiles (group = aligned 8-tile subtree);
//   * warp w reduces tile tau = 8g + w (B1, warp_tile);
//   * the 8 tile values are combined in shared memory + shuffles (first
//     min(3, lg P2) levels of the tile tree) into partials[g];
//   * __threadfence + integer ticket; the last CTA to finish evaluates the
//     remaining levels over partials[0..P2/8) (B2, block_bal), writes *out and
//     resets the ticket.  No floating-point atomics: the tree never depends on
//     arrival order, grid size or occupancy.
// Columns use the same kernel with item -> (column, tile-in-column) mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/nrmf.h"
#include "nrmf_device.cuh"
#include "nrmf_internal.h"

namespace nrmf {

// ------------------------------------------------------------------ kernels
template <typename F>
struct TileJob {
  const F* x;          // base pointer
  int64_t n_items;     // tiles that contain data
  int64_t tpc;         // tiles per column (vector mode: n_items)
  int64_t ld;          // elements between column bases (vector mode: unused)
  int64_t len;         // column length (vector mode: n)
  int64_t p2;          // tiles of the (sub)tree evaluated: power of two >= n_items
  F* tile_out;         // optional per-tile values
  F* partials;         // group partials (workspace)
  unsigned* ticket;    // last-CTA ticket (workspace)
  F* out;              // result (root of the p2-tile tree); unused if !combine
  int combine;         // 0: only write tile values
};

template <typename F, bool VEC>
__global__ void __launch_bounds__(kThreads, 2) nrmf_tiles_kernel(const TileJob<F> job) {
  __shared__ F s_tile[kWarps];
  __shared__ int s_last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_groups = (job.n_items + kWarps - 1) / kWarps;
  const int lgp2 = ilog2_64(job.p2);
  const int glevels = lgp2 < 3 ? lgp2 : 3;
  const int64_t pg = job.p2 >= kWarps ? job.p2 / kWarps : 1;

  for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const int64_t tau = g * kWarps + w;
    F tv = F(0);
    if (tau < job.n_items) {
      const int64_t col = tau / job.tpc, tt = tau - col * job.tpc;
      const F* tb = job.x + col * job.ld + tt * (int64_t)kTile;
      const int64_t rem = job.len - tt * (int64_t)kTile;
      const int valid = rem < kTile ? (int)rem : kTile;
      if (valid == kTile) {
        tv = VEC ? warp_tile<F, kVec>(tb) : warp_tile<F, kScalar>(tb);
      } else {
        tv = warp_tile_exact<F, kPred>(tb, valid);
      }
      if (job.tile_out != nullptr && lane == 0) job.tile_out[tau] = tv;
    }
    if (!job.combine) continue;
    if (lane == 0) s_tile[w] = tv;
    __syncthreads();
    if (w == 0) {
      F v = lane < kWarps ? s_tile[lane] : F(0);
      for (int l = 0; l < glevels; ++l) v = v1h(v, __shfl_xor_sync(0xffffffffu, v, 1 << l));
      if (lane == 0) {
        if (pg == 1) *job.out = v;
        else job.partials[g] = v;
      }
    }
    __syncthreads();
  }
  if (!job.combine || pg == 1) return;

  // deterministic grid combine: last CTA evaluates the top of the tree
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(job.ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const F v = block_bal(job.partials, n_groups, pg);
  if (threadIdx.x == 0) {
    *job.out = v;
    *job.ticket = 0u;  // ready for the next call on this workspace
  }
}

// Balanced tree over vals[0..P) (entries >= nvals are +0) -> *out.  One CTA.
template <typename F>
__global__ void __launch_bounds__(kThreads) bal_kernel(const F* vals, int64_t nvals, int64_t P,
                                                       F* out) {
  const F v = block_bal(vals, nvals, P);
  if (threadIdx.x == 0) *out = v;
}

// Per-column combine for columns longer than one tile: column j has tpc tile
// values vals[j*tpc ..] padded to p2c; then the frob tree over columns
// (p2cols = pow2 >= cols) with group partials per CTA and a last-CTA top.
template <typename F>
__global__ void __launch_bounds__(kThreads) cols_combine_kernel(
    const F* vals, int64_t cols, int64_t tpc, int64_t p2c, F* col_norms, int64_t p2cols,
    F* partials, unsigned* ticket, F* frob) {
  __shared__ int s_last;
  const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  F v = F(0);
  if (j < cols) {
    v = seq_bal(vals + j * tpc, tpc, 0, p2c);
    col_norms[j] = v;
  }
  if (frob == nullptr) return;
  // block level: first min(8, lg p2cols) levels of the frob tree
  const int lg = ilog2_64(p2cols);
  const int bl = lg < 8 ? lg : 8;
  __shared__ F sh[kWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wl = bl < 5 ? bl : 5;
  for (int l = 0; l < wl; ++l) v = v1h(v, __shfl_xor_sync(0xffffffffu, v, 1 << l));
  if (bl > 5) {
    if (lane == 0) sh[w] = v;
    __syncthreads();
    v = lane < kWarps ? sh[lane] : F(0);
    for (int l = 0; l < bl - 5; ++l) v = v1h(v, __shfl_xor_sync(0xffffffffu, v, 1 << l));
  }
  const int64_t pb = p2cols >> bl;  // values left after the block levels
  if (pb == 1) {
    if (threadIdx.x == 0) *frob = v;
    return;
  }
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    const unsigned prev = atomicAdd(ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const F r = block_bal(partials, (int64_t)gridDim.x, pb);
  if (threadIdx.x == 0) {
    *frob = r;
    *ticket = 0u;
  }
}

// ------------------------------------------------------------------ host side
static int64_t pow2_ceil(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

static int device_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = sms > 0 ? sms : 1;
  }
  return cached[dev];
}

template <typename F, bool VEC>
static int blocks_per_sm() {
  static int cached = 0;
  if (cached == 0) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, nrmf_tiles_kernel<F, VEC>, kThreads, 0) !=
            cudaSuccess ||
        b < 1)
      b = 1;
    cached = b;
  }
  return cached;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Workspace layout for one tile-tree evaluation: [ticket: 256 B][partials]
static size_t tree_ws_bytes(int64_t p2, size_t esz) {
  const int64_t pg = p2 >= kWarps ? p2 / kWarps : 1;
  return 256 + align_up((size_t)pg * esz, 256);
}

template <typename F>
static int launch_tree(const TileJob<F>& job_in, bool vec, cudaStream_t s, int grid_override) {
  TileJob<F> job = job_in;
  const int64_t n_groups = (job.n_items + kWarps - 1) / kWarps;
  if (n_groups == 0) return NRMF_OK;
  int64_t grid = (int64_t)device_sms() * (vec ? blocks_per_sm<F, true>() : blocks_per_sm<F, false>());
  if (grid_override > 0) grid = grid_override;
  grid = std::min<int64_t>(grid, n_groups);
  if (vec)
    nrmf_tiles_kernel<F, true><<<(unsigned)grid, kThreads, 0, s>>>(job);
  else
    nrmf_tiles_kernel<F, false><<<(unsigned)grid, kThreads, 0, s>>>(job);
  return cudaGetLastError() == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
}

static int g_grid_override = 0;  // test hook: force a grid size (0 = auto)

template <typename F>
int tree_eval(int64_t n, const F* x, int64_t p2, F* out, void* ws, size_t ws_bytes,
              cudaStream_t s) {
  // Evaluate the balanced tree over p2 tiles (p2 >= ceil(n/T), power of two)
  // of x[0..n) padded with +0; *out = root.  Caller validated arguments.
  const int64_t nt = (n + kTile - 1) / kTile;
  if (nt == 0) {
    if (cudaMemsetAsync(out, 0, sizeof(F), s) != cudaSuccess) return NRMF_ECUDA;
    return NRMF_OK;
  }
  if (ws_bytes < tree_ws_bytes(p2, sizeof(F))) return NRMF_EWORKSPACE;
  TileJob<F> job;
  job.x = x;
  job.n_items = nt;
  job.tpc = nt;
  job.ld = 0;
  job.len = n;
  job.p2 = p2;
  job.tile_out = nullptr;
  job.ticket = reinterpret_cast<unsigned*>(ws);
  job.partials = reinterpret_cast<F*>(static_cast<char*>(ws) + 256);
  job.out = out;
  job.combine = 1;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
  return launch_tree(job, vec, s, g_grid_override);
}

template int tree_eval<double>(int64_t, const double*, int64_t, double*, void*, size_t, cudaStream_t);
template int tree_eval<float>(int64_t, const float*, int64_t, float*, void*, size_t, cudaStream_t);

template <typename F>
int bal_eval(const F* vals, int64_t nvals, int64_t P, F* out, cudaStream_t s) {
  bal_kernel<F><<<1, kThreads, 0, s>>>(vals, nvals, P, out);
  return cudaGetLastError() == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
}
template int bal_eval<double>(const double*, int64_t, int64_t, double*, cudaStream_t);
template int bal_eval<float>(const float*, int64_t, int64_t, float*, cudaStream_t);

size_t tree_workspace(int64_t p2, size_t esz) { return tree_ws_bytes(p2, esz); }

// ---------------------------------------------------------------- vector
template <typename F>
static int nrmf_vec(int64_t n, const F* x, F* out, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || out == nullptr || (n > 0 && (x == nullptr || ws == nullptr))) return NRMF_EINVAL;
  if ((reinterpret_cast<uintptr_t>(x) % sizeof(F)) != 0 ||
      (reinterpret_cast<uintptr_t>(out) % sizeof(F)) != 0)
    return NRMF_EALIGN;
  const int64_t nt = (n + kTile - 1) / kTile;
  return tree_eval<F>(n, x, pow2_ceil(std::max<int64_t>(nt, 1)), out, ws, ws_bytes,
                      static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- columns
// Workspace: [ticket 256][tile values: cols*tpc if tpc>1][partials]
static size_t cols_ws_bytes(int64_t rows, int64_t cols, size_t esz) {
  const int64_t tpc = std::max<int64_t>((rows + kTile - 1) / kTile, 1);
  const int64_t p2cols = pow2_ceil(std::max<int64_t>(cols, 1));
  size_t b = 256;
  if (tpc > 1) b += align_up((size_t)(cols * tpc) * esz, 256);
  const int64_t nblk = (cols + kThreads - 1) / kThreads;
  b += align_up((size_t)std::max<int64_t>({p2cols / kWarps, nblk, 1}) * esz, 256);
  return b;
}

template <typename F>
static int nrmf_cols_impl(int64_t rows, int64_t cols, int64_t ld, const F* A, F* col_norms,
                          F* frob, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rows < 0 || cols < 0 || ld < rows || ld < 0) return NRMF_EINVAL;
  if (cols > 0 && col_norms == nullptr) return NRMF_EINVAL;
  if (rows > 0 && cols > 0 && (A == nullptr || ws == nullptr)) return NRMF_EINVAL;
  if (reinterpret_cast<uintptr_t>(A) % sizeof(F) || reinterpret_cast<uintptr_t>(col_norms) % sizeof(F) ||
      reinterpret_cast<uintptr_t>(frob) % sizeof(F))
    return NRMF_EALIGN;
  if (cols == 0) {
    if (frob && cudaMemsetAsync(frob, 0, sizeof(F), s) != cudaSuccess) return NRMF_ECUDA;
    return NRMF_OK;
  }
  if (rows == 0) {
    if (cudaMemsetAsync(col_norms, 0, (size_t)cols * sizeof(F), s) != cudaSuccess) return NRMF_ECUDA;
    if (frob && cudaMemsetAsync(frob, 0, sizeof(F), s) != cudaSuccess) return NRMF_ECUDA;
    return NRMF_OK;
  }
  if (ws_bytes < cols_ws_bytes(rows, cols, sizeof(F))) return NRMF_EWORKSPACE;
  const int64_t tpc = (rows + kTile - 1) / kTile;
  const int64_t p2cols = pow2_ceil(cols);
  unsigned* ticket = reinterpret_cast<unsigned*>(ws);
  char* base = static_cast<char*>(ws) + 256;
  const bool vec = (reinterpret_cast<uintptr_t>(A) & 15u) == 0 && ((ld * (int64_t)sizeof(F)) & 15) == 0;
  TileJob<F> job;
  job.x = A;
  job.tpc = tpc;
  job.ld = ld;
  job.len = rows;
  job.ticket = ticket;
  if (tpc == 1) {
    // one tile per column: tile value = column norm; frob = tree over columns
    job.n_items = cols;
    job.p2 = p2cols;
    job.tile_out = col_norms;
    job.partials = reinterpret_cast<F*>(base);
    job.out = frob;
    job.combine = frob != nullptr ? 1 : 0;
    return launch_tree(job, vec, s, g_grid_override);
  }
  // multi-tile columns: tile values, then per-column trees + frob tree
  F* vals = reinterpret_cast<F*>(base);
  F* partials = reinterpret_cast<F*>(base + align_up((size_t)(cols * tpc) * sizeof(F), 256));
  job.n_items = cols * tpc;
  job.p2 = 1;
  job.tile_out = vals;
  job.partials = nullptr;
  job.out = nullptr;
  job.combine = 0;
  int st = launch_tree(job, vec, s, g_grid_override);
  if (st != NRMF_OK) return st;
  const int64_t nblk = (cols + kThreads - 1) / kThreads;
  cols_combine_kernel<F><<<(unsigned)nblk, kThreads, 0, s>>>(vals, cols, tpc, pow2_ceil(tpc), col_norms,
                                                            p2cols, partials, ticket, frob);
  return cudaGetLastError() == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
}

// ---------------------------------------------------------------- host input
// Device staging ring: kRing buffers of kChunkTiles tiles; chunk k covers
// tiles [k*C, (k+1)*C) -- an aligned subtree when P2 >= C.
constexpr int kRing = 4;
constexpr int64_t kChunkTiles = 512;

struct HostStreamState {
  cudaStream_t copy = nullptr;
  cudaEvent_t copied[kRing] = {};
  cudaEvent_t consumed[kRing] = {};
  cudaEvent_t start = nullptr;
  bool ok = false;
};
static std::mutex g_host_mu;
static HostStreamState g_host_state[64];

static HostStreamState* host_state() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  HostStreamState& h = g_host_state[dev];
  if (!h.ok) {
    if (cudaStreamCreateWithFlags(&h.copy, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    for (int i = 0; i < kRing; ++i) {
      if (cudaEventCreateWithFlags(&h.copied[i], cudaEventDisableTiming) != cudaSuccess) return nullptr;
      if (cudaEventCreateWithFlags(&h.consumed[i], cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    if (cudaEventCreateWithFlags(&h.start, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    h.ok = true;
  }
  return &h;
}

// [ticket+partials for one chunk][chunk values][result][ring buffers]
static size_t host_ws_bytes(int64_t n, size_t esz) {
  const int64_t nt = std::max<int64_t>((n + kTile - 1) / kTile, 1);
  const int64_t p2 = pow2_ceil(nt);
  const int64_t c = std::min<int64_t>(p2, kChunkTiles);
  const int64_t nchunks = (nt + c - 1) / c;
  return tree_ws_bytes(c, esz) + align_up((size_t)nchunks * esz, 256) + 256 +
         (size_t)kRing * (size_t)(c * kTile) * esz;
}

template <typename F>
static int nrmf_host_impl(int64_t n, const F* host_x, F* host_out, void* ws, size_t ws_bytes,
                          void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 0 || host_out == nullptr || ws == nullptr || (n > 0 && host_x == nullptr)) return NRMF_EINVAL;
  if (reinterpret_cast<uintptr_t>(host_x) % sizeof(F)) return NRMF_EALIGN;
  if (ws_bytes < host_ws_bytes(n, sizeof(F))) return NRMF_EWORKSPACE;
  const int64_t nt = std::max<int64_t>((n + kTile - 1) / kTile, 1);
  const int64_t p2 = pow2_ceil(nt);
  const int64_t c = std::min<int64_t>(p2, kChunkTiles);
  const int64_t nchunks = (nt + c - 1) / c;
  char* p = static_cast<char*>(ws);
  void* tree_ws = p;
  const size_t tws = tree_ws_bytes(c, sizeof(F));
  p += tws;
  F* chunk_vals = reinterpret_cast<F*>(p);
  p += align_up((size_t)nchunks * sizeof(F), 256);
  F* dev_out = reinterpret_cast<F*>(p);
  p += 256;
  F* ring = reinterpret_cast<F*>(p);
  const int64_t chunk_elems = c * kTile;

  std::lock_guard<std::mutex> lock(g_host_mu);
  HostStreamState* h = host_state();
  if (h == nullptr) return NRMF_ECUDA;
  if (n == 0) {
    if (cudaMemsetAsync(dev_out, 0, sizeof(F), s) != cudaSuccess) return NRMF_ECUDA;
  } else {
    // the copy stream must not overwrite staging buffers still read by
    // earlier work on s
    if (cudaEventRecord(h->start, s) != cudaSuccess) return NRMF_ECUDA;
    if (cudaStreamWaitEvent(h->copy, h->start, 0) != cudaSuccess) return NRMF_ECUDA;
    for (int64_t k = 0; k < nchunks; ++k) {
      const int slot = (int)(k % kRing);
      const int64_t e0 = k * chunk_elems;
      const int64_t cnt = std::min<int64_t>(chunk_elems, n - e0);
      F* buf = ring + (int64_t)slot * chunk_elems;
      if (k >= kRing && cudaStreamWaitEvent(h->copy, h->consumed[slot], 0) != cudaSuccess) return NRMF_ECUDA;
      if (cudaMemcpyAsync(buf, host_x + e0, (size_t)cnt * sizeof(F), cudaMemcpyHostToDevice, h->copy) !=
          cudaSuccess)
        return NRMF_ECUDA;
      if (cudaEventRecord(h->copied[slot], h->copy) != cudaSuccess) return NRMF_ECUDA;
      if (cudaStreamWaitEvent(s, h->copied[slot], 0) != cudaSuccess) return NRMF_ECUDA;
      int st = tree_eval<F>(cnt, buf, c, nchunks == 1 ? dev_out : chunk_vals + k, tree_ws, tws, s);
      if (st != NRMF_OK) return st;
      if (cudaEventRecord(h->consumed[slot], s) != cudaSuccess) return NRMF_ECUDA;
    }
    if (nchunks > 1) {
      int st = bal_eval<F>(chunk_vals, nchunks, p2 / c, dev_out, s);
      if (st != NRMF_OK) return st;
    }
  }
  if (cudaMemcpyAsync(host_out, dev_out, sizeof(F), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return NRMF_ECUDA;
  return NRMF_OK;
}

}  // namespace nrmf

// ==================================================================== C ABI
using namespace nrmf;

extern "C" {

const char* nrmf_status_str(int status) {
  switch (status) {
    case NRMF_OK: return "NRMF_OK";
    case NRMF_EINVAL: return "NRMF_EINVAL: invalid argument";
    case NRMF_EALIGN: return "NRMF_EALIGN: pointer not aligned to its element size";
    case NRMF_EWORKSPACE: return "NRMF_EWORKSPACE: workspace too small";
    case NRMF_ESHARD: return "NRMF_ESHARD: not the canonical shard / world not a power of two";
    case NRMF_ECUDA: return "NRMF_ECUDA: CUDA error";
    case NRMF_ENCCL: return "NRMF_ENCCL: NCCL error or NCCL unavailable";
    default: return "NRMF_UNKNOWN";
  }
}

int nrmf_tree_version(void) { return kTreeVersion; }

int nrmf_tree_params(int elem_bytes, int* lanes, int* J, int* tile) {
  if (elem_bytes == 8) {
    if (lanes) *lanes = Cfg<double>::LANES;
    if (J) *J = Cfg<double>::J;
  } else if (elem_bytes == 4) {
    if (lanes) *lanes = Cfg<float>::LANES;
    if (J) *J = Cfg<float>::J;
  } else {
    return NRMF_EINVAL;
  }
  if (tile) *tile = kTile;
  return NRMF_OK;
}

size_t nrmf_workspace_bytes(int64_t n, int elem_bytes) {
  if (n < 0 || (elem_bytes != 4 && elem_bytes != 8)) return 0;
  const int64_t nt = std::max<int64_t>((n + kTile - 1) / kTile, 1);
  return tree_ws_bytes(pow2_ceil(nt), (size_t)elem_bytes);
}

int nrmf_d(int64_t n, const double* x, double* out, void* ws, size_t ws_bytes, void* stream) {
  return nrmf_vec<double>(n, x, out, ws, ws_bytes, stream);
}
int nrmf_s(int64_t n, const float* x, float* out, void* ws, size_t ws_bytes, void* stream) {
  return nrmf_vec<float>(n, x, out, ws, ws_bytes, stream);
}
int nrmf_z_d(int64_t count, const double* z, double* out, void* ws, size_t ws_bytes, void* stream) {
  if (count < 0 || count > INT64_MAX / 2) return NRMF_EINVAL;
  return nrmf_vec<double>(2 * count, z, out, ws, ws_bytes, stream);
}
int nrmf_z_s(int64_t count, const float* z, float* out, void* ws, size_t ws_bytes, void* stream) {
  if (count < 0 || count > INT64_MAX / 2) return NRMF_EINVAL;
  return nrmf_vec<float>(2 * count, z, out, ws, ws_bytes, stream);
}

size_t nrmf_cols_workspace_bytes(int64_t rows, int64_t cols, int elem_bytes) {
  if (rows < 0 || cols < 0 || (elem_bytes != 4 && elem_bytes != 8)) return 0;
  return cols_ws_bytes(rows, cols, (size_t)elem_bytes);
}
int nrmf_cols_d(int64_t rows, int64_t cols, int64_t ld, const double* A, double* col_norms,
                double* frob, void* ws, size_t ws_bytes, void* stream) {
  return nrmf_cols_impl<double>(rows, cols, ld, A, col_norms, frob, ws, ws_bytes, stream);
}
int nrmf_cols_s(int64_t rows, int64_t cols, int64_t ld, const float* A, float* col_norms,
                float* frob, void* ws, size_t ws_bytes, void* stream) {
  return nrmf_cols_impl<float>(rows, cols, ld, A, col_norms, frob, ws, ws_bytes, stream);
}

size_t nrmf_host_workspace_bytes(int64_t n, int elem_bytes) {
  if (n < 0 || (elem_bytes != 4 && elem_bytes != 8)) return 0;
  return host_ws_bytes(n, (size_t)elem_bytes);
}
int nrmf_host_d(int64_t n, const double* host_x, double* host_out, void* ws, size_t ws_bytes,
                void* stream) {
  return nrmf_host_impl<double>(n, host_x, host_out, ws, ws_bytes, stream);
}
int nrmf_host_s(int64_t n, const float* host_x, float* host_out, void* ws, size_t ws_bytes,
                void* stream) {
  return nrmf_host_impl<float>(n, host_x, host_out, ws, ws_bytes, stream);
}

// test hook (not in nrmf.h): force the persistent grid size, 0 = automatic
int nrmf_debug_set_grid(int grid) {
  g_grid_override = grid < 0 ? 0 : grid;
  return NRMF_OK;
}

}  // extern "C"
