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
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/nrmf.h"
#include "nrmf_device.cuh"
#include "nrmf_internal.h"
#include "nrmf_p2p.cuh"

namespace nrmf {

// ------------------------------------------------------------------ kernels
constexpr int kMaxSteps = 8;
constexpr int kMaxFanLg = 8;  // combine steps of 6 levels; the split kernel's last one up to 8 (fan-in 256)
#ifndef NRMF_SAFE_MODE
#define NRMF_SAFE_MODE 1      // stream kernel: safe-node groups from the ring after a flagged group
#endif
#ifndef NRMF_STAGES
#define NRMF_STAGES 2         // TMA ring depth per warp (batches of 4 KiB)
#endif
#ifndef NRMF_BPI
#define NRMF_BPI 1            // batches per loop iteration on the TMA path
#endif
#ifndef NRMF_USE_TMA
#define NRMF_USE_TMA 1        // 0: aligned full tiles use direct LDG.128 instead of the TMA ring
#endif
#ifndef NRMF_SHORT_PAIRS
#define NRMF_SHORT_PAIRS 1    // columns of rows <= 2 batches: two per warp at a time
#endif
#ifndef NRMF_LL_TWO
#define NRMF_LL_TWO 1  // split kernel: the fan-in-256 last step polled by two warps
#endif
#ifndef NRMF_SHORT_PAIRS_ELEM
#define NRMF_SHORT_PAIRS_ELEM 1  // ... also in the element-load kernel (unaligned column blocks)
#endif
#ifndef NRMF_SKIP_FLAGGED
#define NRMF_SKIP_FLAGGED 0   // 1: stream kernel stops evaluating a group at its first flagged tile (C5 -6 %, DNRMF +1.3 %: off)
#endif
#ifndef NRMF_CTA_STEP
#define NRMF_CTA_STEP 1       // stream kernel: first combine step (16 warp groups) inside the CTA
#endif
#ifndef NRMF_MIN_BLOCKS
#define NRMF_MIN_BLOCKS 1     // CTAs per SM the register allocation must allow (16 warps x 128 registers)
#endif
constexpr int kStages = NRMF_STAGES;
constexpr int kBPI = NRMF_BPI;
static_assert(kStages >= kBPI, "the ring must hold one iteration");

#ifdef NRMF_PROBE_TRACE  // dev-only: globaltimer event trace of the tree kernel
__device__ unsigned long long* g_trace = nullptr;
__device__ unsigned g_trace_n = 0;
__device__ unsigned g_trace_cap = 0;
__device__ __forceinline__ void trace(unsigned type, unsigned level, unsigned id) {
  if ((threadIdx.x & 31) != 0 || g_trace == nullptr) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
#ifdef NRMF_PROBE_TRACE2  // one slot per (warp, event type): no atomics (split-kernel timelines)
  if (type < 16) g_trace[((unsigned long long)blockIdx.x * 32 + (threadIdx.x >> 5)) * 16 + type] = t;
  return;
#endif
  const unsigned i = atomicAdd(&g_trace_n, 1u);
  if (i < g_trace_cap) {
    g_trace[2 * i] = ((unsigned long long)type << 56) | ((unsigned long long)level << 48) |
                     ((unsigned long long)blockIdx.x << 24) | (threadIdx.x >> 5);
    g_trace[2 * i + 1] = t;
  }
}
// an event with a time taken earlier (no atomic between the measured points)
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_at(unsigned type, unsigned long long t) {
  if ((threadIdx.x & 31) != 0 || g_trace == nullptr) return;
#ifdef NRMF_PROBE_TRACE2
  if (type < 16) g_trace[((unsigned long long)blockIdx.x * 32 + (threadIdx.x >> 5)) * 16 + type] = t;
  return;
#endif
  const unsigned i = atomicAdd(&g_trace_n, 1u);
  if (i < g_trace_cap) {
    g_trace[2 * i] = ((unsigned long long)type << 56) | ((unsigned long long)blockIdx.x << 24) | (threadIdx.x >> 5);
    g_trace[2 * i + 1] = t;
  }
}
#define NRMF_TRACE(a, b, c) trace(a, b, c)
#define NRMF_TSTAMP(v) const unsigned long long v = gtime()
#define NRMF_TRACE_AT(a, v) trace_at(a, v)
#else
#define NRMF_TRACE(a, b, c) (void)0
#define NRMF_TSTAMP(v) (void)0
#define NRMF_TRACE_AT(a, v) (void)0
#endif

#ifdef NRMF_PROBE_JITTER  // test build only: random delays at every step of the combine protocols
__device__ __forceinline__ void jitter(unsigned salt) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  unsigned h = (unsigned)(t ^ (t >> 17)) * 0x9E3779B1u ^ (salt * 0x85EBCA6Bu) ^ (blockIdx.x * 0xC2B2AE35u) ^
               (threadIdx.x >> 5);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3) != 0) __nanosleep(h % 4000u);  // 0 .. 4 us, three times in four
}
#define NRMF_JITTER(s) jitter(s)
#else
#define NRMF_JITTER(s) (void)0
#endif

// One evaluation of the tile tree.  Work unit of a warp: a "warp group" of
// 2^g0 consecutive tiles (an aligned subtree: its first g0 levels are
// combined in registers); above it, steps of up to 6 levels (fan-in 64) are
// combined by the last-arriving warp of each group (integer counters in the
// workspace).  The shape of the tree never depends on g0, the grid or timing.
template <typename F>
struct TreeJob {
  const F* x;          // base pointer
  int64_t n_items;     // tiles that contain data
  int64_t tpc;         // tiles per column (vector mode: n_items)
  int64_t ld;          // elements between column bases (vector mode: 0)
  int64_t len;         // column length (vector mode: n)
  F* tile_out;         // optional: every tile value (column norms)
  F* vals;             // workspace: warp-group values and higher levels
  unsigned* cnt;       // workspace: arrival counters of every step (zero between calls)
  F* out;              // root of the tree; unused if !combine
  int combine;         // 0: only write tile values
  int top_cr;          // levels above the tiles use cr_hypot (NRMF_TOP_CR)
  int g0;              // tile-tree levels combined inside a warp group (<= 3)
  int cta_minor;       // warp index w * gridDim + block (few groups) instead of block * kWarps + w
  int cta_step0;       // stream kernel: step 0 (fan-in 16 = one CTA's warps of a round) in shared memory
  int nsteps;          // combine steps above the warp groups
  int lg_fan[kMaxSteps];
  int64_t nin[kMaxSteps];      // real (non-padding) inputs of step k (nin[0] = warp groups)
  int64_t val_off[kMaxSteps];  // vals offset of the inputs of step k
  int64_t cnt_off[kMaxSteps];  // cnt offset of the counters of step k
  // rank exchange fused into the root's writer (nrmf_dist_p2p_[ds]): null = none
  char* const* peers;  // device array of the ranks' exchange buffers (nrmf_p2p.cuh)
  unsigned* p_err;     // nullable: set to 1 if a rank's value did not arrive in time
  int p_world, p_rank, p_nr;
  // split kernel: the LAST combine step by flag-in-data slots instead of a
  // counter (ll_*, below); null = counters for every step.  [epoch word |
  // pad to 16 B][slot i: 16 B]...
  char* ll;
};

// The warp that evaluates the tree's root writes it.  With a fused rank
// exchange (job.peers) the root is this rank's subtree value: the same warp
// publishes it to every peer, waits for theirs and evaluates the rank tree
// (rank_exchange, nrmf_p2p.cuh) before writing *out -- the distributed step
// needs no launch after the tree kernel.  Warp-collective.
// (Out of line, with scalar arguments: a reference to the kernel parameter
// would make ptxas copy the whole TreeJob to the stack.)
template <typename F>
__device__ __noinline__ F exchange_root(char* const* peers, unsigned* err, int world, int rank, int nr, int cr,
                                        F v) {
  PeerArgs a{peers, world, rank, err};
  return rank_exchange<F>(v, a, nr, cr);
}
template <typename F>
__device__ __forceinline__ void write_root(const TreeJob<F>& job, F v) {
  if (job.peers != nullptr)
    v = exchange_root<F>(job.peers, job.p_err, job.p_world, job.p_rank, job.p_nr, job.top_cr, v);
  if ((threadIdx.x & 31) == 0) *job.out = v;
}

// One warp evaluates the balanced tree over 2^f (f <= kMaxFanLg) consecutive
// values vals[base ..] (entries >= nvals are +0).  All lanes return the value.
// Exact nodes (IEEE intrinsics or cr_hypot): f <= 6 in one pass (lane l
// takes values 2l, 2l+1 when f = 6), f = 7, 8 as the top levels over 64-value
// subtrees (the same tree; split kernel only).  That part is not inlined:
// inlined, its calls and live values grew the stack frame 80 -> 400 bytes.
template <typename F>
__device__ __forceinline__ F warp_bal_exact6(const F* vals, int64_t nvals, int64_t base, int f, int cr) {
  const int lane = threadIdx.x & 31;
  F v;
  int lv;
  if (f == 6) {
    const int64_t i = base + 2 * lane;
    const F a = i < nvals ? __ldcg(vals + i) : F(0);
    const F b = i + 1 < nvals ? __ldcg(vals + i + 1) : F(0);
    v = top_node(a, b, cr);
    lv = 5;
  } else {
    const int64_t i = base + lane;
    v = (lane < (1 << f) && i < nvals) ? __ldcg(vals + i) : F(0);
    lv = f;
  }
  for (int l = 0; l < lv; ++l) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, 1 << l), cr);
  return v;
}
template <typename F>
__device__ __noinline__ F warp_bal_exact_wide(const F* vals, int64_t nvals, int64_t base, int f, int cr) {
  const F a = warp_bal_exact6<F>(vals, nvals, base, 6, cr);
  const F b = warp_bal_exact6<F>(vals, nvals, base + 64, 6, cr);
  const F l = top_node<F>(a, b, cr);
  if (f == 7) return l;
  const F c = warp_bal_exact6<F>(vals, nvals, base + 128, 6, cr);
  const F d = warp_bal_exact6<F>(vals, nvals, base + 192, 6, cr);
  return top_node<F>(l, top_node<F>(c, d, cr), cr);
}
template <typename F, bool WIDE>
__device__ __forceinline__ F warp_group_bal_exact(const F* vals, int64_t nvals, int64_t base, int f, int cr) {
  if (WIDE && f > 6) return warp_bal_exact_wide<F>(vals, nvals, base, f, cr);
  return warp_bal_exact6<F>(vals, nvals, base, f, cr);
}

// The in-register levels over K (a power of two) values a[0..K) with fast
// checked nodes, each level's K/2^l independent nodes interleaved in ONE
// v1h_fast_n (separate calls would be issued one chain after the other: ptxas
// keeps the source order of long FP64 chains).  Root in a[0].
template <typename F, int K>
__device__ __forceinline__ void in_lane_levels(F (&a)[K], bool& bad) {
  if constexpr (K >= 2) {
    constexpr int H = K / 2;
    F x[H], y[H], h[H];
#pragma unroll
    for (int j = 0; j < H; ++j) {
      x[j] = a[2 * j];
      y[j] = a[2 * j + 1];
    }
    v1h_fast_n<true, H>(x, y, h, bad);
#pragma unroll
    for (int j = 0; j < H; ++j) a[j] = h[j];
    in_lane_levels<F, H>(reinterpret_cast<F(&)[H]>(a), bad);
  }
}

// Fast-node version: f >= 5: lane l takes the K = 2^(f-5) contiguous values
// [lK, lK+K) as an in-register tree, then 5 __shfl_xor levels; f < 5: lanes
// < 2^f one value each, f shuffle levels.  `bad` flags a node outside the
// fast domain; lv = the shuffle levels.
template <typename F, int K>
__device__ __forceinline__ F lane_bal_fast(const F* vals, int64_t nvals, int64_t base, bool& bad) {
  const int lane = threadIdx.x & 31;
  F a[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int64_t i = base + (int64_t)K * lane + j;
    a[j] = i < nvals ? __ldcg(vals + i) : F(0);
  }
  in_lane_levels<F, K>(a, bad);
  return a[0];
}

// The same subtree with fast nodes (v1_hypot top levels): a climb lies on the
// kernel's critical path (the warp's next group waits for it, the last chain
// of climbs is the kernel's tail), and the exact intrinsics' dependent chain
// is ~5x longer.  A node whose larger operand is outside the fast domain (a
// +0 pair of padding, inf, huge/tiny values) or a NaN result: the exact path.
// WIDE: steps of up to 8 levels (the split kernel's plans); otherwise <= 6.
template <typename F, bool WIDE>
__device__ __forceinline__ F warp_group_bal(const F* vals, int64_t nvals, int64_t base, int f, int cr) {
  if (cr) return warp_group_bal_exact<F, WIDE>(vals, nvals, base, f, cr);
  const int lane = threadIdx.x & 31;
  bool bad = false;
  F v;
  int lv = 5;
  if (WIDE && f == 8) v = lane_bal_fast<F, 8>(vals, nvals, base, bad);
  else if (WIDE && f == 7) v = lane_bal_fast<F, 4>(vals, nvals, base, bad);
  else if (f == 6) {
    const int64_t i = base + 2 * lane;
    const F a = i < nvals ? __ldcg(vals + i) : F(0);
    const F b = i + 1 < nvals ? __ldcg(vals + i + 1) : F(0);
    v = v1h_fast<true>(a, b, bad);
  } else {
    const int64_t i = base + lane;
    v = (lane < (1 << f) && i < nvals) ? __ldcg(vals + i) : F(0);
    lv = f;
  }
  for (int l = 0; l < lv; ++l) v = v1h_fast<true>(v, __shfl_xor_sync(0xffffffffu, v, 1 << l), bad);
  // lanes >= 2^lv hold padding the result does not depend on
  if (__any_sync(0xffffffffu, lane < (1 << lv) && (bad || v != v)))
    return warp_group_bal_exact<F, WIDE>(vals, nvals, base, f, cr);
  return v;
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------------------------------
// Last combine step of the split kernel without a counter (small calls: no
// counter to clear, no release fence, no atomic round trip).  Each input of
// the last step is written by the warp that produced it into its 16-byte slot
// together with the call's 64-bit tag (t1, t2) -- {lo32, t1, hi32, t2}, each
// 8-byte half one store/load unit (the flag-in-data scheme of the peer
// exchange, nrmf_p2p.cuh) -- and ONE warp (CTA 0, warp 1: it has no group work
// of its own after its batch) polls the slots until every one carries the
// tag, evaluates the step's balanced subtree in registers (the same tree as
// warp_group_bal), clears the slots it read and writes the root.
// The tag must never be found in stale memory: the workspace header holds a
// 64-bit count of completed calls c (read by every producer at its start,
// advanced by the combiner after the last slot arrived, so graph replays
// work), and the tag is a 64-bit hash of (c + 1, the header's address), both
// halves odd.  A slot is only ever matched by the tag it was written with:
// stale slots of this layout were cleared by the call that read them (even if
// the header was later reset by another call reusing the workspace, its tag
// sequence restarts on cleared slots), slots written by another layout carry
// tags of another address, and garbage matches with probability 2^-64.  Only
// one warp waits, on producers that never wait themselves, so the grid needs
// no co-residency.
__device__ __forceinline__ uint64_t ll_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// this call's number c + 1 (the combiner stores it back) and its tag
template <typename F>
__device__ __forceinline__ uint64_t ll_call(const TreeJob<F>& job) {
  return *reinterpret_cast<volatile unsigned long long*>(job.ll) + 1ull;
}
__device__ __forceinline__ uint64_t ll_tag(const char* ll, uint64_t call) {
  return ll_mix(call ^ ll_mix(reinterpret_cast<uintptr_t>(ll))) | 0x0000000100000001ull;
}
template <typename F>
__device__ __forceinline__ void ll_store(const TreeJob<F>& job, int64_t i, F v, uint64_t tag) {
  NRMF_TRACE(9, 0, 0);
  if ((threadIdx.x & 31) == 0) {
    uint32_t lo, hi;
    to_words(v, lo, hi);
    st_ll2_gpu(job.ll + 16 * (i + 1), lo, hi, (uint32_t)tag, (uint32_t)(tag >> 32));
  }
}
// KP inputs per lane (lanes < 2^f when f <= 5): poll, then the fast tree with
// the exact fallback (as warp_group_bal: any flagged node or NaN).
template <typename F, int KP>
__device__ __noinline__ F ll_gather_combine(char* ll, int64_t nin, int f, int cr, uint64_t tag) {
  const uint32_t t1 = (uint32_t)tag, t2 = (uint32_t)(tag >> 32);
  const int lane = threadIdx.x & 31;
  F a[KP];
  bool ready[KP];
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    const int64_t i = (int64_t)lane * KP + j;
    a[j] = F(0);
    ready[j] = !(i < nin && (KP > 1 || lane < (1 << f)));
  }
  // the lane's last slot index in range (slots past the inputs are re-read
  // harmlessly: their results are ignored)
  const int64_t i_last = nin - 1 < (int64_t)lane * KP ? nin - 1 : (int64_t)lane * KP + KP - 1;
  for (long long spins = 0;; ++spins) {
    // every slot of the lane is loaded in one round, all loads issued before
    // the first compare: one L2 round trip per round, not KP dependent ones
    uint32_t lo[KP], e0[KP], hi[KP], e1[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const int64_t i = (int64_t)lane * KP + j;
      ld_ll_gpu(ll + 16 * ((i < i_last ? i : i_last) + 1), lo[j], e0[j], hi[j], e1[j]);
    }
    bool all = true;
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      if (ready[j]) continue;
      if (e0[j] == t1 && e1[j] == t2) {
        a[j] = from_words<F>(lo[j], hi[j]);
        ready[j] = true;
      } else {
        all = false;
      }
    }
#ifdef NRMF_PROBE_TRACE2
    if (spins == 0) NRMF_TRACE(3, 0, 0);  // first poll round done
    if (spins == 1) NRMF_TRACE(2, 0, 0);  // second
#endif
    if (__all_sync(0xffffffffu, all)) {
#ifdef NRMF_PROBE_TRACE2
      if ((threadIdx.x & 31) == 0 && g_trace != nullptr)
        g_trace[((unsigned long long)blockIdx.x * 32 + (threadIdx.x >> 5)) * 16 + 7] = (unsigned long long)spins + 1;
#endif
      break;
    }
    if (spins > (1ll << 26)) {  // never: every producer of the step writes its slot
#pragma unroll
      for (int j = 0; j < KP; ++j)
        if (!ready[j]) a[j] = sizeof(F) == 8 ? F(__longlong_as_double(0x7ff8000000000000ll)) : F(__int_as_float(0x7fc00000));
      break;
    }
    if (spins > 32) __nanosleep(32);
  }
  NRMF_TSTAMP(t_polled);
  // clear the slots read: a later call with this layout whose call number
  // repeats (header reset by another call sharing the workspace) finds no
  // stale match
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    const int64_t i = (int64_t)lane * KP + j;
    if (i < nin && (KP > 1 || lane < (1 << f))) st_ll2_gpu(ll + 16 * (i + 1), 0u, 0u, 0u, 0u);
  }
  const int lv = f < 5 ? f : 5;
  bool bad = cr != 0;
  F v;
  NRMF_TSTAMP(t_cleared);
  if (!bad) {
    F b[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) b[j] = a[j];
    in_lane_levels<F, KP>(b, bad);
    v = b[0];
    NRMF_TSTAMP(t_inlane);
    for (int l = 0; l < lv; ++l) v = v1h_fast<true>(v, __shfl_xor_sync(0xffffffffu, v, 1 << l), bad);
    bad = __any_sync(0xffffffffu, lane < (1 << lv) && (bad || v != v));
    NRMF_TSTAMP(t_shfl);
    NRMF_TRACE_AT(10, t_polled);
    NRMF_TRACE_AT(11, t_cleared);
    NRMF_TRACE_AT(12, t_inlane);
    NRMF_TRACE_AT(13, t_shfl);
  }
  if (bad) {
#pragma unroll
    for (int st = 1; st < KP; st <<= 1)
#pragma unroll
      for (int j = 0; j < KP; j += 2 * st) a[j] = top_node(a[j], a[j + st], cr);
    v = a[0];
    for (int l = 0; l < lv; ++l) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, 1 << l), cr);
  }
  return v;
}
// Fan-in 256 split over two polling warps (CTA 0's warps 1 and 2): warp
// `half` polls slots [128 half, 128 half + 128), 4 per lane (a poll round of
// 4 loads per lane returns sooner than one of 8 under load), clears them and
// evaluates its 128-input subtree (2 in-lane + 5 shuffle levels, checked fast
// nodes).  Warp 2 leaves its raw inputs, value and flag in xch[0..129] and
// meets warp 1 at named barrier 1; warp 1 evaluates the top node, or -- any
// flagged node or NaN -- the whole 256-input subtree with exact nodes from its
// registers and xch.  The same tree as ll_gather_combine<F, 8>.  Returns the
// root in warp 1 (meaningless in warp 2).
template <typename F>
__device__ __noinline__ F ll_gather_half(char* ll, int64_t nin, int cr, uint64_t tag, int half, F* xch) {
  constexpr int KP = 4;
  const uint32_t t1 = (uint32_t)tag, t2 = (uint32_t)(tag >> 32);
  const int lane = threadIdx.x & 31;
  const int64_t base = (int64_t)half * 128 + (int64_t)lane * KP;
  F a[KP];
  bool ready[KP];
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    a[j] = F(0);
    ready[j] = !(base + j < nin);
  }
  for (long long spins = 0;; ++spins) {
    uint32_t lo[KP], e0[KP], hi[KP], e1[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const int64_t i = base + j < nin ? base + j : (nin > 0 ? nin - 1 : 0);
      ld_ll_gpu(ll + 16 * (i + 1), lo[j], e0[j], hi[j], e1[j]);
    }
    bool all = true;
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      if (ready[j]) continue;
      if (e0[j] == t1 && e1[j] == t2) {
        a[j] = from_words<F>(lo[j], hi[j]);
        ready[j] = true;
      } else {
        all = false;
      }
    }
    if (__all_sync(0xffffffffu, all)) break;
    if (spins > (1ll << 26)) {  // never: every producer of the step writes its slot
#pragma unroll
      for (int j = 0; j < KP; ++j)
        if (!ready[j]) a[j] = sizeof(F) == 8 ? F(__longlong_as_double(0x7ff8000000000000ll)) : F(__int_as_float(0x7fc00000));
      break;
    }
    if (spins > 32) __nanosleep(32);
  }
  bool bad = cr != 0;
  F v = F(0);
  if (!bad) {
    F b[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) b[j] = a[j];
    in_lane_levels<F, KP>(b, bad);
    v = b[0];
    for (int l = 0; l < 5; ++l) v = v1h_fast<true>(v, __shfl_xor_sync(0xffffffffu, v, 1 << l), bad);
    bad = __any_sync(0xffffffffu, bad || v != v);
  }
#pragma unroll
  for (int j = 0; j < KP; ++j)
    if (base + j < nin) st_ll2_gpu(ll + 16 * (base + j + 1), 0u, 0u, 0u, 0u);
  if (half == 1) {
#pragma unroll
    for (int j = 0; j < KP; ++j) xch[lane * KP + j] = a[j];
    if (lane == 0) {
      xch[128] = v;
      xch[129] = bad ? F(1) : F(0);
    }
    asm volatile("bar.sync 1, 64;" ::: "memory");
    return v;
  }
  asm volatile("bar.sync 1, 64;" ::: "memory");
  const F v1 = xch[128];
  bool bad2 = bad || xch[129] != F(0);
  F root = F(0);
  if (!bad2) {
    root = v1h_fast<true>(v, v1, bad2);
    bad2 = bad2 || root != root;
  }
  if (bad2) {  // the whole subtree with exact nodes (v1_hypot or cr_hypot)
    F e[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      F c[KP];
#pragma unroll
      for (int j = 0; j < KP; ++j) c[j] = hh == 0 ? a[j] : xch[lane * KP + j];
#pragma unroll
      for (int st = 1; st < KP; st <<= 1)
#pragma unroll
        for (int j = 0; j < KP; j += 2 * st) c[j] = top_node(c[j], c[j + st], cr);
      F w = c[0];
      for (int l = 0; l < 5; ++l) w = top_node(w, __shfl_xor_sync(0xffffffffu, w, 1 << l), cr);
      e[hh] = w;
    }
    root = top_node(e[0], e[1], cr);
  }
  return root;
}

template <typename F>
__device__ void ll_combine(const TreeJob<F>& job, uint64_t call, F* xch = nullptr) {
  const int K = job.nsteps - 1;
  const int f = job.lg_fan[K];
  const uint64_t tag = ll_tag(job.ll, call);
  NRMF_TRACE(6, 0, 0);
  F v;
  if (NRMF_LL_TWO && f == 8 && xch != nullptr) {
    v = ll_gather_half<F>(job.ll, job.nin[K], job.top_cr, tag, (threadIdx.x >> 5) == 2 ? 1 : 0, xch);
    if ((threadIdx.x >> 5) == 2) return;  // warp 2: its half is in xch
  } else
  switch (f) {
    case 8: v = ll_gather_combine<F, 8>(job.ll, job.nin[K], f, job.top_cr, tag); break;
    case 7: v = ll_gather_combine<F, 4>(job.ll, job.nin[K], f, job.top_cr, tag); break;
    case 6: v = ll_gather_combine<F, 2>(job.ll, job.nin[K], f, job.top_cr, tag); break;
    default: v = ll_gather_combine<F, 1>(job.ll, job.nin[K], f, job.top_cr, tag); break;
  }
  __syncwarp();
  if ((threadIdx.x & 31) == 0) *reinterpret_cast<volatile unsigned long long*>(job.ll) = call;  // completed calls
  write_root(job, v);
  NRMF_TRACE(8, 0, 0);
}

// Node `idx` of step-k input level has been stored by lane 0 and announced
// with counter value `old`.  If this warp was the last arrival of its group,
// evaluate the group's subtree and climb.  Last-arriver combine: who computes
// a node depends on timing, what is computed never does.
template <typename F, bool WIDE = false>
__device__ void climb(const TreeJob<F>& job, int k, int64_t idx, unsigned old, uint64_t ll_t = 0) {
  const int lane = threadIdx.x & 31;
  while (true) {
    const int f = job.lg_fan[k];
    const int64_t g = idx >> f;
    const int64_t fan = int64_t(1) << f;
    const int64_t rem = job.nin[k] - g * fan;
    const unsigned expect = (unsigned)(rem < fan ? rem : fan);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != expect - 1) return;
    NRMF_TRACE(2, k, 0);
    NRMF_JITTER(3);
    if (lane == 0) {
      // acquire by the lane that read the counter: the other arrivals' values
      // (released by their atomics) are visible to it ...
      fence_acq_rel_gpu();
      job.cnt[job.cnt_off[k] + g] = 0u;  // ready for the next call
    }
    __syncwarp();  // ... and to every lane of the warp (bar.warp.sync orders memory)
    const F v = warp_group_bal<F, WIDE>(job.vals + job.val_off[k], job.nin[k], g * fan, f, job.top_cr);
    NRMF_TRACE(3, k, 0);
    if (k + 1 == job.nsteps) {
      write_root(job, v);
      return;
    }
    if (WIDE && job.ll != nullptr && k + 2 == job.nsteps) {  // the last step by slots (split kernel)
      ll_store(job, g, v, ll_t);
      return;
    }
    NRMF_JITTER(1);
    if (lane == 0) {
      job.vals[job.val_off[k + 1] + g] = v;
      NRMF_JITTER(2);
      old = atom_add_release(job.cnt + job.cnt_off[k + 1] + (g >> job.lg_fan[k + 1]), 1u);
    }
    ++k;
    idx = g;
  }
}

// Tile tau -> (base pointer, full?).  One 64-bit division per tile at most.
template <typename F>
__device__ __forceinline__ bool tile_at(const TreeJob<F>& job, int64_t tau, const F*& base, int64_t& remv) {
  const int64_t col = job.ld == 0 ? 0 : (job.tpc == 1 ? tau : tau / job.tpc);
  const int64_t tt = tau - col * job.tpc;
  base = job.x + col * job.ld + tt * (int64_t)kTile;
  remv = job.len - tt * (int64_t)kTile;
  return remv >= kTile;
}

// SMEM-ring loader: batches of the warp's tile NT-tuples (NT consecutive
// tiles of a warp group, all full), in the order the warp visits them, arrive
// by TMA bulk copy (cp.async.bulk, mbarrier complete_tx): for every batch b,
// one stage per tile of the tuple.  Leaves are read from shared memory per
// interleaved chunk (get_row), which keeps only the chunk's rows in registers.
template <typename F, int NT>
struct PipeLoader {
  static constexpr int BPI = 1;
  static constexpr bool kMaybePadding = false;
  __device__ __forceinline__ bool all_padding(int) const { return false; }

  uint32_t ring_s, bar_s;     // shared-window addresses of this warp's ring and barriers
  uint32_t consumed, issued;  // stages consumed / issued (warp-uniform)
  int64_t p_grp;              // producer: warp group of the next tuple to load
  int p_k;                    // producer: first tile (within the group) of that tuple
  int p_b;                    // producer: batch index
  int p_t;                    // producer: tile of the tuple
  const F* p_base[NT];        // producer: bases of the tuple's tiles
  // job geometry (copied: no pointer to the kernel parameter)
  const F* x;
  int64_t n_items, tpc, ld, len, W, n_groups;
  int G;
  uint64_t policy;

  __device__ __forceinline__ bool tile(int64_t tau, const F*& base) const {
    // vector mode (ld == 0): one "column" holding every tile, no division
    const int64_t col = ld == 0 ? 0 : (tpc == 1 ? tau : tau / tpc);
    const int64_t tt = tau - col * tpc;
    base = x + col * ld + tt * (int64_t)kTile;
    return len - tt * (int64_t)kTile >= kTile;
  }
  // is tuple (grp, k) made of NT full tiles with data?
  __device__ __forceinline__ bool tuple_ok(int64_t grp, int k, const F* (&bases)[NT]) const {
    bool ok = k + NT <= G;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int64_t tau = grp * G + k + t;
      ok = ok && tau < n_items && tile(tau, bases[t]);
    }
    return ok;
  }
  __device__ __forceinline__ void seek() {
    while (p_grp < n_groups) {
      if (tuple_ok(p_grp, p_k, p_base)) return;
      p_k += NT;
      if (p_k >= G) {
        p_k = 0;
        p_grp += W;
      }
    }
  }
  __device__ __forceinline__ void issue() {
    if (p_grp >= n_groups) return;
    const uint32_t s = issued % kStages;
    if ((threadIdx.x & 31) == 0)
      bulk_load(ring_s + s * kBatchBytes, p_base[p_t] + (int64_t)p_b * kBatch * Cfg<F>::LANES, kBatchBytes,
                bar_s + s * 8, policy);
    ++issued;
    if (++p_t == NT) {
      p_t = 0;
      if (++p_b == Cfg<F>::J / kBatch) {
        p_b = 0;
        p_k += NT;
        if (p_k >= G) {
          p_k = 0;
          p_grp += W;
        }
        seek();
      }
    }
  }
  __device__ __forceinline__ void begin(int) {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const uint32_t c = consumed + t;
      mbar_wait(bar_s + (c % kStages) * 8, (c / kStages) & 1);
    }
  }
  __device__ __forceinline__ void get_row(int t, int row, F (&o)[Cfg<F>::V]) const {
#ifdef NRMF_FAKE_SMEM  // dev-only timing probe: leaves synthesized in registers (wrong results)
#pragma unroll
    for (int v = 0; v < Cfg<F>::V; ++v) o[v] = F(1) + F(row * 7 + v + t) * F(1e-3) + F(consumed & 3);
    return;
#endif
    const uint32_t addr = ring_s + ((consumed + t) % kStages) * kBatchBytes + (threadIdx.x & 31) * 16 +
                          row * (kBatchBytes / kBatch);
    if constexpr (sizeof(F) == 8) {
      double a0, a1;
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a0), "=d"(a1) : "r"(addr) : "memory");
      o[0] = a0;
      o[1 % Cfg<F>::V] = a1;
    } else {
      float a0, a1, a2, a3;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3)
                   : "r"(addr) : "memory");
      o[0] = a0;
      o[1 % Cfg<F>::V] = a1;
      o[2 % Cfg<F>::V] = a2;
      o[3 % Cfg<F>::V] = a3;
    }
  }
  __device__ __forceinline__ void end(int) {
    __syncwarp();  // every lane holds its leaves: the stages may be refilled
    consumed += NT;
#pragma unroll
    for (int t = 0; t < NT; ++t) issue();
  }
};

// CTA area of the stream kernel (after the kWarps warp blocks): the first
// combine step in shared memory.  kCtaSlots rounds in flight: [values:
// kCtaSlots x 16 F][arrival counters: kCtaSlots u32][round tags: kCtaSlots u32].
constexpr int kCtaSlots = 4;
template <typename F>
struct CtaSmem {
  static constexpr uint32_t kVals = 0;
  static constexpr uint32_t kCnt = kCtaSlots * 16 * sizeof(F);
  static constexpr uint32_t kTag = kCnt + kCtaSlots * 4;
  static constexpr uint32_t kBytes = kTag + kCtaSlots * 4;
};

// Per-warp shared-memory block of the stream kernel (offsets from its base):
// [ring: kStages x 4 KiB][stash][group thread values][mbarriers], 128-aligned.
// UNAL: the ring of the unaligned-vector stream kernel: a stage holds the
// 16-byte-aligned span around its batch (4 KiB + 16 bytes).
template <typename F, bool UNAL = false>
struct WarpSmem {
  static constexpr uint32_t kStage = UNAL ? kBatchBytes + 16 : kBatchBytes;
  static constexpr uint32_t kRing = 0;
  static constexpr uint32_t kStash = kStages * kStage;
  static constexpr uint32_t kXs = kStash + kStashBytes<F>;
  static constexpr uint32_t kBars = kXs + kGroupXsBytes<F>;
  static constexpr uint32_t kBytes = (kBars + kStages * 8 + 127) / 128 * 128;
};
static_assert(kWarps * WarpSmem<double, true>::kBytes + CtaSmem<double>::kBytes <= 227 * 1024 &&
                  kWarps * WarpSmem<float, true>::kBytes + CtaSmem<float>::kBytes <= 227 * 1024,
              "stream kernel shared memory");

// Stream loader (contiguous tiles: a vector, or back-to-back columns of T
// multiple length; 16-byte aligned): the batches of a full warp group (G
// consecutive full tiles, G*T contiguous elements) are contiguous in memory,
// and a warp visits groups gw, gw+W, ...  The producer is a pointer walk:
// +4 KiB per batch, +(W-1) groups at a group's end; it stops after the warp's
// last full group (a partial last group of the call goes through
// single_tile).  Every consumed stage is refilled at once, so the slot to fill
// is always the one just consumed.  State: 5 registers plus kernel-uniform
// values.
// GAP: column blocks with a gap between columns (ld > rows, rows a multiple
// of T, 16-byte aligned columns): the walk also skips (ld - rows) elements at
// every column end, and a new group's start is computed from its tile index.
// UNAL (vectors whose base is a multiple of sizeof(F) but not of 16 bytes,
// the paper's unaligned case): a batch starting at byte offset
// `off` = x mod 16 is fetched as the aligned span [B - off, B - off + 4 KiB
// + 16), and the lanes read their rows `off` bytes into the stage with
// element-sized shared loads.  The span stays inside the array because the
// kernel streams only groups with a group before them (group >= 1) and at
// least 16 bytes of the array after them (the others go through single_tile).
template <typename F, bool GAP = false, bool UNAL = false>
struct StreamLoader {
  static constexpr int BPI = 1;
  static constexpr bool kMaybePadding = false;
  __device__ __forceinline__ bool all_padding(int) const { return false; }
  using L = WarpSmem<F, UNAL>;

  uint32_t my_s;         // this warp's block (WarpSmem)
  uint32_t consumed;     // stages consumed (warp-uniform)
  const char* p_ptr;     // next batch to load
  int p_left;            // batches left in its group
  int groups_left;       // further groups after it (-1: nothing left to load)
  int group_batches;     // G * J / kBatch            (kernel-uniform)
  int64_t skip_bytes;    // (W - 1) groups in bytes   (kernel-uniform)
  // GAP only
  int p_grp;             // group being loaded
  int col_left;          // batches left in the current column
  int grp_step;          // W                          (kernel-uniform)
  int col_batches;       // tpc * J / kBatch           (kernel-uniform)
  int64_t col_skip;      // (ld - rows) in bytes       (kernel-uniform)
  int64_t tpc, ld;       // tiles per column, leading dimension (kernel-uniform)
  const F* x;
  int g0;                // (kernel-uniform)
  uint32_t off;          // UNAL only: x mod 16 in bytes (kernel-uniform)

  __device__ __forceinline__ void seek(int grp) {
    const int64_t tau = (int64_t)grp << g0;
    const int64_t col = tau / tpc, tt = tau - col * tpc;
    p_ptr = reinterpret_cast<const char*>(x + col * ld + tt * (int64_t)kTile);
    col_left = (int)(tpc - tt) * (Cfg<F>::J / kBatch);
  }

  __device__ __forceinline__ void issue(uint32_t slot) {
    if (groups_left < 0) return;
    if ((threadIdx.x & 31) == 0)
      bulk_load(my_s + L::kRing + slot * L::kStage, UNAL ? p_ptr - off : p_ptr, L::kStage,
                my_s + L::kBars + slot * 8, stream_l2_policy());
    p_ptr += kBatchBytes;
    if (GAP && --col_left == 0) {
      col_left = col_batches;
      p_ptr += col_skip;
    }
    if (--p_left == 0) {
      p_left = group_batches;
      --groups_left;
      if (GAP) {
        p_grp += grp_step;
        if (groups_left >= 0) seek(p_grp);
      } else {
        p_ptr += skip_bytes;
      }
    }
  }
  __device__ __forceinline__ void begin(int) {
    mbar_wait(my_s + L::kBars + (consumed % kStages) * 8, (consumed / kStages) & 1);
  }
  // consume `nb` batches without reading them (the ring keeps streaming)
  __device__ __noinline__ void drain(int nb) {
    for (int i = 0; i < nb; ++i) {
      begin(i);
      end(i);
    }
  }
  __device__ __forceinline__ void get_row(int, int row, F (&o)[Cfg<F>::V]) const {
#ifdef NRMF_FAKE_SMEM  // dev-only energy/timing probe: leaves synthesized in registers (wrong results)
#pragma unroll
    for (int v = 0; v < Cfg<F>::V; ++v) o[v] = F(1) + F(row * 7 + v) * F(1e-3) + F(consumed & 3);
    return;
#endif
    const uint32_t addr = my_s + L::kRing + (consumed % kStages) * L::kStage + (threadIdx.x & 31) * 16 +
                          row * (kBatchBytes / kBatch) + (UNAL ? off : 0u);
    if constexpr (UNAL) {
      // element-aligned only: one shared load per element
#pragma unroll
      for (int v = 0; v < Cfg<F>::V; ++v) ld_shared(addr + v * (uint32_t)sizeof(F), o[v]);
    } else if constexpr (sizeof(F) == 8) {
      double a0, a1;
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a0), "=d"(a1) : "r"(addr) : "memory");
      o[0] = a0;
      o[1 % Cfg<F>::V] = a1;
    } else {
      float a0, a1, a2, a3;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3)
                   : "r"(addr) : "memory");
      o[0] = a0;
      o[1 % Cfg<F>::V] = a1;
      o[2 % Cfg<F>::V] = a2;
      o[3 % Cfg<F>::V] = a3;
    }
  }
  __device__ __forceinline__ void end(int) {
    __syncwarp();  // every lane holds its leaves: the stage may be refilled
    const uint32_t slot = consumed % kStages;
    ++consumed;
    issue(slot);
  }
};

// Step 0 of the combine inside the CTA (stream kernel, CTA-major warps): the
// 16 warp groups of CTA-block b = grp >> 4 are the 16 warps' groups of one
// round (grp & 15 == warp), an aligned subtree of 16 groups.  Each warp
// deposits its group value in the round's shared-memory slot and counts in.
// The block is then evaluated (4 levels, fast nodes with exact fallback) and
// announced to the global step 1 -- not by its last arriver but by the first
// warp to finish its NEXT round, which finds the slot complete and claims it:
// the last arriver of a round is systematically the same, slowest warp of the
// CTA (tools/trace_probe.py), and making it do the combine and the global
// climbs on top delayed it by ~3 us per round; it ended the kernel ~50 us
// after the others.  A warp without a next round claims at once (and the
// round's completer either has a next round, where it will try, or claims at
// once), so every round is claimed exactly once (CAS on the slot's tag).
// Slot r % kCtaSlots serves round r + kCtaSlots after the claimer frees it
// (tag r -> r|claimed -> r + kCtaSlots); a warp that far ahead waits.
constexpr unsigned kClaimed = 0x80000000u;
__device__ __forceinline__ unsigned ld_volatile_shared_u32(uint32_t a) {
  unsigned v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_cta_shared_u32(uint32_t a) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_u32(uint32_t a, unsigned v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_cta_shared(uint32_t a, unsigned v) {
  asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned cas_acq_rel_cta_shared(uint32_t a, unsigned cmp, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void fence_acq_rel_cta() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }

// Claim round rr's slot if complete and unclaimed; if claimed, evaluate CTA
// block b and announce it to step 1 (climbing if last there).
template <typename F>
__device__ __forceinline__ void cta_try(const TreeJob<F>& job, uint32_t cta_s, int rr, int b, int n_groups) {
  using C = CtaSmem<F>;
  const int lane = threadIdx.x & 31;
  const uint32_t slot = (uint32_t)rr & (kCtaSlots - 1);
  const uint32_t vs = cta_s + C::kVals + slot * 16 * (uint32_t)sizeof(F);
  const uint32_t cs = cta_s + C::kCnt + slot * 4, ts = cta_s + C::kTag + slot * 4;
  const int expect = n_groups - 16 * b < 16 ? n_groups - 16 * b : 16;
  unsigned got = 0;
  NRMF_JITTER(4);
  if (lane == 0 && ld_volatile_shared_u32(ts) == (unsigned)rr && ld_volatile_shared_u32(cs) == (unsigned)expect) {
    NRMF_JITTER(5);
    got = cas_acq_rel_cta_shared(ts, (unsigned)rr, (unsigned)rr | kClaimed) == (unsigned)rr;
  }
  if (!__shfl_sync(0xffffffffu, got, 0)) return;
  // lane 0 read the complete count (written by the arrivals' release adds):
  // its fence makes every arrival's value visible to it, and __syncwarp
  // extends that ordering to the warp's other lanes
  if (lane == 0) fence_acq_rel_cta();
  __syncwarp();
  NRMF_TRACE(2, 15, 0);
  F v = F(0);
  if (lane < expect) ld_shared(vs + lane * (uint32_t)sizeof(F), v);
  bool bad = job.top_cr != 0;
  if (!bad) {
    F u = v;
    for (int l = 0; l < 4; ++l) u = v1h_fast<true>(u, __shfl_xor_sync(0xffffffffu, u, 1 << l), bad);
    bad = __any_sync(0xffffffffu, lane < 16 && (bad || u != u));  // lanes >= 16: padding, not used
    if (!bad) v = u;
  }
  if (bad)
    for (int l = 0; l < 4; ++l) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, 1 << l), job.top_cr);
  __syncwarp();
  NRMF_JITTER(6);
  if (lane == 0) {  // free the slot for round rr + kCtaSlots (its values are read)
    st_shared_u32(cs, 0u);
    fence_acq_rel_cta();
    st_shared_u32(ts, (unsigned)(rr + kCtaSlots));
  }
  NRMF_TRACE(3, 15, 0);
  if (job.nsteps == 1) {
    write_root(job, v);
    return;
  }
  unsigned old1 = 0;
  if (lane == 0) {
    job.vals[job.val_off[1] + b] = v;
    old1 = atom_add_release(job.cnt + job.cnt_off[1] + (b >> job.lg_fan[1]), 1u);
  }
  climb(job, 1, b, old1);
}

// Group grp (round r of this warp) has value gv: deposit it, then claim the
// previous round and, without a next round, this one.
template <typename F>
__device__ __forceinline__ void cta_arrive(const TreeJob<F>& job, uint32_t cta_s, int grp, int r, int W, F gv,
                                           int n_groups) {
  using C = CtaSmem<F>;
  const int lane = threadIdx.x & 31;
  const uint32_t slot = (uint32_t)r & (kCtaSlots - 1);
  if (lane == 0) {
    const uint32_t ts = cta_s + C::kTag + slot * 4;
    // slot still serves round r - kCtaSlots until its claimer frees it; the
    // acquire orders this round's value store and count after the claimer's
    // reads and counter reset
    while (ld_acquire_cta_shared_u32(ts) != (unsigned)r) __nanosleep(64);
    NRMF_JITTER(7);
    st_shared(cta_s + C::kVals + (slot * 16 + (grp & 15)) * (uint32_t)sizeof(F), gv);
    NRMF_JITTER(8);
    red_add_release_cta_shared(cta_s + C::kCnt + slot * 4, 1u);
  }
  __syncwarp();
  NRMF_JITTER(9);
  const int b = grp >> 4;
  if (r >= 1) cta_try<F>(job, cta_s, r - 1, b - W / 16, n_groups);
  if (grp + W >= n_groups) cta_try<F>(job, cta_s, r, b, n_groups);
}

// Value of tile tau when it is not part of a pipelined tuple: a full tile by
// LDG (fast nodes, exact fallback), a partial one by the exact path, +0 for a
// padding tile beyond the data.
template <typename F, bool VEC>
__device__ __forceinline__ F single_tile(const TreeJob<F>& job, int64_t tau) {
  if (tau >= job.n_items) return F(0);
  const F* tb;
  int64_t remv;
  if (tile_at(job, tau, tb, remv)) return VEC ? warp_tile<F, kVec>(tb) : warp_tile<F, kScalar>(tb);
  bool bad = false;
  const F v = warp_tile_padded<F>(tb, (int)remv, bad);
  if (!bad && v == v) return v;
  return warp_tile_exact<F, kPred>(tb, (int)remv);
}

// Values of tiles tau and tau + 1 (short columns: partial tiles of one
// length), beyond the data +0; bad or NaN: each tile by the exact path.
template <typename F>
__device__ __forceinline__ void short_pair(const TreeJob<F>& job, int64_t tau, F (&tv)[2]) {
  tv[0] = tv[1] = F(0);
  if (tau >= job.n_items) return;
  const F *tb0, *tb1;
  int64_t remv;
  tile_at(job, tau, tb0, remv);
  if (tau + 1 >= job.n_items) {
    tv[0] = single_tile<F, false>(job, tau);
    return;
  }
  tile_at(job, tau + 1, tb1, remv);
  bool bad = false;
  if (remv <= kBatch * Cfg<F>::LANES) warp_tiles_short2<F, true>(tb0, tb1, (int)remv, bad, tv[0], tv[1]);
  else warp_tiles_short2<F, false>(tb0, tb1, (int)remv, bad, tv[0], tv[1]);
  if (bad || tv[0] != tv[0] || tv[1] != tv[1]) {
    tv[0] = warp_tile_exact<F, kPred>(tb0, (int)remv);
    tv[1] = warp_tile_exact<F, kPred>(tb1, (int)remv);
  }
}

// SHORT: the element-load kernel's instance for short column blocks (every
// column one partial tile of <= 2 batches), with the paired-column path; the
// plain element-load instance keeps its code.
template <typename F, bool TMA, int NT, bool STREAM, bool GAP = false, bool UNAL = false, bool SHORT = false>
__global__ void __launch_bounds__(kThreads, NRMF_MIN_BLOCKS) nrmf_tree_kernel(const TreeJob<F> job) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr bool kPipe = TMA && NRMF_USE_TMA;
  constexpr bool kStream = kPipe && STREAM && NT == 1;
  static_assert(!UNAL || (kStream && !GAP), "UNAL: the vector stream kernel only");
  using WS = WarpSmem<F, UNAL>;
  // tile loads outside the ring: 16-byte vectors unless the base is unaligned
  constexpr LoadMode kTileMode = UNAL ? kScalar : kVec;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // group and warp indices are 32-bit (a call has < 2^31 tiles: n < 2^43);
  // fewer live 64-bit values leave more registers to the node chains
  const int W = (int)gridDim.x * kWarps;
  // global warp index: CTA-major (a CTA streams kWarps consecutive groups)
  // when every warp has work; CTA-minor for calls with fewer groups than
  // warps, so that consecutive groups go to different SMs
  const int gw = job.cta_minor ? w * (int)gridDim.x + (int)blockIdx.x : (int)blockIdx.x * kWarps + w;
  const int G = 1 << job.g0;
  const int n_groups = (int)((job.n_items + G - 1) >> job.g0);
  // stream mode: warp groups made only of full tiles (tiles are contiguous:
  // a vector, or columns with ld == rows == a multiple of T)
  int n_full = kStream ? (int)((job.ld == 0 ? job.len / kTile : job.n_items) >> job.g0) : 0;
  // UNAL: the first streamed group is 1 (group 0's span would start before
  // x), and the last full group is streamed only if at least 16 bytes of the
  // array follow it (its last span ends 16 - off bytes past the group)
  const uint32_t u_off = UNAL ? (uint32_t)(reinterpret_cast<uintptr_t>(job.x) & 15u) : 0u;
  if (UNAL && n_full > 0 &&
      (job.len - ((int64_t)n_full << job.g0) * kTile) * (int64_t)sizeof(F) < 16)
    --n_full;
  const int s_lo = UNAL ? 1 : 0;

  StreamLoader<F, GAP, UNAL> sl;
  if (kStream) {
    using L = WS;
    sl.my_s = smem_u32(smem) + w * L::kBytes;
    if (lane == 0) {
      for (int st = 0; st < kStages; ++st) mbar_init(sl.my_s + L::kBars + st * 8, 1);
      fence_mbar_init();
    }
    __syncwarp();
    sl.consumed = 0;
    sl.group_batches = G * (Cfg<F>::J / kBatch);
    sl.p_left = sl.group_batches;
    // groups gw, gw + W, ... in [s_lo, n_full): this warp streams 1 + groups_left of them
    const int first = gw < s_lo ? gw + W : gw;
    sl.groups_left = first < n_full ? (int)((n_full - 1 - first) / W) : -1;
    sl.off = u_off;
    if (GAP) {
      sl.x = job.x;
      sl.tpc = job.tpc;
      sl.ld = job.ld;
      sl.grp_step = W;
      sl.col_batches = (int)job.tpc * (Cfg<F>::J / kBatch);
      sl.col_skip = (job.ld - job.len) * (int64_t)sizeof(F);
      sl.g0 = job.g0;
      sl.p_grp = gw;
      if (sl.groups_left >= 0) sl.seek(gw);
    } else {
      sl.p_ptr = reinterpret_cast<const char*>(job.x + first * G * (int64_t)kTile);
      sl.skip_bytes = (W - 1) * G * (int64_t)kTile * (int64_t)sizeof(F);
    }
    for (int st = 0; st < kStages; ++st) sl.issue(st);
  }
  const uint32_t cta_s = smem_u32(smem) + kWarps * WS::kBytes;
  if (kStream && job.cta_step0) {
    if (threadIdx.x < kCtaSlots) {
      st_shared_u32(cta_s + CtaSmem<F>::kCnt + threadIdx.x * 4, 0u);
      st_shared_u32(cta_s + CtaSmem<F>::kTag + threadIdx.x * 4, threadIdx.x);
    }
    __syncthreads();
  }

  PipeLoader<F, NT> pl;
  if (kPipe && !kStream) {
    pl.ring_s = smem_u32(smem + w * (kStages * kBatchBytes));
    pl.bar_s = smem_u32(smem + kWarps * kStages * kBatchBytes) + w * kStages * 8;
    if (lane == 0) {
      for (int st = 0; st < kStages; ++st) mbar_init(pl.bar_s + st * 8, 1);
      fence_mbar_init();
    }
    __syncwarp();
    pl.consumed = pl.issued = 0;
    pl.p_grp = gw;
    pl.p_k = pl.p_b = pl.p_t = 0;
    pl.W = W;
    pl.G = G;
    pl.n_groups = n_groups;
    pl.policy = stream_l2_policy();
    pl.x = job.x;
    pl.n_items = job.n_items;
    pl.tpc = job.tpc;
    pl.ld = job.ld;
    pl.len = job.len;
    pl.seek();
    for (int st = 0; st < kStages; ++st) pl.issue();
  }

  NRMF_TRACE(0, 0, 0);
  // safe mode (stream kernel): after a group that needed the exact path, the
  // warp evaluates its next groups with the safe node straight from the ring
  // (no fast pass to discard, no re-read from global memory) until a group
  // whose leaves all lie in the fast domain.  Same tree, same bits.
  // (fp64 only: C5 is an fp64 config, and the fp32 kernel's hot loop lost
  // 2 % to the extra code)
  constexpr bool kSafeMode = NRMF_SAFE_MODE && kStream && sizeof(F) == 8;
  bool safe_mode = false;
  for (int grp = gw, rnd = 0; grp < n_groups; grp += W, ++rnd) {
    F s0[1], s1[1], s2[1], gv[1];
    NodeTop ne{job.top_cr};
    bool group_done = false;
    if (kStream && !(kSafeMode && safe_mode) && grp >= s_lo && grp < n_full) {
      // full warp group of a vector call: per tile the thread values go to
      // the warp's xs area, then the cross-thread and group levels of all G
      // tiles at once (group_cross).  A flagged leaf or a NaN tile value
      // recomputes the group with the exact path below.
      NodeFast node;
      for (int k = 0; k < G; ++k) {  // rolled
        const F c = warp_tile_lanes<F>(sl, node, sl.my_s + WS::kStash);
        st_shared(sl.my_s + WS::kXs + (k * 32 + lane) * (uint32_t)sizeof(F), c);
#if NRMF_SKIP_FLAGGED
        // a flagged tile sends the whole group to the fallback: the group's
        // remaining batches are only drained from the ring, not evaluated
        if (k + 1 < G && __any_sync(0xffffffffu, node.bad)) {
          sl.drain((G - 1 - k) * (Cfg<F>::J / kBatch));
          break;
        }
#endif
      }
      __syncwarp();
#ifdef NRMF_PROBE_NO_GROUPCROSS  // dev-only timing probe: no cross-thread/group levels (wrong results)
      if (!__any_sync(0xffffffffu, node.bad)) {
        ld_shared(sl.my_s + WS::kXs + lane * (uint32_t)sizeof(F), gv[0]);
        group_done = true;
      }
#else
      if (!__any_sync(0xffffffffu, node.bad))
        group_done = group_cross<F>(node, sl.my_s + WS::kXs, G, job.top_cr, gv[0],
                                    job.tile_out != nullptr ? job.tile_out + grp * G : nullptr);
#endif
      if (!group_done) {
        // exact path: the G tile values through the xs area, then the lg G
        // group levels as a shuffle tree (contiguous pairs, the same tree)
        const uint32_t xs = sl.my_s + WS::kXs;
        for (int k = 0; k < G; ++k) {  // rolled
          const F* tb = job.x + (grp * G + k) * (int64_t)kTile;  // contiguous tiles
          if (GAP) {
            int64_t remv;
            tile_at(job, grp * G + k, tb, remv);  // a full tile of a gapped column block
          }
          const F tv = warp_tile_exact<F, kTileMode>(tb, kTile);
          if (lane == 0) {
            st_shared(xs + k * (uint32_t)sizeof(F), tv);
            if (job.tile_out != nullptr) job.tile_out[grp * G + k] = tv;
          }
        }
        __syncwarp();
        F v = F(0);
        if (lane < G) ld_shared(xs + lane * (uint32_t)sizeof(F), v);
        __syncwarp();
        for (int off = 1; off < G; off <<= 1) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, off), job.top_cr);
        gv[0] = v;
        group_done = true;
        if constexpr (kSafeMode) safe_mode = true;
      }
    }
    if constexpr (kSafeMode) {
    if (safe_mode && !group_done && grp >= s_lo && grp < n_full) {
      NodeSafeChk node;
      const uint32_t xs = sl.my_s + WS::kXs;
      for (int k = 0; k < G; ++k) {  // rolled
        F c = warp_tile_lanes<F>(sl, node, sl.my_s + WS::kStash);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) c = node(c, __shfl_xor_sync(0xffffffffu, c, off));
        if (lane == 0) {
          st_shared(xs + k * (uint32_t)sizeof(F), c);
          if (job.tile_out != nullptr) job.tile_out[grp * G + k] = c;
        }
      }
      __syncwarp();
      F v = F(0);
      if (lane < G) ld_shared(xs + lane * (uint32_t)sizeof(F), v);
      __syncwarp();
      for (int off = 1; off < G; off <<= 1) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, off), job.top_cr);
      gv[0] = v;
      group_done = true;
      safe_mode = __any_sync(0xffffffffu, node.bad);
    }
    }
    // short columns (every tile one column of rows <= 2 batches): two
    // columns at a time (warp_tiles_short2: element loads, any alignment),
    // merged like the loop below -- in the TMA column kernel and, for column
    // blocks that are not 16-byte aligned, the element-load kernel's SHORT
    // instance
    if ((TMA || (SHORT && NRMF_SHORT_PAIRS_ELEM)) && !kStream && NRMF_SHORT_PAIRS && !group_done &&
        job.tpc == 1 && job.ld != 0 && G >= 2 &&
        job.len <= 2 * kBatch * Cfg<F>::LANES) {
      for (int k = 0; k < G; k += 2) {  // rolled
        F tv[2];
        short_pair<F>(job, grp * G + k, tv);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int64_t tau = grp * G + k + t;
          if (job.tile_out != nullptr && lane == 0 && tau < job.n_items) job.tile_out[tau] = tv[t];
          gv[0] = tv[t];
          if (G == 8) counter_merge<F, 1, 8>(k + t, gv, s0, s1, s2, ne);
          else if (G == 4) counter_merge<F, 1, 4>(k + t, gv, s0, s1, s2, ne);
          else counter_merge<F, 1, 2>(k + t, gv, s0, s1, s2, ne);
        }
      }
      group_done = true;
    }
    // the stream kernel merges a (partial) group's tile values through its xs
    // area (groups of up to 16 tiles); the other kernels by counter_merge
    const bool xs_merge = kStream && !group_done;
    for (int k = 0; k < G && !group_done; k += NT) {  // rolled
      F tv[NT];
      const F* bases[NT];
      if (kPipe && !kStream && pl.tuple_ok(grp, k, bases)) {
        NodeFast node;
        warp_tiles_impl<F, NT>(pl, node, tv);
        const bool bad = __any_sync(0xffffffffu, node.bad);
#pragma unroll
        for (int t = 0; t < NT; ++t)
          if (bad || tv[t] != tv[t]) tv[t] = warp_tile_exact<F, kVec>(bases[t], kTile);
      } else {
#pragma unroll
        for (int t = 0; t < NT; ++t) tv[t] = (k + t < G) ? single_tile<F, TMA && !UNAL>(job, grp * G + k + t) : F(0);
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (k + t >= G) break;
        const int64_t tau = grp * G + k + t;
        if (job.tile_out != nullptr && lane == 0 && tau < job.n_items) job.tile_out[tau] = tv[t];
        gv[0] = tv[t];
        if (kStream) {
          if (lane == 0) st_shared(sl.my_s + WS::kXs + (k + t) * (uint32_t)sizeof(F), tv[t]);
          continue;
        }
        if (G == 8) counter_merge<F, 1, 8>(k + t, gv, s0, s1, s2, ne);
        else if (G == 4) counter_merge<F, 1, 4>(k + t, gv, s0, s1, s2, ne);
        else if (G == 2) counter_merge<F, 1, 2>(k + t, gv, s0, s1, s2, ne);
      }
    }
    if (kStream && xs_merge) {
      __syncwarp();
      F v = F(0);
      if (lane < G) ld_shared(sl.my_s + WS::kXs + lane * (uint32_t)sizeof(F), v);
      __syncwarp();
      for (int off = 1; off < G; off <<= 1) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, off), job.top_cr);
      gv[0] = v;
    }
    NRMF_TRACE(1, 0, 0);
    if (!job.combine) continue;
#ifdef NRMF_PROBE_NO_ANNOUNCE  // dev-only timing probe: no announce/climb (wrong results)
    if (lane == 0 && gv[0] == F(-1)) *job.out = gv[0];
    continue;
#endif
    if (job.nsteps == 0) {  // the warp group is the whole tree
      write_root(job, gv[0]);
      continue;
    }
    if (kStream && job.cta_step0) {
      cta_arrive<F>(job, cta_s, grp, rnd, W, gv[0], n_groups);
      continue;
    }
    // announce this warp group; the last arriver of its 2^lg_fan group climbs.
    unsigned old = 0;
    NRMF_JITTER(10);
    if (lane == 0) {
      job.vals[job.val_off[0] + grp] = gv[0];
      old = atom_add_release(job.cnt + job.cnt_off[0] + (grp >> job.lg_fan[0]), 1u);
    }
    climb(job, 0, grp, old);
  }
  NRMF_TRACE(4, 0, 0);
}

// Small calls (few tiles): one CTA per warp group of G tiles, and the NIT
// batches of each tile (8 rows = depth-3 subtrees of every lane) on NIT
// different warps, so a tile costs the latency of one batch plus the levels
// above it instead of NIT sequential batches on one warp.  The batch values
// meet in a shared-memory stash; warp 0 evaluates the levels above the
// batches (lanes_from_batches), the cross-thread and group levels
// (group_cross), announces the group and climbs -- the same tree as the
// persistent kernel.  A flagged leaf, a NaN or a partial tile: warp 0
// recomputes the group with the exact path.
constexpr int kSplitWarps = 8;
template <typename F, int MODE>
__global__ void __launch_bounds__(kSplitWarps * 32, 2) nrmf_split_kernel(const TreeJob<F> job) {
  constexpr int V = Cfg<F>::V, NIT = Cfg<F>::J / kBatch;
  static_assert(kSplitWarps % NIT == 0, "whole tiles per CTA");
  __shared__ __align__(16) unsigned char stash[kSplitWarps * 32 * 16];  // [tile k][batch it][thread]
  __shared__ __align__(16) F xs[kSplitWarps / NIT * 32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = 1 << job.g0;
  const int64_t grp = blockIdx.x;
  const int k = w / NIT, it = w % NIT;
  NRMF_TRACE(0, 0, 0);
  const bool ll_comb = job.ll != nullptr && blockIdx.x == 0 && w == 1;
  // fan-in 256: warp 2 polls the upper half of the slots (ll_gather_half)
  const bool ll_two = NRMF_LL_TWO && job.ll != nullptr && blockIdx.x == 0 && job.nsteps >= 1 &&
                      job.lg_fan[job.nsteps - 1] == 8;
  __shared__ F ll_xch[130];
  // this call's number (the combiner; the producers' slot tag is hashed from
  // it after the batch phase): the header load -- a DRAM round trip with a
  // cold L2 -- is issued behind the batch loads, not ahead of them
  const bool need_hdr = job.ll != nullptr && (w == 0 || ll_comb || (ll_two && w == 2));
  uint64_t ll_c = 0;
  // are all G tiles of the group full tiles with data?
  bool full = (grp + 1) * G <= job.n_items;
  for (int t = 0; t < G && full; ++t) {
    const F* tb;
    int64_t remv;
    full = tile_at(job, grp * G + t, tb, remv);
  }
  bool flagged = false;
  if (full && k < G) {
    NodeFast node;
    GlobalLoader<F, MODE> ld;
    int64_t remv;
    const F* tb;
    tile_at(job, grp * G + k, tb, remv);
    ld.tb = tb;
    ld.valid = kTile;
    ld.begin(it);
    if (need_hdr) ll_c = ll_call(job);
#ifdef NRMF_PROBE_TRACE2  // the batch's loads have landed (the compare waits on them)
    if (ld.u[kBatch - 1][V - 1] == F(-1234.5)) flagged = true;
    NRMF_TRACE(14, 0, 0);
#endif
    F r[V];
    batch_lanes<F>(ld, node, r);
    st_stash(smem_u32(stash) + ((k * NIT + it) * 32 + lane) * 16, r);
    flagged |= node.bad;
    NRMF_TRACE(5, 0, 0);
  } else if (need_hdr) {
    ll_c = ll_call(job);
  }
  // one barrier (no flag to clear before the loads): the stash is complete
  // and every warp knows whether any batch of the CTA flagged a leaf
  const bool any_bad = __syncthreads_or(flagged) != 0;
  NRMF_TRACE(15, 0, 0);
  if (ll_comb) {
    if (job.peers != nullptr) prefetch_exchange(job.peers, job.p_rank);  // it polls long before the root
    ll_combine(job, ll_c, ll_two ? ll_xch : (F*)nullptr);
    return;
  }
  if (ll_two && w == 2) {
    ll_combine(job, ll_c, ll_xch);
    return;
  }
  if (w != 0) return;
  F gv = F(0);
  bool done = false;
  if (full && !any_bad) {
    NodeFast node;
    for (int t = 0; t < G; ++t) {
      F u[NIT][V];
#pragma unroll
      for (int i = 0; i < NIT; ++i) ld_stash(smem_u32(stash) + ((t * NIT + i) * 32 + lane) * 16, u[i]);
      st_shared(smem_u32(xs) + (t * 32 + lane) * (uint32_t)sizeof(F), lanes_from_batches<F>(u, node));
    }
    __syncwarp();
    done = group_cross<F>(node, smem_u32(xs), G, job.top_cr, gv,
                          job.tile_out != nullptr ? job.tile_out + grp * G : nullptr);
  }
  if (!done) {
    F s0[1], s1[1], s2[1], g[1];
    NodeTop ne{job.top_cr};
    for (int t = 0; t < G; ++t) {
      const int64_t tau = grp * G + t;
      g[0] = single_tile<F, MODE == kVec>(job, tau);
      if (job.tile_out != nullptr && lane == 0 && tau < job.n_items) job.tile_out[tau] = g[0];
      if (G == 8) counter_merge<F, 1, 8>(t, g, s0, s1, s2, ne);
      else if (G == 4) counter_merge<F, 1, 4>(t, g, s0, s1, s2, ne);
      else if (G == 2) counter_merge<F, 1, 2>(t, g, s0, s1, s2, ne);
    }
    gv = g[0];
  }
  NRMF_TRACE(1, 0, 0);
  if (!job.combine) return;
  if (job.nsteps == 0) {
    write_root(job, gv);
    return;
  }
  NRMF_JITTER(11);
  const uint64_t ll_t = job.ll != nullptr ? ll_tag(job.ll, ll_c) : 0ull;
  if (job.ll != nullptr && job.nsteps == 1) {  // the group is an input of the last step
    ll_store(job, grp, gv, ll_t);
    return;
  }
  unsigned old = 0;
  if (lane == 0) {
    job.vals[job.val_off[0] + grp] = gv;
    old = atom_add_release(job.cnt + job.cnt_off[0] + (grp >> job.lg_fan[0]), 1u);
  }
  climb<F, true>(job, 0, grp, old, ll_t);
  NRMF_TRACE(4, 0, 0);
}

// Balanced tree over vals[0..P) (entries >= nvals are +0) -> *out.  One CTA.
template <typename F>
__global__ void __launch_bounds__(kAuxThreads) bal_kernel(const F* vals, int64_t nvals, int64_t P,
                                                       F* out, int cr) {
  const F v = block_bal(vals, nvals, P, cr);
  if (threadIdx.x == 0) *out = v;
}

// Per-column combine for columns longer than one tile: column j has tpc tile
// values vals[j*tpc ..] padded to p2c; then the frob tree over columns
// (p2cols = pow2 >= cols) with group partials per CTA and a last-CTA top.
template <typename F>
__global__ void __launch_bounds__(kAuxThreads) cols_combine_kernel(
    const F* vals, int64_t cols, int64_t tpc, int64_t p2c, F* col_norms, int64_t p2cols,
    F* partials, unsigned* ticket, F* frob, int cr) {
  __shared__ int s_last;
  const int64_t j = (int64_t)blockIdx.x * kAuxThreads + threadIdx.x;
  F v = F(0);
  if (j < cols) {
    v = seq_bal(vals + j * tpc, tpc, 0, p2c, cr);
    col_norms[j] = v;
  }
  if (frob == nullptr) return;
  // block level: first min(8, lg p2cols) levels of the frob tree
  const int lg = ilog2_64(p2cols);
  const int bl = lg < 8 ? lg : 8;
  __shared__ F sh[kAuxWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wl = bl < 5 ? bl : 5;
  for (int l = 0; l < wl; ++l) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, 1 << l), cr);
  if (bl > 5) {
    if (lane == 0) sh[w] = v;
    __syncthreads();
    v = lane < kAuxWarps ? sh[lane] : F(0);
    for (int l = 0; l < bl - 5; ++l) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, 1 << l), cr);
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
  const F r = block_bal(partials, (int64_t)gridDim.x, pb, cr);
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


static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
constexpr uintptr_t kWsAlign = 16;  // nrmf.h: workspaces are 16-byte aligned

// Plan of the combine over p2 tiles of which n_items are real: g0 levels
// inside each warp group, then steps of 6 levels (fan-in 64); first_fan = 4:
// the first step is the stream kernel's CTA step; last_fan = 8: the last step
// may take up to 8 levels (split kernel).
struct Plan {
  int g0 = 0;
  int nsteps = 0;
  int lg_fan[kMaxSteps] = {};
  int64_t nin[kMaxSteps] = {};
  int64_t val_off[kMaxSteps] = {};
  int64_t cnt_off[kMaxSteps] = {};
  int64_t n_vals = 0;
  int64_t n_cnt = 0;
};

static Plan make_plan(int64_t n_items, int64_t p2, int g0_max, int first_fan = 6, int last_fan = 6) {
  Plan pl;
  int L = 0;
  while ((int64_t(1) << L) < p2) ++L;
  pl.g0 = L < g0_max ? L : g0_max;
  L -= pl.g0;
  int64_t nin = (n_items + (int64_t(1) << pl.g0) - 1) >> pl.g0;
  int64_t voff = 0, coff = 0;
  while (L > 0) {
    // steps of 6 levels (fan-in 64); with last_fan = 8 (the split kernel)
    // the last step may take up to 8: one climb of 8 levels instead of two
    // climbs and an atomic round trip in between (C1, 2^20 fp64: 13.3 ->
    // 12.4 us).  In the persistent kernel the wider climb code cost 0.3-0.8 %
    // at 2^24..2^30 (tools/size_sweep.py A/B), so it stays at 6 there.
    const int fmax = pl.nsteps == 0 && first_fan < 6 ? first_fan : (L <= last_fan ? L : 6);
    const int f = L < fmax ? L : fmax;
    const int k = pl.nsteps++;
    pl.lg_fan[k] = f;
    pl.nin[k] = nin;
    pl.cnt_off[k] = coff;
    pl.val_off[k] = voff;
    const int64_t groups = (nin + (int64_t(1) << f) - 1) >> f;
    coff += groups;
    voff += nin;
    nin = groups;
    L -= f;
  }
  pl.n_vals = voff;
  pl.n_cnt = coff;
  return pl;
}

// Workspace of one tree evaluation: [counters][values] (worst case g0 = 0)
static size_t tree_ws_bytes(int64_t n_items, int64_t p2, size_t esz) {
  size_t b = 0;
  for (int ff : {6, 4, 8}) {  // fan-in 64 steps, a first CTA step of 16, or a last step up to 256
    for (int g0 = 0; g0 <= (ff == 8 ? 4 : 0); ++g0) {
      const Plan pl = ff == 8 ? make_plan(n_items, p2, g0, 6, 8) : make_plan(n_items, p2, 0, ff);
      // the split kernel's last-step slots (ll_*): an epoch word and 16 B per input
      const size_t ll = ff == 8 && pl.nsteps >= 1 ? align_up(16 * (size_t)(1 + pl.nin[pl.nsteps - 1]), 256) : 0;
      b = std::max(b, align_up((size_t)pl.n_cnt * 4, 256) + align_up((size_t)pl.n_vals * esz, 256) + ll + 256);
    }
  }
  return b;
}

template <typename F>
static TreeJob<F> make_job(const F* x, int64_t n_items, int64_t tpc, int64_t ld, int64_t len, F* tile_out,
                           F* out, int combine, int top_cr, void* ws, size_t cnt_bytes, const Plan& pl) {
  TreeJob<F> job;
  job.x = x;
  job.n_items = n_items;
  job.tpc = tpc;
  job.ld = ld;
  job.len = len;
  job.tile_out = tile_out;
  job.cnt = reinterpret_cast<unsigned*>(ws);
  job.vals = reinterpret_cast<F*>(static_cast<char*>(ws) + cnt_bytes);
  job.out = out;
  job.combine = combine;
  job.top_cr = top_cr;
  job.g0 = pl.g0;
  job.cta_minor = 0;
  job.cta_step0 = 0;
  job.peers = nullptr;
  job.p_err = nullptr;
  job.p_world = job.p_rank = job.p_nr = 0;
  job.ll = nullptr;
  job.nsteps = pl.nsteps;
  for (int k = 0; k < kMaxSteps; ++k) {
    job.lg_fan[k] = pl.lg_fan[k];
    job.nin[k] = pl.nin[k];
    job.val_off[k] = pl.val_off[k];
    job.cnt_off[k] = pl.cnt_off[k];
  }
  return job;
}

template <typename F>
static void set_exchange(TreeJob<F>& job, const RankExchange* rx) {
  if (rx == nullptr) return;
  job.peers = rx->peers;
  job.p_err = rx->err;
  job.p_world = rx->world;
  job.p_rank = rx->rank;
  job.p_nr = rx->nr;
}

#ifndef NRMF_NT
#define NRMF_NT 1             // tiles reduced in lockstep per warp when warp groups allow it
#endif

// Dynamic shared memory: stream kernel kWarps x WarpSmem; column (PipeLoader)
// kernel [ring: kWarps x kStages x 4 KiB][barriers].
template <typename F, bool TMA, bool STREAM = false, bool UNAL = false>
static size_t kernel_smem() {
  if (!(TMA && NRMF_USE_TMA)) return 0;
  if (STREAM) return (size_t)kWarps * WarpSmem<F, UNAL>::kBytes + CtaSmem<F>::kBytes;
  return (size_t)kWarps * kStages * kBatchBytes + (size_t)kWarps * kStages * 8;
}

// Function attributes (the dynamic shared memory opt-in) belong to a device's
// context: they are set, and the occupancy cached, once per device.
constexpr int kMaxDevices = 64;
template <typename F, bool TMA, int NT, bool STREAM, bool GAP = false, bool UNAL = false, bool SHORT = false>
static int blocks_per_sm() {
  static std::atomic<int> cached[kMaxDevices];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return 1;
  int b = cached[dev].load(std::memory_order_acquire);
  if (b != 0) return b;
  std::lock_guard<std::mutex> lock(mu);
  b = cached[dev].load(std::memory_order_relaxed);
  if (b != 0) return b;
  const size_t sm = kernel_smem<F, TMA, STREAM, UNAL>();
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(nrmf_tree_kernel<F, TMA, NT, STREAM, GAP, UNAL, SHORT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, nrmf_tree_kernel<F, TMA, NT, STREAM, GAP, UNAL, SHORT>, kThreads,
                                                    sm) !=
          cudaSuccess ||
      b < 1)
    b = 1;
  cached[dev].store(b, std::memory_order_release);
  return b;
}

static int g_grid_override = 0;  // test hook: force a grid size (0 = automatic)
static int g_g0_override = -1;   // dev hook: force the warp-group level count g0 (-1 = automatic)
static int g_cta_step0 = NRMF_CTA_STEP;  // dev hook: first combine step in shared memory (stream kernel)
static int g_gap_stream = 1;     // test hook: gapped column blocks on the stream kernel (0: general kernel)
static int g_split_ll = 1;       // test hook: the split kernel's last step by slots (0: by a counter)
static int g_unal_stream = 1;    // test hook: unaligned vectors on the stream kernel (0: element-load kernel)

// Launch the tree kernel over items (tiles) with mapping (tpc, ld, len).
template <typename F>
static int launch_tree(const F* x, int64_t n_items, int64_t tpc, int64_t ld, int64_t len, int64_t p2,
                       F* tile_out, F* out, int combine, void* ws, size_t ws_bytes, bool vec,
                       cudaStream_t s, int flags, const RankExchange* rx = nullptr) {
  const int top_cr = flags & NRMF_TOP_CR;
  // NRMF_WS_CLEAN: the caller guarantees the arrival counters are zero (nrmf.h)
  const bool clean = (flags & NRMF_WS_CLEAN) != 0;
  if (n_items == 0) return NRMF_OK;
  if (n_items >= (int64_t(1) << 31) - 64) return NRMF_EINVAL;  // kernels index tiles/groups in 32 bits (n < 2^43)
  // contiguous tiles (a vector, or whole columns of T-multiple length stored
  // back to back): warp groups are contiguous, the pointer-walk producer applies
  const bool stream = vec && (ld == 0 || (ld == len && len % kTile == 0));
  // column blocks with gaps (ld > rows, rows a multiple of T; vec implies
  // 16-byte aligned columns): the stream kernel with the gap-skipping walk
  const bool gap = vec && g_gap_stream && ld > len && len % kTile == 0;
  // a vector whose base is element- but not 16-byte aligned (the paper's
  // unaligned case): the stream kernel with shifted spans (StreamLoader UNAL)
  const bool ustream = !vec && ld == 0 && g_unal_stream;
  // short column blocks that are not 16-byte aligned: the element-load
  // kernel's SHORT instance (paired columns)
  const bool eshort = !vec && !ustream && ld != 0 && tpc == 1 && len <= 2 * kBatch * Cfg<F>::LANES;
  int64_t grid = (int64_t)device_sms() * (gap       ? blocks_per_sm<F, true, 1, true, true>()
                                          : stream  ? blocks_per_sm<F, true, 1, true>()
                                          : ustream ? blocks_per_sm<F, true, 1, true, false, true>()
                                          : vec     ? blocks_per_sm<F, true, NRMF_NT, false>()
                                          : eshort  ? blocks_per_sm<F, false, 1, false, false, false, true>()
                                                    : blocks_per_sm<F, false, 1, false>());
  if (g_grid_override > 0) grid = g_grid_override;
  // warp groups of up to 8 tiles while there is enough work for every warp
  // Small calls: the split kernel (one CTA per group of G tiles, one warp per
  // batch) while it needs at most two waves of CTAs.
  {
    constexpr int NIT = Cfg<F>::J / kBatch;
    int g0s = 0;
    while ((int64_t(1) << (g0s + 1)) * NIT <= kSplitWarps && (int64_t(1) << (g0s + 1)) <= p2 && combine) ++g0s;
    if (!combine) g0s = 0;
    const int64_t n_groups = (n_items + (int64_t(1) << g0s) - 1) >> g0s;
    if (g_grid_override == 0 && n_groups <= 4 * (int64_t)device_sms()) {
      const Plan pl = combine ? make_plan(n_items, p2, g0s, 6, kMaxFanLg)
                              : make_plan(n_items, int64_t(1) << g0s, g0s);
      const size_t cnt_bytes = align_up((size_t)pl.n_cnt * 4, 256);
      const size_t vals_bytes = align_up((size_t)pl.n_vals * sizeof(F), 256);
      // the last step by flag-in-data slots (ll_*): no counter, never cleared
      const bool ll = combine && pl.nsteps >= 1 && g_split_ll;
      const size_t ll_bytes = ll ? align_up(16 * (size_t)(1 + pl.nin[pl.nsteps - 1]), 256) : 0;
      const size_t need = cnt_bytes + vals_bytes + ll_bytes + 256;
      if (combine && ws_bytes < need) return NRMF_EWORKSPACE;
      // counters of the steps below the last (none for a one-step plan)
      const int64_t n_cnt = ll ? pl.cnt_off[pl.nsteps - 1] : pl.n_cnt;
      if (combine && !clean && n_cnt > 0 && cudaMemsetAsync(ws, 0, (size_t)n_cnt * 4, s) != cudaSuccess)
        return NRMF_ECUDA;
      TreeJob<F> job = make_job(x, n_items, tpc, ld, len, tile_out, out, combine, top_cr, ws, cnt_bytes, pl);
      set_exchange(job, rx);
      if (ll) job.ll = static_cast<char*>(ws) + cnt_bytes + vals_bytes;
      if (vec) nrmf_split_kernel<F, kVec><<<(unsigned)n_groups, kSplitWarps * 32, 0, s>>>(job);
      else nrmf_split_kernel<F, kScalar><<<(unsigned)n_groups, kSplitWarps * 32, 0, s>>>(job);
      return cudaGetLastError() == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
    }
  }
  // Warp-group size G = 2^g0 (<= 8 tiles; 16 for fp32 on the stream kernel).
  // The persistent warps take groups round-robin, so the makespan is
  // ceil(groups / W) groups of G tiles, and a group costs about G + c tiles
  // (its cross-thread tail and announce).  c = 1/12 tile, fitted to forced-g0
  // timings at n = 2^22..2^30 (tools/g0_sweep.py --both --lg=...): it was 1/3
  // (4/3 for fp32) before the CTA combine step made the announce cheap; with
  // 1/12 fp64 2^26 runs G = 1 (132 -> 123 us) and fp32 2^27 G = 2 (100 ->
  // 94 us), the other sizes keep their G.  Take the G minimising
  // ceil(groups / W) * (G + c), the larger on ties.  The tree does not depend
  // on g0.
  constexpr double kGroupCost = 1.0 / 12.0;
  int g0_max = 0;
  // groups of up to kMaxGroup tiles on the stream kernel, 8 elsewhere
  // (the column kernel's counter merge has three levels)
  const int gmax = (stream || gap || ustream) ? (sizeof(F) == 4 ? 4 : 3) : 3;
  {
    const int64_t W = grid * kWarps;
    double best = 0.0;
    for (int g = gmax; g >= 0; --g) {
      const int64_t groups = (n_items + (int64_t(1) << g) - 1) >> g;
      const double cost = (double)((groups + W - 1) / W) * ((double)(1 << g) + kGroupCost);
      if (g == gmax || cost < best - 1e-9) {
        best = cost;
        g0_max = g;
      }
    }
  }
  // without a combine (tile values only) the warp groups still batch the
  // cross-thread levels of their tiles; their group value is not used
  if (g_g0_override >= 0) g0_max = std::min(g_g0_override, gmax);
  // stream kernel with every warp busy (CTA-major warps): the first combine
  // step is the CTA's 16 warp groups of a round, in shared memory
  Plan pl = combine ? make_plan(n_items, p2, g0_max)
                    : make_plan(n_items, int64_t(1) << g0_max, g0_max);
  bool cta_step0 = false;
  if ((stream || gap || ustream) && combine && kWarps == 16 && g_cta_step0 &&
      ((n_items + (int64_t(1) << pl.g0) - 1) >> pl.g0) >= grid * kWarps) {
    const Plan p4 = make_plan(n_items, p2, g0_max, 4);
    if (p4.nsteps >= 1 && p4.lg_fan[0] == 4 && p4.g0 == pl.g0) {
      pl = p4;
      cta_step0 = true;
    }
  }
  const size_t cnt_bytes = align_up((size_t)pl.n_cnt * 4, 256);
  const size_t need = cnt_bytes + align_up((size_t)pl.n_vals * sizeof(F), 256) + 256;
  if (combine && ws_bytes < need) return NRMF_EWORKSPACE;
  // counters start at zero on every call, whatever the workspace last held
  // (the last arrivers also leave them zero; this makes reuse of one
  // workspace across calls of different shapes or functions safe) -- unless
  // the caller vouches for them (NRMF_WS_CLEAN: a workspace dedicated to one
  // call shape, e.g. a captured graph's; the call is then one kernel)
  if (combine && !clean && pl.n_cnt > 0 && cudaMemsetAsync(ws, 0, (size_t)pl.n_cnt * 4, s) != cudaSuccess)
    return NRMF_ECUDA;
  TreeJob<F> job = make_job(x, n_items, tpc, ld, len, tile_out, out, combine, top_cr, ws, cnt_bytes, pl);
  set_exchange(job, rx);
  const int64_t n_groups = (n_items + (int64_t(1) << pl.g0) - 1) >> pl.g0;
  job.cta_minor = n_groups < grid * kWarps;
  job.cta_step0 = cta_step0 ? 1 : 0;
  grid = std::min<int64_t>(grid, n_groups);
  if (gap) {
    nrmf_tree_kernel<F, true, 1, true, true><<<(unsigned)grid, kThreads, kernel_smem<F, true, true>(), s>>>(job);
  } else if (stream) {
    nrmf_tree_kernel<F, true, 1, true><<<(unsigned)grid, kThreads, kernel_smem<F, true, true>(), s>>>(job);
  } else if (ustream) {
    nrmf_tree_kernel<F, true, 1, true, false, true>
        <<<(unsigned)grid, kThreads, kernel_smem<F, true, true, true>(), s>>>(job);
  } else if (vec && pl.g0 >= 1 && NRMF_NT == 2) {
    blocks_per_sm<F, true, NRMF_NT, false>();
    nrmf_tree_kernel<F, true, NRMF_NT, false><<<(unsigned)grid, kThreads, kernel_smem<F, true>(), s>>>(job);
  } else if (vec) {
    blocks_per_sm<F, true, 1, false>();
    nrmf_tree_kernel<F, true, 1, false><<<(unsigned)grid, kThreads, kernel_smem<F, true>(), s>>>(job);
  } else if (eshort) {
    nrmf_tree_kernel<F, false, 1, false, false, false, true>
        <<<(unsigned)grid, kThreads, kernel_smem<F, false>(), s>>>(job);
  } else {
    nrmf_tree_kernel<F, false, 1, false><<<(unsigned)grid, kThreads, kernel_smem<F, false>(), s>>>(job);
  }
  return cudaGetLastError() == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
}

template <typename F>
int tree_eval(int64_t n, const F* x, int64_t p2, F* out, void* ws, size_t ws_bytes, cudaStream_t s,
              int flags, const RankExchange* rx) {
  // Evaluate the balanced tree over p2 tiles (p2 >= ceil(n/T), power of two)
  // of x[0..n) padded with +0; *out = root.  Caller validated arguments.
  const int64_t nt = (n + kTile - 1) / kTile;
  if (nt == 0) {
    if (cudaMemsetAsync(out, 0, sizeof(F), s) != cudaSuccess) return NRMF_ECUDA;
    return NRMF_OK;
  }
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
  return launch_tree<F>(x, nt, nt, 0, n, p2, nullptr, out, 1, ws, ws_bytes, vec, s, flags, rx);
}

template int tree_eval<double>(int64_t, const double*, int64_t, double*, void*, size_t, cudaStream_t, int,
                               const RankExchange*);
template int tree_eval<float>(int64_t, const float*, int64_t, float*, void*, size_t, cudaStream_t, int,
                              const RankExchange*);

template <typename F>
int bal_eval(const F* vals, int64_t nvals, int64_t P, F* out, cudaStream_t s, int top_cr) {
  bal_kernel<F><<<1, kAuxThreads, 0, s>>>(vals, nvals, P, out, top_cr);
  return cudaGetLastError() == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
}
template int bal_eval<double>(const double*, int64_t, int64_t, double*, cudaStream_t, int);
template int bal_eval<float>(const float*, int64_t, int64_t, float*, cudaStream_t, int);

size_t tree_workspace(int64_t p2, size_t esz) { return tree_ws_bytes(p2, p2, esz); }

// ---------------------------------------------------------------- vector
template <typename F>
static int nrmf_vec(int64_t n, const F* x, F* out, int flags, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || out == nullptr || (n > 0 && (x == nullptr || ws == nullptr))) return NRMF_EINVAL;
  if ((reinterpret_cast<uintptr_t>(x) % sizeof(F)) != 0 ||
      (reinterpret_cast<uintptr_t>(out) % sizeof(F)) != 0 || (reinterpret_cast<uintptr_t>(ws) % kWsAlign) != 0)
    return NRMF_EALIGN;
  const int64_t nt = (n + kTile - 1) / kTile;
  return tree_eval<F>(n, x, pow2_ceil(std::max<int64_t>(nt, 1)), out, ws, ws_bytes,
                      static_cast<cudaStream_t>(stream), flags);
}

// ---------------------------------------------------------------- columns
// rows <= T: one tile per column, the tree kernel writes col_norms (its tile
// values) and combines them into frob.  rows > T: tile values into the
// workspace, then per-column trees and the frob tree (cols_combine_kernel).
// Workspace (rows > T): [ticket 256][tile values cols*tpc][block partials]
// p2cols: size of the Frobenius tree over the columns (0: pow2 >= cols; a
// larger power of two when the columns are one rank's aligned subtree of a
// sharded matrix, nrmf_cols_dist_[ds]).
static size_t cols_ws_bytes(int64_t rows, int64_t cols, size_t esz, int64_t p2cols = 0) {
  const int64_t tpc = std::max<int64_t>((rows + kTile - 1) / kTile, 1);
  if (p2cols == 0) p2cols = pow2_ceil(std::max<int64_t>(cols, 1));
  if (tpc == 1) return tree_ws_bytes(std::max<int64_t>(cols, 1), p2cols, esz);
  const int64_t nblk = (cols + kAuxThreads - 1) / kAuxThreads;
  return 256 + align_up((size_t)(cols * tpc) * esz, 256) + align_up((size_t)std::max<int64_t>(nblk, 1) * esz, 256);
}

template <typename F>
static int nrmf_cols_impl(int64_t rows, int64_t cols, int64_t ld, const F* A, F* col_norms,
                          F* frob, int flags, void* ws, size_t ws_bytes, void* stream, int64_t p2_override = 0) {
  const int cr = flags & NRMF_TOP_CR;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rows < 0 || cols < 0 || ld < rows || ld < 0) return NRMF_EINVAL;
  if (cols > 0 && col_norms == nullptr) return NRMF_EINVAL;
  if (rows > 0 && cols > 0 && (A == nullptr || ws == nullptr)) return NRMF_EINVAL;
  if (reinterpret_cast<uintptr_t>(A) % sizeof(F) || reinterpret_cast<uintptr_t>(col_norms) % sizeof(F) ||
      reinterpret_cast<uintptr_t>(frob) % sizeof(F) || reinterpret_cast<uintptr_t>(ws) % kWsAlign)
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
  if (ws_bytes < cols_ws_bytes(rows, cols, sizeof(F), p2_override)) return NRMF_EWORKSPACE;
  const int64_t tpc = (rows + kTile - 1) / kTile;
  const int64_t p2cols = p2_override > 0 ? p2_override : pow2_ceil(cols);
  const bool vec = (reinterpret_cast<uintptr_t>(A) & 15u) == 0 && ((ld * (int64_t)sizeof(F)) & 15) == 0;
  if (tpc == 1)
    return launch_tree<F>(A, cols, 1, ld, rows, p2cols, col_norms, frob, frob != nullptr ? 1 : 0, ws, ws_bytes,
                          vec, s, flags);
  unsigned* ticket = reinterpret_cast<unsigned*>(ws);
  char* base = static_cast<char*>(ws) + 256;
  F* vals = reinterpret_cast<F*>(base);
  F* partials = reinterpret_cast<F*>(base + align_up((size_t)(cols * tpc) * sizeof(F), 256));
  int st = launch_tree<F>(A, cols * tpc, tpc, ld, rows, 1, vals, nullptr, 0, ws, ws_bytes, vec, s, cr);
  if (st != NRMF_OK) return st;
  if (frob != nullptr && !(flags & NRMF_WS_CLEAN) && cudaMemsetAsync(ticket, 0, sizeof(unsigned), s) != cudaSuccess)
    return NRMF_ECUDA;
  const int64_t nblk = (cols + kAuxThreads - 1) / kAuxThreads;
  cols_combine_kernel<F><<<(unsigned)nblk, kAuxThreads, 0, s>>>(vals, cols, tpc, pow2_ceil(tpc), col_norms,
                                                            p2cols, partials, ticket, frob, cr);
  return cudaGetLastError() == cudaSuccess ? NRMF_OK : NRMF_ECUDA;
}

template <typename F>
int cols_eval(int64_t rows, int64_t cols, int64_t ld, const F* A, F* col_norms, F* frob, int64_t p2cols,
              int flags, void* ws, size_t ws_bytes, cudaStream_t s) {
  return nrmf_cols_impl<F>(rows, cols, ld, A, col_norms, frob, flags, ws, ws_bytes, s, p2cols);
}
template int cols_eval<double>(int64_t, int64_t, int64_t, const double*, double*, double*, int64_t, int, void*,
                               size_t, cudaStream_t);
template int cols_eval<float>(int64_t, int64_t, int64_t, const float*, float*, float*, int64_t, int, void*,
                              size_t, cudaStream_t);
size_t cols_workspace(int64_t rows, int64_t cols, int64_t p2cols, size_t esz) {
  return cols_ws_bytes(rows, cols, esz, p2cols);
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
  return tree_ws_bytes(c, c, esz) + align_up((size_t)nchunks * esz, 256) + 256 +
         (size_t)kRing * (size_t)(c * kTile) * esz;
}

template <typename F>
static int nrmf_host_impl(int64_t n, const F* host_x, F* host_out, int flags, void* ws, size_t ws_bytes,
                          void* stream) {
  const int cr = flags & NRMF_TOP_CR;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 0 || host_out == nullptr || ws == nullptr || (n > 0 && host_x == nullptr)) return NRMF_EINVAL;
  if (reinterpret_cast<uintptr_t>(host_x) % sizeof(F) || reinterpret_cast<uintptr_t>(ws) % kWsAlign)
    return NRMF_EALIGN;
  if (ws_bytes < host_ws_bytes(n, sizeof(F))) return NRMF_EWORKSPACE;
  const int64_t nt = std::max<int64_t>((n + kTile - 1) / kTile, 1);
  const int64_t p2 = pow2_ceil(nt);
  const int64_t c = std::min<int64_t>(p2, kChunkTiles);
  const int64_t nchunks = (nt + c - 1) / c;
  char* p = static_cast<char*>(ws);
  void* tree_ws = p;
  const size_t tws = tree_ws_bytes(c, c, sizeof(F));
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
      int st = tree_eval<F>(cnt, buf, c, nchunks == 1 ? dev_out : chunk_vals + k, tree_ws, tws, s, cr);
      if (st != NRMF_OK) return st;
      if (cudaEventRecord(h->consumed[slot], s) != cudaSuccess) return NRMF_ECUDA;
    }
    if (nchunks > 1) {
      int st = bal_eval<F>(chunk_vals, nchunks, p2 / c, dev_out, s, cr);
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
  return tree_ws_bytes(nt, pow2_ceil(nt), (size_t)elem_bytes);
}

static bool flags_ok(int flags) { return (flags & ~(NRMF_TOP_CR | NRMF_WS_CLEAN)) == 0; }

int nrmf_d(int64_t n, const double* x, double* out, void* ws, size_t ws_bytes, void* stream) {
  return nrmf_vec<double>(n, x, out, 0, ws, ws_bytes, stream);
}
int nrmf_s(int64_t n, const float* x, float* out, void* ws, size_t ws_bytes, void* stream) {
  return nrmf_vec<float>(n, x, out, 0, ws, ws_bytes, stream);
}
int nrmf_ex_d(int64_t n, const double* x, double* out, int flags, void* ws, size_t ws_bytes, void* stream) {
  if (!flags_ok(flags)) return NRMF_EINVAL;
  return nrmf_vec<double>(n, x, out, flags, ws, ws_bytes, stream);
}
int nrmf_ex_s(int64_t n, const float* x, float* out, int flags, void* ws, size_t ws_bytes, void* stream) {
  if (!flags_ok(flags)) return NRMF_EINVAL;
  return nrmf_vec<float>(n, x, out, flags, ws, ws_bytes, stream);
}
int nrmf_z_d(int64_t count, const double* z, double* out, void* ws, size_t ws_bytes, void* stream) {
  if (count < 0 || count > INT64_MAX / 2) return NRMF_EINVAL;
  return nrmf_vec<double>(2 * count, z, out, 0, ws, ws_bytes, stream);
}
int nrmf_z_s(int64_t count, const float* z, float* out, void* ws, size_t ws_bytes, void* stream) {
  if (count < 0 || count > INT64_MAX / 2) return NRMF_EINVAL;
  return nrmf_vec<float>(2 * count, z, out, 0, ws, ws_bytes, stream);
}

size_t nrmf_cols_workspace_bytes(int64_t rows, int64_t cols, int elem_bytes) {
  if (rows < 0 || cols < 0 || (elem_bytes != 4 && elem_bytes != 8)) return 0;
  return cols_ws_bytes(rows, cols, (size_t)elem_bytes);
}
int nrmf_cols_d(int64_t rows, int64_t cols, int64_t ld, const double* A, double* col_norms,
                double* frob, void* ws, size_t ws_bytes, void* stream) {
  return nrmf_cols_impl<double>(rows, cols, ld, A, col_norms, frob, 0, ws, ws_bytes, stream);
}
int nrmf_cols_s(int64_t rows, int64_t cols, int64_t ld, const float* A, float* col_norms,
                float* frob, void* ws, size_t ws_bytes, void* stream) {
  return nrmf_cols_impl<float>(rows, cols, ld, A, col_norms, frob, 0, ws, ws_bytes, stream);
}
int nrmf_cols_ex_d(int64_t rows, int64_t cols, int64_t ld, const double* A, double* col_norms,
                   double* frob, int flags, void* ws, size_t ws_bytes, void* stream) {
  if (!flags_ok(flags)) return NRMF_EINVAL;
  return nrmf_cols_impl<double>(rows, cols, ld, A, col_norms, frob, flags, ws, ws_bytes, stream);
}
int nrmf_cols_ex_s(int64_t rows, int64_t cols, int64_t ld, const float* A, float* col_norms,
                   float* frob, int flags, void* ws, size_t ws_bytes, void* stream) {
  if (!flags_ok(flags)) return NRMF_EINVAL;
  return nrmf_cols_impl<float>(rows, cols, ld, A, col_norms, frob, flags, ws, ws_bytes, stream);
}

size_t nrmf_host_workspace_bytes(int64_t n, int elem_bytes) {
  if (n < 0 || (elem_bytes != 4 && elem_bytes != 8)) return 0;
  return host_ws_bytes(n, (size_t)elem_bytes);
}
int nrmf_host_d(int64_t n, const double* host_x, double* host_out, void* ws, size_t ws_bytes,
                void* stream) {
  return nrmf_host_impl<double>(n, host_x, host_out, 0, ws, ws_bytes, stream);
}
int nrmf_host_s(int64_t n, const float* host_x, float* host_out, void* ws, size_t ws_bytes,
                void* stream) {
  return nrmf_host_impl<float>(n, host_x, host_out, 0, ws, ws_bytes, stream);
}
int nrmf_host_ex_d(int64_t n, const double* host_x, double* host_out, int flags, void* ws, size_t ws_bytes,
                   void* stream) {
  if (!flags_ok(flags)) return NRMF_EINVAL;
  return nrmf_host_impl<double>(n, host_x, host_out, flags, ws, ws_bytes, stream);
}
int nrmf_host_ex_s(int64_t n, const float* host_x, float* host_out, int flags, void* ws, size_t ws_bytes,
                   void* stream) {
  if (!flags_ok(flags)) return NRMF_EINVAL;
  return nrmf_host_impl<float>(n, host_x, host_out, flags, ws, ws_bytes, stream);
}

// test hook (not in nrmf.h): force the persistent grid size, 0 = automatic
#ifdef NRMF_PROBE_TRACE
int nrmf_debug_set_trace(void* buf, unsigned cap) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  unsigned z = 0;
  if (cudaMemcpyToSymbol(nrmf::g_trace, &p, sizeof(p)) != cudaSuccess) return NRMF_ECUDA;
  if (cudaMemcpyToSymbol(nrmf::g_trace_cap, &cap, sizeof(cap)) != cudaSuccess) return NRMF_ECUDA;
  if (cudaMemcpyToSymbol(nrmf::g_trace_n, &z, sizeof(z)) != cudaSuccess) return NRMF_ECUDA;
  return NRMF_OK;
}
#endif

int nrmf_debug_set_g0(int g0) {
  g_g0_override = (g0 < 0 || g0 > 4) ? -1 : g0;
  return NRMF_OK;
}

int nrmf_debug_set_gap_stream(int on) {
  g_gap_stream = on != 0;
  return NRMF_OK;
}

int nrmf_debug_set_unal_stream(int on) {
  g_unal_stream = on != 0;
  return NRMF_OK;
}

int nrmf_debug_set_split_ll(int on) {
  g_split_ll = on != 0;
  return NRMF_OK;
}

int nrmf_debug_set_cta_step(int on) {
  g_cta_step0 = on != 0;
  return NRMF_OK;
}

int nrmf_debug_set_grid(int grid) {
  g_grid_override = grid < 0 ? 0 : grid;
  return NRMF_OK;
}

}  // extern "C"
