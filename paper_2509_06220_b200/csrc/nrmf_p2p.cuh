// nrmf_p2p.cuh -- the rank level of the tree through peer memory:
// one warp per rank writes the rank's subtree value into every peer's slot
// over NVLink (P2P stores to CUDA-IPC-mapped buffers), publishes it with a
// flag, waits for every rank's flag in its own buffer and evaluates the rank
// tree itself -- the same tree as the ncclAllGather + rank-tree-kernel path
// (e:hr P:216-231; fixed order as P:1077-1084 requires), without an NCCL
// launch.
//
// Peer buffer (kP2PBytes, one per rank, zero-filled once): two parity halves
// (epoch & 1) of kP2PMaxRanks 16-byte slots, and the rank's call counter
// (epoch) at kP2PEpochOff.  Slot r of rank p's buffer receives rank r's value
// for call e as {lo32, e, hi32, e}: each aligned 8-byte half carries the
// epoch beside its 32 data bits and is stored and loaded as one unit (the
// "LL" flag-in-data idea NCCL uses for small messages), so a reader that sees
// epoch e in both halves has the whole value -- no system-scope fence on
// either side (a release/acquire pair across GPUs costs microseconds).  Call
// e writes half e&1; a rank can only reach call e+2 after finishing call e+1,
// which needs every rank's e+1 value, which a rank writes only after it has
// finished reading call e -- so a half is never overwritten while read.  The
// epoch lives in device memory and is advanced by the exchange itself (1, 2,
// 3, ... on every rank, since every rank makes the same calls), so a call can
// be captured in a CUDA graph and replayed.
#pragma once

#include <cstdint>

#include "nrmf_device.cuh"

namespace nrmf {

constexpr int kP2PMaxRanks = 32;
constexpr int kP2PSlot = 16;
constexpr int kP2PHalf = kP2PMaxRanks * kP2PSlot;  // 512 B
constexpr int kP2PEpochOff = 2 * kP2PHalf;
constexpr int kP2PBytes = 1280;
static_assert(kP2PEpochOff + 4 <= kP2PBytes, "p2p buffer");

struct PeerArgs {
  char* const* peers;  // device array: peers[r] = rank r's buffer as mapped here (peers[rank] = own)
  int world;           // <= kP2PMaxRanks
  int rank;
  unsigned* err;       // nullable: set to 1 if a value did not arrive in time
};

__device__ __forceinline__ void st_ll(char* p, uint32_t lo, uint32_t hi, uint32_t e) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(lo), "r"(e), "r"(hi), "r"(e)
               : "memory");
}
__device__ __forceinline__ void st_ll2(char* p, uint32_t lo, uint32_t hi, uint32_t e0, uint32_t e1) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(lo), "r"(e0), "r"(hi), "r"(e1)
               : "memory");
}
__device__ __forceinline__ void ld_ll(const char* p, uint32_t& lo, uint32_t& e0, uint32_t& hi, uint32_t& e1) {
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(lo), "=r"(e0), "=r"(hi), "=r"(e1)
               : "l"(p) : "memory");
}
// GPU-scope forms for slots read on the same device (the split kernel's last
// step): strong .gpu loads and stores stay in this GPU's L2 coherence domain
// (the .sys-scope volatile forms above are for peer memory)
__device__ __forceinline__ void st_ll2_gpu(char* p, uint32_t lo, uint32_t hi, uint32_t e0, uint32_t e1) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(lo), "r"(e0), "r"(hi), "r"(e1)
               : "memory");
}
__device__ __forceinline__ void ld_ll_gpu(const char* p, uint32_t& lo, uint32_t& e0, uint32_t& hi, uint32_t& e1) {
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(lo), "=r"(e0), "=r"(hi), "=r"(e1)
               : "l"(p) : "memory");
}
__device__ __forceinline__ void to_words(double v, uint32_t& lo, uint32_t& hi) {
  lo = (uint32_t)__double2loint(v);
  hi = (uint32_t)__double2hiint(v);
}
__device__ __forceinline__ void to_words(float v, uint32_t& lo, uint32_t& hi) {
  lo = __float_as_uint(v);
  hi = 0u;
}
template <typename F>
__device__ __forceinline__ F from_words(uint32_t lo, uint32_t hi) {
  if constexpr (sizeof(F) == 8) return __hiloint2double((int)hi, (int)lo);
  else return __uint_as_float(lo);
}

// Pull this rank's exchange buffer (epoch word, both slot halves) and the
// peer-pointer array into L2 ahead of rank_exchange, whose reads of them are
// otherwise dependent DRAM misses (pointer, then epoch) at the very end of the
// call.  Called by a warp with idle time before it writes the root (the split
// kernel's slot-polling warp).  Warp-collective; prefetches only, no ordering.
__device__ __forceinline__ void prefetch_exchange(char* const* peers, int rank) {
  const int lane = threadIdx.x & 31;
  if (lane < 2) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(peers) + lane * 128));
  const char* own = peers[rank];
  if (lane * 128 < kP2PBytes) asm volatile("prefetch.global.L2 [%0];" ::"l"(own + lane * 128));
}

// Warp-collective (all 32 lanes).  Returns, in every lane, the balanced tree
// over the first nr rank values (nr a power of two <= world: the ranks that
// own part of the tile tree), with v1_hypot or cr_hypot (cr) at every node.
template <typename F>
__device__ F rank_exchange(F local, const PeerArgs& a, int nr, int cr) {
  const int lane = threadIdx.x & 31;
  unsigned* const own_epoch = reinterpret_cast<unsigned*>(a.peers[a.rank] + kP2PEpochOff);
  const uint32_t epoch = *reinterpret_cast<volatile unsigned*>(own_epoch) + 1u;
  const uint32_t half = (epoch & 1u) * kP2PHalf;
  uint32_t wlo, whi;
  to_words(local, wlo, whi);
  if (lane < a.world)  // lane p publishes this rank's value in peer p's buffer
    st_ll(a.peers[lane] + half + a.rank * kP2PSlot, wlo, whi, epoch);
  F v = F(0);
  if (lane < a.world) {  // lane r waits for rank r's value in this rank's buffer
    const char* slot = a.peers[a.rank] + half + lane * kP2PSlot;
    uint32_t lo, e0, hi, e1;
    bool ok = true;
    for (long long spins = 0;; ++spins) {
      ld_ll(slot, lo, e0, hi, e1);
      if (e0 == epoch && e1 == epoch) break;
      if (spins > (1ll << 24)) {  // ~ seconds: a rank did not call; report, do not hang
        ok = false;
        break;
      }
      if (spins > 64) __nanosleep(64);
    }
    if (ok) {
      v = from_words<F>(lo, hi);
    } else {
      v = sizeof(F) == 8 ? F(__longlong_as_double(0x7ff8000000000000ll)) : F(__int_as_float(0x7fc00000));
      if (a.err != nullptr) atomicExch(a.err, 1u);
    }
  }
  __syncwarp();
  if (lane == 0) *reinterpret_cast<volatile unsigned*>(own_epoch) = epoch;  // next call: epoch + 1
  if (lane >= nr) v = F(0);
  for (int off = 1; off < nr; off <<= 1) v = top_node(v, __shfl_xor_sync(0xffffffffu, v, off), cr);
  return v;
}

}  // namespace nrmf
