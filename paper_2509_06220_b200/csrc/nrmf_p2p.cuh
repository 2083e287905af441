// nrmf_p2p.cuh -- the rank level of the tree through peer memory:
// one warp per rank writes the rank's subtree value into every peer's slot
// over NVLink (P2P stores to CUDA-IPC-mapped buffers), publishes it with a
// flag, waits for every rank's flag in its own buffer and evaluates the rank
// tree itself -- the same tree as the ncclAllGather + rank-tree-kernel path
// (e:hr P:216-231; fixed order as P:1077-1084 requires), without an NCCL
// launch.
//
// Peer buffer (kP2PBytes, one per rank, zero-filled once): two parity halves
// (epoch & 1) of [flags: kP2PMaxRanks x u32][values: kP2PMaxRanks x 8 B], and
// the rank's call counter (epoch) at kP2PEpochOff.  Call e writes half e&1; a
// rank can only reach call e+2 after finishing call e+1, which needs every
// rank's e+1 flag, which a rank writes only after it has finished reading call
// e -- so a half is never overwritten while read.  The epoch lives in device
// memory and is advanced by the exchange itself (1, 2, 3, ... on every rank,
// since every rank makes the same calls), so a call can be captured in a CUDA
// graph and replayed.
#pragma once

#include <cstdint>

#include "nrmf_device.cuh"

namespace nrmf {

constexpr int kP2PMaxRanks = 32;
constexpr int kP2PHalf = kP2PMaxRanks * 4 + kP2PMaxRanks * 8;  // 384 B
constexpr int kP2PEpochOff = 2 * kP2PHalf;
constexpr int kP2PBytes = 1024;
static_assert(kP2PEpochOff + 4 <= kP2PBytes, "p2p buffer");

struct PeerArgs {
  char* const* peers;  // device array: peers[r] = rank r's buffer as mapped here (peers[rank] = own)
  int world;           // <= kP2PMaxRanks
  int rank;
  unsigned* err;       // nullable: set to 1 if a flag did not arrive in time
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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
  if (lane < a.world) {  // lane p publishes this rank's value in peer p's buffer
    char* pb = a.peers[lane] + half;
    volatile F* slot = reinterpret_cast<volatile F*>(pb + kP2PMaxRanks * 4 + a.rank * 8);
    *slot = local;
    __threadfence_system();  // the value is visible before the flag
    st_release_sys(reinterpret_cast<unsigned*>(pb) + a.rank, epoch);
  }
  F v = F(0);
  if (lane < a.world) {  // lane r waits for rank r's value in this rank's buffer
    const char* own = a.peers[a.rank] + half;
    const unsigned* flag = reinterpret_cast<const unsigned*>(own) + lane;
    bool ok = true;
    for (long long spins = 0; ld_acquire_sys(flag) != epoch; ++spins) {
      if (spins > (1ll << 24)) {  // ~ seconds: a rank did not call; report, do not hang
        ok = false;
        break;
      }
      __nanosleep(128);
    }
    if (ok) {
      v = *reinterpret_cast<const volatile F*>(own + kP2PMaxRanks * 4 + lane * 8);
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
