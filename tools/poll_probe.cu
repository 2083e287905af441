// Dev probe: latency of one poll round of the split kernel's last step (one
// warp, 8 x 16-byte slots per lane = 4 KiB, all loads issued before the first
// compare), for several load flavours, with the slots L2-resident (warm) or
// after a 256 MiB write (the bench's L2 flush).  Prints cycles per round.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/poll_probe.bin tools/poll_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__device__ __forceinline__ void ld16(const char* p, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  if (KIND == 0)
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
  else if (KIND == 1)
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
  else if (KIND == 2)
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
  else if (KIND == 4)
    asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
  else if (KIND == 5)
    asm volatile("ld.relaxed.gpu.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
  else
    asm volatile("ld.acquire.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
}

template <int KIND, int KP>
__global__ void poll(const char* slots, int rounds, long long* out, unsigned* sink, const double* busy) {
  const int lane = threadIdx.x & 31;
  if (blockIdx.x != 0 || threadIdx.x >= 32) {  // background: the split kernel's load + FP64 work
    if (busy == nullptr) return;
    const double* p = busy + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16;
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) v += __ldcs(p + j);
    for (int k = 0; k < 3000; ++k) v = __fma_rn(v, 0.999999, 1e-3);
    if (v == 12345.0) *sink = 1;
    return;
  }
  unsigned acc = 0;
  long long t0 = clock64();
  long long first = 0;
  for (int r = 0; r < rounds; ++r) {
    uint32_t a[KP], b[KP], c[KP], d[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) ld16<KIND>(slots + 16 * (lane * KP + j), a[j], b[j], c[j], d[j]);
    bool all = true;
#pragma unroll
    for (int j = 0; j < KP; ++j) all &= (b[j] ^ d[j]) == 0u;
    if (__all_sync(0xffffffffu, all) && a[0] == 0xdeadbeefu) break;  // a branch on the vote, as in the combiner
    acc += a[0] + c[KP - 1];
    if (r == 0) first = clock64() - t0;
  }
  long long t1 = clock64();
  if (lane == 0) {
    out[0] = first;
    out[1] = (t1 - t0 - first) / (rounds > 1 ? rounds - 1 : 1);
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  char* slots;
  long long* out;
  unsigned* sink;
  char* flush;
  cudaMalloc(&slots, 1 << 20);
  cudaMemset(slots, 0, 1 << 20);
  cudaMalloc(&out, 16);
  cudaMalloc(&sink, 4);
  cudaMalloc(&flush, 256u << 20);
  double* busy;
  cudaMalloc(&busy, 2 * 256 * 256 * 16 * sizeof(double));  // 16 MiB
  const char* names[6] = {"relaxed.gpu", "volatile", "cg", "acquire.gpu", "relaxed.sys", "rlx.gpu.noL1"};
  const int kinds[5] = {0, 1, 4, 5, 3};
  for (int bz = 0; bz < 2; ++bz)
  for (int ki = 0; ki < 5; ++ki)
  for (int kp = 1; kp <= 8; kp *= 2) {
      const int kind = kinds[ki];
      const int fl = 1;
      const unsigned grid = bz ? 512 : 1;
      const double* bp = bz ? busy : nullptr;
      long long h[2], acc0 = 0, acc1 = 0;
      const int reps = 10;
      for (int rep = 0; rep < reps; ++rep) {
        if (fl) cudaMemsetAsync(flush, rep, 256u << 20);
#define L(K, P) if (kind == K && kp == P) poll<K, P><<<grid, 256>>>(slots, 16, out, sink, bp);
#define LL(K) L(K, 1) L(K, 2) L(K, 4) L(K, 8)
        LL(0) LL(1) LL(3) LL(4) LL(5)
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        acc0 += h[0];
        acc1 += h[1];
      }
      printf("%s %-12s KP=%d: first round %6lld cycles, later rounds %6lld cycles\n", bz ? "busy grid" : "alone    ",
             names[kind], kp, acc0 / reps, acc1 / reps);
    }
  return 0;
}
