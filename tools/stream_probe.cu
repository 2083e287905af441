// Dev probe: what limits the stream loader's read bandwidth?  4 GiB read per
// launch, median of 20 launches (after 5), each variant once:
//   grid   : grid-stride LDG.128 over the whole array (the plain streaming read)
//   wLDG   : persistent 148 x 16 warps, each warp streams its own contiguous
//            chunks (C bytes, round-robin like the tree kernel) with LDG.128
//   wTMA S x B : the same chunks through a per-warp ring of S stages of B
//            bytes (cp.async.bulk + mbarrier), consumed by LDS.128 (the tree
//            kernel's loader), 16 or fewer warps per CTA
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp tools/stream_probe.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../paper_2509_06220_b200/csrc/nrmf_device.cuh"
using namespace nrmf;

__global__ void grid_k(const float4* x, long long n4, float* out) {
  float s = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(x + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.f) out[0] = s;
}

// warp w of the grid streams chunks w, w + W, ... of `chunk` bytes
__global__ void wldg_k(const char* x, long long bytes, long long chunk, float* out) {
  const int lane = threadIdx.x & 31;
  const long long W = (long long)gridDim.x * (blockDim.x / 32);
  const long long gw = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5);
  float s = 0;
  for (long long c = gw; c * chunk < bytes; c += W) {
    const float4* p = reinterpret_cast<const float4*>(x + c * chunk);
    for (long long i = lane; i < chunk / 16; i += 32 * 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(p + i + u * 32);
#pragma unroll
      for (int u = 0; u < 4; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (s == 12345.f) out[0] = s;
}

template <int S, int B>
__global__ void wtma_k(const char* x, long long bytes, long long chunk, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x / 32;
  const long long W = (long long)gridDim.x * nw;
  const long long gw = blockIdx.x * (long long)nw + w;
  const uint32_t ring = smem_u32(smem) + w * (S * B + 64);
  const uint32_t bars = ring + S * B;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bars + s * 8, 1);
    fence_mbar_init();
  }
  __syncwarp();
  // batches of this warp: chunk c = gw + k W, batch b within it
  const long long per_chunk = chunk / B;
  long long next_c = gw, next_b = 0;
  auto issue = [&](int slot) {
    if (next_c * chunk >= bytes) return;
    if (lane == 0) bulk_load(ring + slot * B, x + next_c * chunk + next_b * B, B, bars + slot * 8, policy_evict_first());
    if (++next_b == per_chunk) { next_b = 0; next_c += W; }
  };
  for (int s = 0; s < S; ++s) issue(s);
  float acc = 0;
  uint32_t consumed = 0;
  for (long long c = gw; c * chunk < bytes; c += W) {
    for (long long b = 0; b < per_chunk; ++b) {
      const int slot = consumed % S;
      mbar_wait(bars + slot * 8, (consumed / S) & 1);
#pragma unroll
      for (int r = 0; r < B / 512; ++r) {
        float a0, a1, a2, a3;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3)
                     : "r"(ring + slot * B + r * 512 + lane * 16) : "memory");
        acc += a0 + a1 + a2 + a3;
      }
      __syncwarp();
      ++consumed;
      issue(slot);
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

template <typename L>
float timeit(L launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int r = 0; r < 25; ++r) {
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 5) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

template <int S, int B>
void run_tma(const char* x, long long bytes, long long chunk, int warps, float* out) {
  const size_t sm = (size_t)warps * (S * B + 64);
  cudaFuncSetAttribute(wtma_k<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const float ms = timeit([&] { wtma_k<S, B><<<148, warps * 32, sm>>>(x, bytes, chunk, out); });
  const cudaError_t e = cudaGetLastError();
  printf("wTMA %dx%-5d warps %2d chunk %7lld: %.4f ms  %.0f GB/s %s\n", S, B, warps, chunk, ms, bytes / ms / 1e6,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const long long bytes = 1ll << 32;
  char* x;
  float* out;
  cudaMalloc(&x, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(x, 0, bytes);
  float ms = timeit([&] { grid_k<<<148 * 4, 512>>>(reinterpret_cast<const float4*>(x), bytes / 16, out); });
  printf("grid                              : %.4f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
  for (long long chunk : {16384ll, 65536ll, 262144ll}) {
    ms = timeit([&] { wldg_k<<<148, 512>>>(x, bytes, chunk, out); });
    printf("wLDG warps 16 chunk %7lld          : %.4f ms  %.0f GB/s\n", chunk, ms, bytes / ms / 1e6);
  }
  for (long long chunk : {16384ll, 65536ll, 262144ll}) {
    run_tma<2, 4096>(x, bytes, chunk, 16, out);
    run_tma<3, 4096>(x, bytes, chunk, 16, out);
    run_tma<4, 4096>(x, bytes, chunk, 12, out);
    run_tma<2, 8192>(x, bytes, chunk, 12, out);
    run_tma<4, 4096>(x, bytes, chunk, 8, out);
    run_tma<2, 16384>(x, bytes, chunk, 6, out);
  }
  cudaDeviceSynchronize();
  return 0;
}
