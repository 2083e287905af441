// Dev microbenchmark: do FP64 (DFMA) and XU (MUFU) instructions share issue?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp64(double x) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ float rcp32(float x) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

// ND DFMA + NR MUFU.RCP64H + NF MUFU.RCP (f32) per iteration, independent chains
template <int ND, int NR, int NF>
__global__ void __launch_bounds__(256, 1) k(double* out, int iters) {
  double d[ND > 0 ? ND : 1], r[NR > 0 ? NR : 1];
  float f[NF > 0 ? NF : 1];
  for (int c = 0; c < ND; ++c) d[c] = 1.0 + threadIdx.x * 1e-4 + c;
  for (int c = 0; c < NR; ++c) r[c] = 1.5 + threadIdx.x * 1e-4 + c;
  for (int c = 0; c < NF; ++c) f[c] = 1.5f + threadIdx.x * 1e-4f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < ND; ++c) d[c] = __fma_rn(d[c], 1.0000001, 1e-9);
#pragma unroll
    for (int c = 0; c < NR; ++c) r[c] = rcp64(r[c]);
#pragma unroll
    for (int c = 0; c < NF; ++c) f[c] = rcp32(f[c]);
  }
  double s = 0;
  for (int c = 0; c < ND; ++c) s += d[c];
  for (int c = 0; c < NR; ++c) s += r[c];
  for (int c = 0; c < NF; ++c) s += f[c];
  if (s == 12345.0) out[0] = s;
}

template <int ND, int NR, int NF>
void run() {
  double* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  k<ND, NR, NF><<<sms * 2, 256>>>(out, 10);
  cudaEventRecord(e0);
  k<ND, NR, NF><<<sms * 2, 256>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  // cycles per iteration per warp per SMSP
  double warps_per_smsp = 2.0 * 8 / 4;
  double cyc = ms * 1e-3 * 1.965e9 / iters / warps_per_smsp;
  printf("DFMA x%d + RCP64H x%d + RCP32 x%d : %.1f cycles/iter/warp (pred: shared %.1f, separate %.1f)\n", ND, NR, NF,
         cyc, ND * 2.2 + NR * 8.0 + NF * 8.0, ND * 2.2 > (NR + NF) * 8.0 ? ND * 2.2 : (NR + NF) * 8.0);
}

int main() {
  run<16, 0, 0>(); run<0, 4, 0>(); run<0, 0, 4>(); run<16, 4, 0>(); run<16, 0, 4>(); run<8, 2, 0>(); run<8, 0, 2>();
  return 0;
}
