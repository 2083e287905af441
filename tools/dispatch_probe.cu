// Dev microbenchmark: does an FP64 warp instruction block dispatch of other
// instructions on the same SMSP for its 2 pipe cycles?
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NI, int NF>
__global__ void __launch_bounds__(256, 1) k(double* out, int iters) {
  double d[ND > 0 ? ND : 1];
  unsigned u[NI > 0 ? NI : 1];
  float f[NF > 0 ? NF : 1];
  for (int c = 0; c < ND; ++c) d[c] = 1.0 + threadIdx.x * 1e-4 + c;
  for (int c = 0; c < NI; ++c) u[c] = threadIdx.x * 7 + c;
  for (int c = 0; c < NF; ++c) f[c] = 1.0f + threadIdx.x * 1e-4f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < (ND > NI ? ND : NI); ++c) {
      if (c < ND) d[c] = __fma_rn(d[c], 1.0000001, 1e-9);
      if (c < NI) u[c] = (u[c] ^ 0x9e3779b9u) + 0x7f4a7c15u;   // 1 LOP3 + 1 IADD (or fused)
    }
#pragma unroll
    for (int c = 0; c < NF; ++c) f[c] = __fmaf_rn(f[c], 1.0000001f, 1e-9f);
  }
  double s = 0;
  for (int c = 0; c < ND; ++c) s += d[c];
  for (int c = 0; c < NI; ++c) s += u[c];
  for (int c = 0; c < NF; ++c) s += f[c];
  if (s == 12345.0) out[0] = s;
}

template <int ND, int NI, int NF>
void run() {
  double* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  k<ND, NI, NF><<<sms * 2, 256>>>(out, 10);
  cudaEventRecord(e0);
  k<ND, NI, NF><<<sms * 2, 256>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double cyc = ms * 1e-3 * 1.965e9 / iters / 4.0;  // per warp-iteration per SMSP (4 warps/SMSP)
  printf("DFMA x%2d + INT x%2d + FFMA x%2d: %.1f cycles/iter/warp\n", ND, NI, NF, cyc);
}

int main() {
  run<16, 0, 0>(); run<0, 16, 0>(); run<16, 16, 0>(); run<0, 0, 16>(); run<16, 0, 16>(); run<8, 16, 0>();
  return 0;
}
