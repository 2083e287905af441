// Dev microbenchmark: DFMA/DMUL throughput vs number of distinct register operands.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(double* out, int iters, double a, double b) {
  constexpr int C = 8;
  double x[C], y[C], z[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { x[c] = 1.0 + threadIdx.x * 1e-4 + c; y[c] = a + c * 1e-7; z[c] = b + c * 1e-9; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (MODE == 0) x[c] = __fma_rn(x[c], 1.0000001, 1e-9);   // 1 reg
      if (MODE == 1) x[c] = __fma_rn(x[c], y[c], 1e-9);        // 2 regs
      if (MODE == 2) x[c] = __fma_rn(x[c], y[c], z[c]);        // 3 regs
      if (MODE == 3) x[c] = __dmul_rn(x[c], y[c]);             // DMUL 2 regs
      if (MODE == 4) x[c] = __fma_rn(y[c], z[c], x[c]);        // 3 regs, acc last
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}

template <int MODE>
void run(const char* name) {
  double* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  k<MODE><<<sms * 2, 256>>>(out, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  k<MODE><<<sms * 2, 256>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double cyc = ms * 1e-3 * 1.965e9 / iters / 4.0 / 8;  // per warp-instruction per SMSP
  printf("%-28s %.2f cycles per warp-instr per SMSP\n", name, cyc);
}

int main() {
  run<0>("DFMA 1 reg operand"); run<1>("DFMA 2 reg operands"); run<2>("DFMA 3 reg operands");
  run<3>("DMUL 2 reg operands"); run<4>("DFMA 3 regs (acc last)");
  return 0;
}
