// Dev microbenchmark: FP64 pipe throughput and DFMA/MUFU latency on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fma_rn(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __fma_rn(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}

__global__ void rcp_lat(double* out, long long* cyc, int iters) {
  double x = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps = 4; warps <= 32; warps *= 2) {
    dim3 grid(sms * 1), block(32 * warps);
    dfma_tput<8><<<grid, block>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_tput<8><<<grid, block>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)sms * 32 * warps * 8 * iters;
    printf("dfma tput: %2d warps/SM x 8 chains: %.3f ms -> %.1f TFMA/s, %.1f DFMA/clk/SM at 1.965GHz\n",
           warps, ms, fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / 1.965e9);
  }
  dfma_lat<<<1, 32>>>(out, cyc, 1000, 1.0000001, 1e-9);
  dfma_lat<<<1, 32>>>(out, cyc, iters, 1.0000001, 1e-9);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dfma latency: %.2f cycles\n", (double)c / iters);
  rcp_lat<<<1, 32>>>(out, cyc, iters);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("rcp64h latency: %.2f cycles\n", (double)c / iters);
  return 0;
}
