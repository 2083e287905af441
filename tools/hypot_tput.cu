// Dev microbenchmark: throughput of the fast node sequence alone (registers
// only), K independent chains per thread, to separate the node cost from the
// tree / memory structure.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_06220_b200/csrc/nrmf_device.cuh"
using namespace nrmf;

template <int K, typename F>
__global__ void __launch_bounds__(256, 1) tput(F* out, int iters) {
  F a[K], b[K], h[K];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < K; ++k) { a[k] = F(1.5) + F(threadIdx.x) * F(1e-3) + F(k); b[k] = F(0.75) + F(k) * F(0.01); }
  for (int i = 0; i < iters; ++i) {
    v1h_fast_n<false, K>(a, b, h, bad);
#pragma unroll
    for (int k = 0; k < K; ++k) { b[k] = a[k]; a[k] = h[k] * F(0.5); }
  }
  F s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += a[k];
  if (s == F(12345) || bad) out[0] = s;
}

template <int K, typename F>
void run(int warps, const char* name) {
  F* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  dim3 grid(sms * warps / 8), block(256);
  tput<K, F><<<grid, block>>>(out, 10);
  cudaEventRecord(e0);
  tput<K, F><<<grid, block>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double hyp = (double)grid.x * 256 * K * iters;
  printf("%s K=%d warps/SM=%d: %.1f Ghypot/s -> 2^30 in %.3f ms (%.2f hypot/clk/SM @1.965)\n", name, K, warps,
         hyp / ms / 1e6, (double)(1 << 30) / (hyp / ms) , hyp / (ms * 1e-3) / sms / 1.965e9);
  cudaFree(out);
}

int main() {
  run<1, double>(8, "fp64"); run<2, double>(8, "fp64"); run<4, double>(8, "fp64"); run<8, double>(8, "fp64");
  run<1, double>(16, "fp64"); run<2, double>(16, "fp64"); run<4, double>(16, "fp64");
  run<1, double>(32, "fp64"); run<2, double>(32, "fp64");
  run<1, float>(16, "fp32"); run<4, float>(16, "fp32"); run<4, float>(32, "fp32");
  return 0;
}
