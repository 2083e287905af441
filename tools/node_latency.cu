// Dev microbenchmark: latency of one dependent fast node (v1h_fast_n<.,1>),
// one warp, a chain of `iters` nodes, timed with clock64 -- the per-level
// cost of the latency-bound tree tops (C1).  Also the same
// chain with a __shfl_xor between levels (the cross-thread levels) and the
// IEEE-intrinsic node for comparison.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_06220_b200/csrc/nrmf_device.cuh"
using namespace nrmf;

template <typename F, int MODE>
__global__ void chain(F* out, long long* cyc, int iters) {
  F a = F(1.5) + F(threadIdx.x) * F(1e-3), b = F(0.75);
  bool bad = false;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    F h;
    if (MODE == 0) h = v1h_fast<false>(a, b, bad);
    else if (MODE == 1) h = v1h_fast<false>(a, __shfl_xor_sync(0xffffffffu, a, 1 + (i & 15)), bad);
    else h = v1h(a, b);
    b = a;
    a = h * F(0.5);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (a == F(12345) || bad) out[0] = a;
}

template <typename F, int MODE>
void run(const char* name) {
  F* out; long long* cyc; cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
  const int iters = 4096;
  chain<F, MODE><<<1, 32>>>(out, cyc, 16);
  chain<F, MODE><<<1, 32>>>(out, cyc, iters);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%s: %.1f cycles per dependent node (%.3f us at 1.965 GHz)\n", name, (double)c / iters, (double)c / iters / 1965.0);
}

int main() {
  run<double, 0>("fp64 fast node");
  run<double, 1>("fp64 fast node + shfl");
  run<double, 2>("fp64 IEEE-intrinsic node");
  run<float, 0>("fp32 fast node");
  run<float, 1>("fp32 fast node + shfl");
  return 0;
}
