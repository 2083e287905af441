// Dev microbenchmark: FP64-pipe cost of DFMA/DMUL as a function of the number
// of distinct register operands (register-file bank model: a double occupies
// one even and one odd register, so k distinct double sources need k reads
// per bank).  Cycles are measured with clock64() inside the kernel, so the
// result does not depend on the (unknown) SM clock under load.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256, 1) k(double* out, long long* cyc, int iters) {
  constexpr int C = 8;
  double x[C], y[C], z[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    x[c] = 1.0 + threadIdx.x * 1e-4 + c;
    y[c] = 0.999999 - c * 1e-7 + threadIdx.x * 1e-12;
    z[c] = 1e-9 * (c + 1) + threadIdx.x * 1e-15;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (OP == 0) x[c] = __fma_rn(x[c], y[c], z[c]);     // 3 distinct registers
      if (OP == 1) x[c] = __fma_rn(x[c], y[c], 1e-9);     // 2 distinct + immediate
      if (OP == 3) x[c] = __dmul_rn(x[c], y[c]);           // 2 distinct
      if (OP == 4) x[c] = __fma_rn(x[c], y[0], z[0]);      // 3 distinct, 2 shared across chains
      if (OP == 5) x[c] = __fma_rn(-x[c], x[c], 1.0);      // 1 distinct
      if (OP == 6) {  // 32-bit selects, operands of equal parity (hi words: both odd)
        const bool p = __double2hiint(x[c]) > __double2hiint(y[c]);
        x[c] = __hiloint2double(p ? __double2hiint(y[c]) : __double2hiint(z[c]), __double2loint(x[c]));
      }
      if (OP == 7) {  // 32-bit selects, operands of different parity (hi of y, lo of z)
        const bool p = __double2hiint(x[c]) > __double2hiint(y[c]);
        x[c] = __hiloint2double(p ? __double2hiint(y[c]) : __double2loint(z[c]), __double2loint(x[c]));
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name) {
  double* out;
  long long* cyc;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&out, 64);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  const int iters = 4000;
  k<OP><<<sms, 256>>>(out, cyc, 10);
  k<OP><<<sms, 256>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  // per SM: 8 warps, 2 per SMSP, 8 ops per iteration
  const double warp_instr_per_smsp = 2.0 * 8 * iters;
  printf("%-28s %.2f cycles per warp-instruction per SMSP\n", name, avg / warp_instr_per_smsp);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("DFMA 3 distinct regs");
  run<4>("DFMA 3 regs, 2 chain-shared");
  run<1>("DFMA 2 regs + imm");
  run<3>("DMUL 2 regs");
  run<5>("DFMA 1 reg + imm");
  run<6>("ISETP+SEL same parity (per pair)");
  run<7>("ISETP+SEL mixed parity (per pair)");
  return 0;
}
