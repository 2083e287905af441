// Dev probe kernels for tools/timer_probe.py (ctypes): a globaltimer spin and
// the smallest globaltimer step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/timer_probe_k.so tools/timer_probe_k.cu
#include <cuda_runtime.h>
__global__ void spin(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)ns);
}
__global__ void ticks(unsigned long long* out, int n) {
  unsigned long long prev, t, best = ~0ull;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  for (int i = 0; i < n; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { if (t - prev < best) best = t - prev; prev = t; }
  }
  out[0] = best;
}
extern "C" int launch_spin(long long ns, void* stream) {
  spin<<<1, 32, 0, (cudaStream_t)stream>>>(ns);
  return (int)cudaGetLastError();
}
extern "C" int launch_ticks(void* out, int n, void* stream) {
  ticks<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long*)out, n);
  return (int)cudaGetLastError();
}
