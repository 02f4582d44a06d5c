// Microbenchmark: issue/throughput of scalar FFMA/FADD vs packed FFMA2/FADD2
// on sm_100a (used to decide whether the stencil should pack cell pairs).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pk(float a, float b){ unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float a[8]; unsigned long long p[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 0.001f + i; p[i] = pk(a[i], a[i] + 1.f); }
  const unsigned long long S = pk(s, s);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = __fmaf_rn(a[i], s, 0.5f);
      if (MODE == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(p[i]) : "l"(S));
      if (MODE == 2) a[i] = __fadd_rn(a[i], s);
      if (MODE == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(S));
    }
  }
  float r = 0; for (int i = 0; i < 8; ++i) { r += a[i]; float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(p[i])); r += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 8, 1024>>>(d, iters, 0.999f);
      if (mode == 1) k<1><<<148 * 8, 1024>>>(d, iters, 0.999f);
      if (mode == 2) k<2><<<148 * 8, 1024>>>(d, iters, 0.999f);
      if (mode == 3) k<3><<<148 * 8, 1024>>>(d, iters, 0.999f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double lane_ops = 148.0 * 8 * 1024 * iters * 8 * ((mode & 1) ? 2 : 1);
      if (rep) printf("mode %d (%s): %.3f ms, %.2f T lane-ops/s\n", mode,
                      mode == 0 ? "FFMA" : mode == 1 ? "FFMA2" : mode == 2 ? "FADD" : "FADD2", ms, lane_ops / ms / 1e9);
    }
  }
  return 0;
}
