// Checks that sm_100 packed fp32 ops (add/sub/mul/fma .rn.f32x2) equal the
// scalar IEEE RN ops bit for bit, including subnormal inputs and results.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float rnd(uint64_t z, int kind) {
  uint32_t b = (uint32_t)z;
  if (kind == 1) b &= 0x807FFFFFu;                  // subnormal
  if (kind == 2) b = (b & 0x80FFFFFFu) | 0x00800000u; // tiny normal
  if (kind == 3) b = (b & 0x83FFFFFFu) | 0x3C000000u; // moderate
  return __uint_as_float(b);
}
__global__ void k(unsigned long long n, unsigned long long* bad) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const int kind = i & 3;
    float a0 = rnd(splitmix(4 * i), kind), a1 = rnd(splitmix(4 * i + 1), 3 - kind);
    float b0 = rnd(splitmix(4 * i + 2), kind), b1 = rnd(splitmix(4 * i + 3), kind);
    float c0 = rnd(splitmix(~i), (kind + 1) & 3), c1 = rnd(splitmix(~i ^ 77), kind);
    unsigned long long A, B, C, D;
    asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b0), "f"(b1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(C) : "f"(c0), "f"(c1));
    float d0, d1;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d0), "=f"(d1) : "l"(D));
    if (__float_as_uint(d0) != __float_as_uint(__fadd_rn(a0, b0)) || __float_as_uint(d1) != __float_as_uint(__fadd_rn(a1, b1))) atomicAdd(bad + 0, 1);
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d0), "=f"(d1) : "l"(D));
    if (__float_as_uint(d0) != __float_as_uint(__fsub_rn(a0, b0)) || __float_as_uint(d1) != __float_as_uint(__fsub_rn(a1, b1))) atomicAdd(bad + 1, 1);
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d0), "=f"(d1) : "l"(D));
    if (__float_as_uint(d0) != __float_as_uint(__fmul_rn(a0, b0)) || __float_as_uint(d1) != __float_as_uint(__fmul_rn(a1, b1))) atomicAdd(bad + 2, 1);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(A), "l"(B), "l"(C));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d0), "=f"(d1) : "l"(D));
    if (__float_as_uint(d0) != __float_as_uint(__fmaf_rn(a0, b0, c0)) || __float_as_uint(d1) != __float_as_uint(__fmaf_rn(a1, b1, c1))) atomicAdd(bad + 3, 1);
  }
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4 * sizeof(unsigned long long));
  cudaMemset(d, 0, 4 * sizeof(unsigned long long));
  const unsigned long long n = 1ull << 30;
  k<<<148 * 16, 256>>>(n, d);
  unsigned long long h[4];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("mismatches over %llu pairs: add %llu sub %llu mul %llu fma %llu\n", n, h[0], h[1], h[2], h[3]);
  return (h[0] | h[1] | h[2] | h[3]) ? 1 : 0;
}
