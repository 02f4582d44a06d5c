// analysis.cuh -- device-side snapshot statistics for batched sweeps
// (reference proj/include/rdcnn/sweep.hpp:48-112: growth_curve and
// classify_outcome), so a 4096-grid parameter sweep never ships its frames
// to the host.  Per grid and frame:
//   * min and max of the u layer (classify_outcome's minmax_element),
//   * the median exactly as std::nth_element(size/2) picks it: the element
//     of rank floor(n/2) in ascending order, found by radix selection on the
//     order-preserving integer image of the floating-point bit pattern,
//   * the count of cells with |double(x) - median| > threshold (growth_curve).
// All comparisons are exact, so the results equal the reference's on the
// same (finite) frames.  One CTA per (grid); frames are planar rows*cols.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rdcnn_dev {

template <class T>
struct Key;
template <>
struct Key<float> {
  using U = uint32_t;
  static constexpr int kBits = 32;
  __device__ __forceinline__ static U of(float x) {
    const U b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  }
  __device__ __forceinline__ static float value(U k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
  }
};
template <>
struct Key<double> {
  using U = unsigned long long;
  static constexpr int kBits = 64;
  __device__ __forceinline__ static U of(double x) {
    const U b = (U)__double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
  }
  __device__ __forceinline__ static double value(U k) {
    return __longlong_as_double((long long)((k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
  }
};

constexpr int kStatThreads = 512;

// min, max and the rank-floor(n/2) element of each grid's frame.
template <class T>
__global__ void __launch_bounds__(kStatThreads) frame_stats_kernel(const T* __restrict__ frames,
                                                                    long long n, double* mins,
                                                                    double* maxs, double* medians) {
  using K = Key<T>;
  using U = typename K::U;
  const T* x = frames + (size_t)blockIdx.x * (size_t)n;
  __shared__ unsigned hist[256];
  __shared__ U s_prefix;
  __shared__ long long s_rank;
  __shared__ T s_min[kStatThreads / 32], s_max[kStatThreads / 32];

  // min / max
  T mn = x[0], mx = x[0];
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const T v = x[i];
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const T a = __shfl_xor_sync(0xFFFFFFFFu, mn, o), b = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    s_min[threadIdx.x >> 5] = mn;
    s_max[threadIdx.x >> 5] = mx;
  }
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_rank = n / 2;  // nth_element(begin + size/2)
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = s_min[w] < mn ? s_min[w] : mn;
      mx = s_max[w] > mx ? s_max[w] : mx;
    }
    mins[blockIdx.x] = (double)mn;
    maxs[blockIdx.x] = (double)mx;
  }

  // radix select, 8 bits per pass from the top
  for (int shift = K::kBits - 8; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const U prefix = s_prefix;
    const U mask_hi = shift + 8 >= K::kBits ? U(0) : (~U(0) << (shift + 8));
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      const U k = K::of(x[i]);
      if ((k & mask_hi) == prefix) atomicAdd(&hist[(k >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long r = s_rank;
      int b = 0;
      for (; b < 255 && r >= (long long)hist[b]; ++b) r -= hist[b];
      s_rank = r;
      s_prefix = prefix | ((U)b << shift);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) medians[blockIdx.x] = (double)K::value(s_prefix);
}

// Cells with |double(x) - median| > threshold (sweep.hpp:60-62).
template <class T>
__global__ void __launch_bounds__(kStatThreads) frame_active_kernel(const T* __restrict__ frames,
                                                                     long long n,
                                                                     const double* medians,
                                                                     const double* thresholds,
                                                                     long long* counts) {
  const T* x = frames + (size_t)blockIdx.x * (size_t)n;
  const double med = medians[blockIdx.x], thr = thresholds[blockIdx.x];
  long long c = 0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x)
    c += fabs(__dsub_rn((double)x[i], med)) > thr;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  __shared__ long long s[kStatThreads / 32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    counts[blockIdx.x] = t;
  }
}

}  // namespace rdcnn_dev
