// fhn_resident.cuh -- one persistent launch for mid-size single lattices
// (512^2 .. 1536^2): the whole torus lives in the shared memory of the SMs
// for the entire advance.
//
// Why: a mid-size lattice cannot fill the chip with the wavefront kernel's
// long segments, so its launches are latency-bound (1024^2: ~10 us per
// 4-level launch, 385-409k Mcell-updates/s with graphs).  Here
//   * CTA p (one per SM, 16 warps, co-resident by cooperative launch) owns R
//     consecutive rows and keeps them, plus K halo rows above and below, in
//     two shared-memory buffers (u and v planes of R + 2K rows);
//   * a block of K levels runs level by level between the two buffers (each
//     thread owns one 4-column group of a row range and keeps a 3-row
//     register window; column neighbours are read from shared memory, with
//     the torus column wrap), the computed rows shrinking by one per level
//     on each side, so after K levels the R owned rows are exact;
//   * then the K top and K bottom owned rows go to a global exchange slot
//     (double-buffered by block parity), a release store publishes the
//     block number, and the CTA acquires both ring neighbours' words and
//     copies their edge rows (from L2) into its halo rows -- no grid-wide
//     barrier, only the two neighbours synchronise.
// Arithmetic is fhn_cell, unchanged, so results are bit-identical to the
// wavefront kernel.  Blow-up: the own rows of every block's last level are
// folded for finiteness; on a non-finite value the host re-runs the advance
// on the wavefront path, which reports the exact iteration and leaves the
// post-blow-up state (the input buffer is never written).
#pragma once

#include "fhn_stencil.cuh"

namespace rdcnn_dev {

constexpr int kResidentThreads = 512;

struct ResidentArgs {
  const float* u_in;
  const float* v_in;
  float* u_out;
  float* v_out;
  int rows, cols;
  int R;          // rows per CTA (the last CTA may own fewer, >= K)
  int P;          // CTAs in the ring
  long long steps;
  ParamsT<float> p;
  float* xbuf;    // [P][2 parity][2 sides][K rows][2 planes][cols]
  unsigned* flags;        // [P], zero at launch: blocks published
  unsigned* bad;          // set to 1 when the advance produced a non-finite value
};

// Shared memory of a CTA: 2 buffers x 2 planes x (R + 2K) rows x cols floats.
__host__ __device__ constexpr size_t resident_smem_bytes(int R, int K, int cols) {
  return (size_t)2 * 2 * (size_t)(R + 2 * K) * (size_t)cols * sizeof(float);
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <int K, int kArith>
__global__ void __launch_bounds__(kResidentThreads, 1) fhn_resident_kernel(const ResidentArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* const sm = reinterpret_cast<float*>(smem_raw);
  const int P = a.P;
  const int p = blockIdx.x;
  const int cols = a.cols;
  const int G = cols / 4;
  const int own = min(a.R, a.rows - p * a.R);
  const int nr = own + 2 * K;              // buffer rows in use
  const int NR = a.R + 2 * K;              // buffer rows allocated
  const size_t plane = (size_t)NR * cols;  // floats per plane
  float* const buf[2] = {sm, sm + 2 * plane};
  const int tid = threadIdx.x;
  const Params prm = a.p;
  const float neg_eps = -prm.eps;

  // Load rows p*R-K .. p*R+own+K-1 (torus wrap) into buffer 0.
  const int row0 = p * a.R - K;
  for (int i = tid; i < nr * G; i += kResidentThreads) {
    const int r = i / G, g = i - r * G;
    int gr = row0 + r;
    gr = gr < 0 ? gr + a.rows : gr >= a.rows ? gr - a.rows : gr;
    const size_t go = (size_t)gr * cols + 4 * g;
    const float4 u = __ldg(reinterpret_cast<const float4*>(a.u_in + go));
    const float4 v = __ldg(reinterpret_cast<const float4*>(a.v_in + go));
    *reinterpret_cast<float4*>(buf[0] + (size_t)r * cols + 4 * g) = u;
    *reinterpret_cast<float4*>(buf[0] + plane + (size_t)r * cols + 4 * g) = v;
  }
  __syncthreads();

  // Thread -> (column group, row part).
  const int nparts = kResidentThreads / G;
  const int g = tid % G;
  const int part = tid / G;
  const bool active = part < nparts;
  const int gl = g == 0 ? G - 1 : g - 1;
  const int gr = g == G - 1 ? 0 : g + 1;

  const long long nblocks = (a.steps + K - 1) / K;
  const int pp = p == 0 ? P - 1 : p - 1;
  const int pn = p + 1 == P ? 0 : p + 1;
  const size_t xside = (size_t)K * 2 * cols;  // floats of one side's edge rows (both planes)
  int cur = 0;
  Finite<float> fin;
  for (long long b = 0; b < nblocks; ++b) {
    const long long left = a.steps - b * K;
    const int L = left < K ? (int)left : K;
    for (int t = 1; t <= L; ++t) {
      const float* su = buf[cur];
      const float* sv = buf[cur] + plane;
      float* du = buf[cur ^ 1];
      float* dv = buf[cur ^ 1] + plane;
      const int lo0 = t, hi0 = nr - t;
      const int ch = (hi0 - lo0 + nparts - 1) / nparts;
      const int lo = lo0 + part * ch;
      const int hi = min(hi0, lo + ch);
      if (active && lo < hi) {
        Row<4, float> up, ce, dn;
        auto ld = [&](int r, Row<4, float>& x) {
          const float4 u = *reinterpret_cast<const float4*>(su + (size_t)r * cols + 4 * g);
          const float4 v = *reinterpret_cast<const float4*>(sv + (size_t)r * cols + 4 * g);
          x.u[0] = u.x; x.u[1] = u.y; x.u[2] = u.z; x.u[3] = u.w;
          x.v[0] = v.x; x.v[1] = v.y; x.v[2] = v.z; x.v[3] = v.w;
        };
        ld(lo - 1, up);
        ld(lo, ce);
        for (int r = lo; r < hi; ++r) {
          ld(r + 1, dn);
          const size_t ro = (size_t)r * cols;
          const float ul = su[ro + 4 * gl + 3], vl = sv[ro + 4 * gl + 3];
          const float ur = su[ro + 4 * gr], vr = sv[ro + 4 * gr];
          Row<4, float> o;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float u_l = k > 0 ? ce.u[k - 1] : ul;
            const float u_r = k < 3 ? ce.u[k + 1] : ur;
            const float v_l = k > 0 ? ce.v[k - 1] : vl;
            const float v_r = k < 3 ? ce.v[k + 1] : vr;
            fhn_cell<float, kArith>(ce.u[k], ce.v[k], u_r, u_l, dn.u[k], up.u[k], v_r, v_l, dn.v[k], up.v[k], prm,
                                    neg_eps, o.u[k], o.v[k]);
          }
          *reinterpret_cast<float4*>(du + ro + 4 * g) = make_float4(o.u[0], o.u[1], o.u[2], o.u[3]);
          *reinterpret_cast<float4*>(dv + ro + 4 * g) = make_float4(o.v[0], o.v[1], o.v[2], o.v[3]);
          if (t == L && r >= K && r < K + own) fold_finite<4, float>(fin, o);
          up = ce;
          ce = dn;
        }
      }
      cur ^= 1;
      __syncthreads();
    }
    if (b + 1 == nblocks) break;
    // Exchange: own rows [K, 2K) and [own, own+K) out, halo rows in.
    const float* fu = buf[cur];
    const float* fv = buf[cur] + plane;
    float* const xs = a.xbuf + ((size_t)p * 2 + (size_t)(b & 1)) * 2 * xside;
    for (int i = tid; i < 2 * K * G; i += kResidentThreads) {
      const int side = i / (K * G);
      const int rem = i - side * K * G;
      const int r = rem / G, gg = rem - r * G;
      const int br = side == 0 ? K + r : own + r;
      const float4 u = *reinterpret_cast<const float4*>(fu + (size_t)br * cols + 4 * gg);
      const float4 v = *reinterpret_cast<const float4*>(fv + (size_t)br * cols + 4 * gg);
      float* x = xs + side * xside + (size_t)r * 2 * cols;
      __stcg(reinterpret_cast<float4*>(x + 4 * gg), u);
      __stcg(reinterpret_cast<float4*>(x + cols + 4 * gg), v);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_gpu(a.flags + p, (unsigned)(b + 1));
      while (ld_acquire_gpu(a.flags + pp) < (unsigned)(b + 1)) __nanosleep(32);
      while (ld_acquire_gpu(a.flags + pn) < (unsigned)(b + 1)) __nanosleep(32);
    }
    __syncthreads();
    const float* xp = a.xbuf + ((size_t)pp * 2 + (size_t)(b & 1)) * 2 * xside + xside;  // prev's bottom rows
    const float* xn = a.xbuf + ((size_t)pn * 2 + (size_t)(b & 1)) * 2 * xside;          // next's top rows
    float* hu = buf[cur];
    float* hv = buf[cur] + plane;
    for (int i = tid; i < 2 * K * G; i += kResidentThreads) {
      const int side = i / (K * G);
      const int rem = i - side * K * G;
      const int r = rem / G, gg = rem - r * G;
      const float* x = (side == 0 ? xp : xn) + (size_t)r * 2 * cols;
      const int br = side == 0 ? r : own + K + r;
      *reinterpret_cast<float4*>(hu + (size_t)br * cols + 4 * gg) = __ldcg(reinterpret_cast<const float4*>(x + 4 * gg));
      *reinterpret_cast<float4*>(hv + (size_t)br * cols + 4 * gg) =
          __ldcg(reinterpret_cast<const float4*>(x + cols + 4 * gg));
    }
    __syncthreads();
  }
  // Blow-up: non-finite values are absorbing, so the fold over every block's
  // last-level own rows is non-finite iff some block blew up.
  if (__syncthreads_or(!(fin.m <= 3.402823466e38f)) && tid == 0) atomicExch(a.bad, 1u);

  // Own rows out.
  const float* fu = buf[cur];
  const float* fv = buf[cur] + plane;
  for (int i = tid; i < own * G; i += kResidentThreads) {
    const int r = i / G, gg = i - r * G;
    const size_t go = (size_t)(p * a.R + r) * cols + 4 * gg;
    __stcs(reinterpret_cast<float4*>(a.u_out + go), *reinterpret_cast<const float4*>(fu + (size_t)(K + r) * cols + 4 * gg));
    __stcs(reinterpret_cast<float4*>(a.v_out + go), *reinterpret_cast<const float4*>(fv + (size_t)(K + r) * cols + 4 * gg));
  }
}

}  // namespace rdcnn_dev
