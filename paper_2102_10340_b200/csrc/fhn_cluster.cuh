// fhn_cluster.cuh -- persistent thread-block-cluster kernel for small single
// lattices (SURVEY.md §7 "launch-bound small grids"; cfg1 = 256^2 x 1000).
//
// The whole advance is ONE launch of ONE cluster of C CTAs (C <= 16,
// non-portable size).  CTA c owns R = rows / C consecutive rows; each warp
// owns RW consecutive rows and lane l owns W consecutive columns of them, so
// the state lives in registers for all `steps` iterations.  Per step:
//   1. each warp publishes its first and last row (u, v) into the CTA's
//      shared exchange rows of this step's parity; the CTA's first/last row
//      also goes into the previous/next CTA's halo row by st.async, whose
//      bytes are counted on the RECEIVER's mbarrier (complete_tx) -- the
//      torus ring across the cluster;
//   2. every thread arrives (release) on this parity's local mbarrier after
//      its own stores, the warp computes its interior rows (1..RW-2,
//      registers only) and then waits on it: the barrier completes when all
//      threads of the CTA have published; the CTA's two edge warps also wait
//      for both halo rows' bytes on the halo mbarrier.  There is no per-step cluster barrier and no
//      GPU-scope fence: a CTA synchronises only with its ring neighbours;
//   3. the edge rows: up/down rows from shared memory, left/right columns
//      from warp shuffles (the row wraps around the warp: the torus column
//      wrap), the reference cell update (fhn_cell, strict or fast).
// Blow-up: each warp records the first step whose output it saw non-finite
// (atomicMin); the host re-runs exactly that many steps from the call's
// input (kept: output goes to the other buffer), leaving the post-blow-up
// state and the exact iteration (engine.hpp:79, BlowUpError(iter+1)).
//
// Shared memory layout per CTA: two local mbarriers, two halo mbarriers, then
// X[2 parities][R + 2 rows][2 planes][W/4 chunks][32 lanes] float4 -- chunk-
// major so each STS.128/LDS.128 of a warp is 512 contiguous bytes (no bank
// conflicts).  Row 0 is the top halo, rows 1..R the CTA's own (only each
// warp's first and last are written), row R+1 the bottom halo.
#pragma once

#include "fhn_stencil.cuh"

namespace rdcnn_dev {

struct ClusterArgs {
  const float* u_in;
  const float* v_in;
  float* u_out;
  float* v_out;
  int rows, cols;
  int R;                 // rows per CTA (= warps per CTA x rows per warp)
  long long steps;
  ParamsT<float> p;
  long long* first_bad;  // preset to all-ones; atomicMin of the 1-based first non-finite step
};

constexpr int kClusterMax = 16;

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, unsigned v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void lds_v4(uint32_t addr, float& a, float& b, float& c, float& d) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
               : "r"(addr)
               : "memory");
}

// Asynchronous DSMEM store that counts its bytes on the RECEIVER's mbarrier
// (complete_tx): the receiver learns the halo row has landed by waiting on
// its own barrier, with no memory fence on either side.
__device__ __forceinline__ void stas_v4(uint32_t addr, float a, float b, float c, float d, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];\n"
               ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity_cta(uint32_t mbar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAITC_%=;\n"
      "}\n" ::"r"(mbar), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t mbar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(mbar), "r"(parity)
      : "memory");
}

// Bytes of dynamic shared memory for R rows per CTA: 32-byte header (four
// mbarriers) + the exchange rows.
template <int W>
constexpr int cluster_smem_bytes(int R) {
  return 32 + 2 * (R + 2) * 2 * W * 32 * 4;
}

template <int W>
__device__ __forceinline__ void publish_row(uint32_t addr, const float (&u)[W], const float (&v)[W]) {
  constexpr uint32_t kPlane = W / 4 * 32 * 16;
#pragma unroll
  for (int c = 0; c < W / 4; ++c) {
    sts_v4(addr + c * 512, u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3]);
    sts_v4(addr + c * 512 + kPlane, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
}
template <int W>
__device__ __forceinline__ void publish_row_remote(uint32_t addr, const float (&u)[W], const float (&v)[W],
                                                   uint32_t mbar) {
  constexpr uint32_t kPlane = W / 4 * 32 * 16;
#pragma unroll
  for (int c = 0; c < W / 4; ++c) {
    stas_v4(addr + c * 512, u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3], mbar);
    stas_v4(addr + c * 512 + kPlane, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3], mbar);
  }
}
template <int W>
__device__ __forceinline__ void read_row(uint32_t addr, float (&u)[W], float (&v)[W]) {
  constexpr uint32_t kPlane = W / 4 * 32 * 16;
#pragma unroll
  for (int c = 0; c < W / 4; ++c) {
    lds_v4(addr + c * 512, u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3]);
    lds_v4(addr + c * 512 + kPlane, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
}

// One row of one step: left/right by shuffles (the warp is the whole row, so
// lane 31's right neighbour is lane 0: the torus column wrap).
template <int W, int kArith>
__device__ __forceinline__ void cluster_row(const float (&uu)[W], const float (&vu)[W], const float (&uc)[W],
                                            const float (&vc)[W], const float (&ud)[W], const float (&vd)[W],
                                            float (&un)[W], float (&vn)[W], const ParamsT<float>& p,
                                            float neg_eps, int lane_l, int lane_r) {
  const float ul = __shfl_sync(kFull, uc[W - 1], lane_l);
  const float ur = __shfl_sync(kFull, uc[0], lane_r);
  const float vl = __shfl_sync(kFull, vc[W - 1], lane_l);
  const float vr = __shfl_sync(kFull, vc[0], lane_r);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const float u_l = k > 0 ? uc[k - 1] : ul;
    const float u_r = k < W - 1 ? uc[k + 1] : ur;
    const float v_l = k > 0 ? vc[k - 1] : vl;
    const float v_r = k < W - 1 ? vc[k + 1] : vr;
    fhn_cell<float, kArith>(uc[k], vc[k], u_r, u_l, ud[k], uu[k], v_r, v_l, vd[k], vu[k], p, neg_eps, un[k],
                           vn[k]);
  }
}

// Strict cell update (fhn_cell) split at the exchange wait: the part that
// needs only the warp's own rows -- the row's left/right sum, plus the row
// below when it is the warp's own, and both reaction terms -- runs before
// the wait; the rest after it.  Same operations in the same order
// (kernels.hpp:63-72, model.hpp:37-56), so bit-identical to fhn_cell.
struct EdgePre {
  float su, sv, f1, f2, m4v;  // m4v = RN(4 * vc) of the v Laplacian's tail
};

template <bool kDnOwn, int kArith>
__device__ __forceinline__ void cell_pre(float uc, float vc, float ur, float ul, float vr, float vl, float ud,
                                         float vd, const ParamsT<float>& p, float neg_eps, EdgePre& e) {
  e.su = add_rn(ur, ul);
  e.sv = add_rn(vr, vl);
  if constexpr (kDnOwn) {
    e.su = add_rn(e.su, ud);
    e.sv = add_rn(e.sv, vd);
  }
  const float uu3 = kArith >= kStrictDiv2 ? div3_rn2(mul_rn(uc, uc)) : div3_rn(mul_rn(uc, uc));
  e.f1 = sub_rn(mul_rn(uc, sub_rn(p.c, uu3)), vc);
  e.f2 = mul_rn(neg_eps, add_rn(sub_rn(uc, mul_rn(p.b, vc)), p.a));
  e.m4v = mul_rn(4.0f, vc);
}

template <bool kDnOwn, int kArith>
__device__ __forceinline__ void cell_post(float uc, float vc, float ud, float vd, float uu, float vu,
                                          const EdgePre& e, const ParamsT<float>& p, float& un, float& vn) {
  float su = e.su, sv = e.sv;
  if constexpr (!kDnOwn) {
    su = add_rn(su, ud);
    sv = add_rn(sv, vd);
  }
  const float lap_u = fma_rn(-4.0f, uc, add_rn(su, uu));  // as fhn_cell: exact when 4*uc is finite
  const float lap_v = sub_rn(add_rn(sv, vu), e.m4v);
  un = add_rn(uc, mul_rn(p.dt, add_rn(e.f1, mul_rn(p.du, lap_u))));
  const float dv_lap = kArith == kStrictDiv2U ? lap_v : mul_rn(p.dv, lap_v);  // as fhn_cell
  vn = add_rn(vc, mul_rn(p.dt, add_rn(e.f2, dv_lap)));
}

// Pre-wait half of one edge row: left/right by shuffles, as cluster_row.
template <int W, bool kDnOwn, int kArith>
__device__ __forceinline__ void edge_pre(const float (&uc)[W], const float (&vc)[W], const float (&ud)[W],
                                         const float (&vd)[W], EdgePre (&e)[W], const ParamsT<float>& p,
                                         float neg_eps, int lane_l, int lane_r) {
  const float ul = __shfl_sync(kFull, uc[W - 1], lane_l);
  const float ur = __shfl_sync(kFull, uc[0], lane_r);
  const float vl = __shfl_sync(kFull, vc[W - 1], lane_l);
  const float vr = __shfl_sync(kFull, vc[0], lane_r);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    cell_pre<kDnOwn, kArith>(uc[k], vc[k], k < W - 1 ? uc[k + 1] : ur, k > 0 ? uc[k - 1] : ul, k < W - 1 ? vc[k + 1] : vr,
                     k > 0 ? vc[k - 1] : vl, ud[k], vd[k], p, neg_eps, e[k]);
  }
}

// W columns per lane, RW consecutive rows per warp, R = warps * RW rows per CTA.
template <int RW>
struct ClusterThreads {  // launch bound: 4-row warps keep ~200 registers
  static constexpr int value = RW >= 4 ? 256 : 512;
};

// kArith: kStrictArith, kFastArith or kStrictDiv2U (the host maps
// kStrictDiv2 to kStrictArith here: both are exact; fewer instances).
template <int W, int RW, int kArith>
__global__ void __launch_bounds__(ClusterThreads<RW>::value, 1) fhn_cluster_kernel(const ClusterArgs a) {
  static_assert(W % 4 == 0, "W must be a multiple of 4 (float4 chunks)");
  constexpr uint32_t kRow = 2 * (W / 4) * 32 * 16;  // bytes of one exchange row (u, v)
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const unsigned crank = cluster_ctarank();
  const unsigned C = cluster_nctarank();
  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const int nw = int(blockDim.x >> 5);
  const int R = a.R;  // = nw * RW
  const int grow0 = int(crank) * R + warp * RW;  // this warp's first lattice row
  const ParamsT<float> p = a.p;
  const float neg_eps = -p.eps;  // model.hpp:45 negates eps first
  const int lane_l = (lane + 31) & 31, lane_r = (lane + 1) & 31;

  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t lbar = base;         // two mbarriers (step parity): the CTA's own rows are in
  const uint32_t mbar = base + 16;    // two mbarriers (step parity): both halo rows landed
  const uint32_t X = base + 32;       // exchange rows, local row i at X + i*kRow
  const uint32_t par_bytes = (uint32_t)(R + 2) * kRow;
  const uint32_t lane_off = (uint32_t)lane * 16;
  const uint32_t my_first = X + (uint32_t)(1 + warp * RW) * kRow + lane_off;
  const uint32_t my_last = my_first + (uint32_t)(RW - 1) * kRow;
  const uint32_t above = my_first - kRow;  // the previous warp's last row (or the top halo)
  const uint32_t below = my_last + kRow;   // the next warp's first row (or the bottom halo)
  // Ring: the CTA's first row -> prev CTA's bottom halo (row R+1); its last
  // row -> next CTA's top halo (row 0); each counted on the receiver's mbarrier.
  const unsigned prev = (crank + C - 1) % C, next = (crank + 1) % C;
  const uint32_t to_prev = mapa_shared(X + (uint32_t)(R + 1) * kRow + lane_off, prev);
  const uint32_t to_next = mapa_shared(X + lane_off, next);
  const uint32_t mbar_prev = mapa_shared(mbar, prev), mbar_next = mapa_shared(mbar, next);
  const bool cta_first = warp == 0, cta_last = warp == nw - 1;

  float u[RW][W], v[RW][W];
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const size_t off = (size_t)(grow0 + r) * a.cols + (size_t)lane * W;
#pragma unroll
    for (int k = 0; k < W; k += 4) {
      const float4 x = *reinterpret_cast<const float4*>(a.u_in + off + k);
      const float4 y = *reinterpret_cast<const float4*>(a.v_in + off + k);
      u[r][k] = x.x; u[r][k + 1] = x.y; u[r][k + 2] = x.z; u[r][k + 3] = x.w;
      v[r][k] = y.x; v[r][k + 1] = y.y; v[r][k + 2] = y.z; v[r][k + 3] = y.w;
    }
  }
  // Per parity: lbar completes when all 32*nw threads of this CTA have
  // published (arrive, release); mbar when both halo rows' bytes have landed
  // (complete_tx from the ring neighbours' st.async; armed by thread 0).
  if (threadIdx.x == 0) {
    mbar_init(lbar, (unsigned)(32 * nw));  // every thread releases its own exchange-row stores
    mbar_init(lbar + 8, (unsigned)(32 * nw));
    mbar_init(mbar, 1);
    mbar_init(mbar + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cluster_barrier();  // mbarriers ready in every CTA before any DSMEM store

  // Dataflow, no per-step cluster barrier: a CTA waits only for its own warps
  // and its two ring neighbours.  Write-after-read safety with one step of
  // slack: the rows of parity p are rewritten at step n+2 only by a writer
  // that has waited at step n+1 for data its readers publish after finishing
  // step n (siblings: all 32*nw arrivals; a neighbour: this CTA's edge row,
  // published by the very warp that read the halo).
  Finite<float> fin;
  bool flagged = false;
  for (long long done = 0; done < a.steps; ++done) {
    const uint32_t par = (uint32_t)(done & 1) * par_bytes;
    const uint32_t pb = (uint32_t)(done & 1) * 8u;
    const uint32_t lb = lbar + pb, mb = mbar + pb;  // this step's barriers
    // 1. publish the warp's edge rows (the CTA's edge rows to the ring neighbours)
    publish_row<W>(my_first + par, u[0], v[0]);
    if (RW > 1) publish_row<W>(my_last + par, u[RW - 1], v[RW - 1]);
    if (cta_first) publish_row_remote<W>(to_prev + par, u[0], v[0], mbar_prev + (mb - mbar));
    if (cta_last) publish_row_remote<W>(to_next + par, u[RW - 1], v[RW - 1], mbar_next + (mb - mbar));
    // Every thread arrives (release) after its own stores, so each reader's
    // acquire-wait orders exactly the stores it reads -- no reliance on a
    // warp barrier's cumulativity.
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(lb) : "memory");
    if (warp == 0 && lane == 0) mbar_arrive_expect_tx(mb, 2u * kRow);  // arms the two halo rows' bytes
    // 2. interior rows need only this warp's registers: overlap the wait
    float un[RW][W], vn[RW][W];
#pragma unroll
    for (int r = 1; r < RW - 1; ++r)
      cluster_row<W, kArith>(u[r - 1], v[r - 1], u[r], v[r], u[r + 1], v[r + 1], un[r], vn[r], p, neg_eps, lane_l,
                            lane_r);
    // Their finiteness folds before the wait too: after it only the edge
    // rows' work is on the step's critical path (the neighbours wait for
    // those rows).  (Deferring the edge rows' fold to the next step's
    // pre-wait phase measured 2 % slower: profiles/README.md.)
#pragma unroll
    for (int r = 1; r < RW - 1; ++r)
#pragma unroll
      for (int k = 0; k < W; ++k) fin.add(un[r][k], vn[r][k]);
    const unsigned phase = (unsigned)((done >> 1) & 1);
    // 2b. strict mode: the edge rows' own-row half before the wait
    EdgePre e_top[W], e_bot[W];
    if constexpr (kArith != kFastArith) {
      if constexpr (RW == 1) {
        edge_pre<W, false, kArith>(u[0], v[0], u[0], v[0], e_top, p, neg_eps, lane_l, lane_r);
      } else {
        edge_pre<W, true, kArith>(u[0], v[0], u[1], v[1], e_top, p, neg_eps, lane_l, lane_r);
        edge_pre<W, false, kArith>(u[RW - 1], v[RW - 1], u[RW - 1], v[RW - 1], e_bot, p, neg_eps, lane_l, lane_r);
      }
    }
    mbar_wait_parity_cta(lb, phase);
    if (cta_first || cta_last) mbar_wait_parity(mb, phase);
    // 3. edge rows with the neighbours' rows from shared memory
    if constexpr (kArith != kFastArith) {
      float ua[W], va[W], ub[W], vb[W];
      read_row<W>(above + par, ua, va);
      read_row<W>(below + par, ub, vb);
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if constexpr (RW == 1) {
          cell_post<false, kArith>(u[0][k], v[0][k], ub[k], vb[k], ua[k], va[k], e_top[k], p, un[0][k], vn[0][k]);
        } else {
          cell_post<true, kArith>(u[0][k], v[0][k], 0.0f, 0.0f, ua[k], va[k], e_top[k], p, un[0][k], vn[0][k]);
          cell_post<false, kArith>(u[RW - 1][k], v[RW - 1][k], ub[k], vb[k], u[RW - 2][k], v[RW - 2][k], e_bot[k], p,
                           un[RW - 1][k], vn[RW - 1][k]);
        }
      }
    } else {
      float ua[W], va[W], ub[W], vb[W];
      read_row<W>(above + par, ua, va);
      read_row<W>(below + par, ub, vb);
      if constexpr (RW == 1) {
        cluster_row<W, kArith>(ua, va, u[0], v[0], ub, vb, un[0], vn[0], p, neg_eps, lane_l, lane_r);
      } else {
        cluster_row<W, kArith>(ua, va, u[0], v[0], u[1], v[1], un[0], vn[0], p, neg_eps, lane_l, lane_r);
        cluster_row<W, kArith>(u[RW - 2], v[RW - 2], u[RW - 1], v[RW - 1], ub, vb, un[RW - 1], vn[RW - 1], p,
                              neg_eps, lane_l, lane_r);
      }
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      fin.add(un[0][k], vn[0][k]);
      if (RW > 1) fin.add(un[RW - 1][k], vn[RW - 1][k]);
    }
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int k = 0; k < W; ++k) {
        u[r][k] = un[r][k];
        v[r][k] = vn[r][k];
      }
    // Blow-up: record the first step whose output went non-finite (exact per
    // lane; the minimum over lanes and warps is the lattice's).  Each lane
    // tests its own running fold (no warp reduction on the step's critical
    // path).  The run continues -- stopping would need every CTA to agree on
    // the step -- and the host re-runs exactly that many steps from the
    // untouched input.
    if (!flagged && __float_as_uint(fin.m) >= 0x7F800000u) {
      flagged = true;
      atomicMin(reinterpret_cast<unsigned long long*>(a.first_bad), (unsigned long long)(done + 1));
    }
  }
  cluster_barrier();
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const size_t off = (size_t)(grow0 + r) * a.cols + (size_t)lane * W;
#pragma unroll
    for (int k = 0; k < W; k += 4) {
      *reinterpret_cast<float4*>(a.u_out + off + k) = make_float4(u[r][k], u[r][k + 1], u[r][k + 2], u[r][k + 3]);
      *reinterpret_cast<float4*>(a.v_out + off + k) = make_float4(v[r][k], v[r][k + 1], v[r][k + 2], v[r][k + 3]);
    }
  }
  // No CTA exits while a peer could still store into its shared memory: the
  // last DSMEM stores precede the barrier above.
}

}  // namespace rdcnn_dev
