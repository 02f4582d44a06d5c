// fhn_rowring.cuh -- the K-level wavefront with NO halo lanes: one thread-
// block cluster covers a whole torus row.
//
// The wavefront kernel (fhn_stencil.cuh) gives every warp its own 32-lane
// column band; the outermost lane on each side is halo (its columns go stale
// one per level and are recomputed by the neighbouring band), so a 4096-wide
// torus needs 35 bands x 32 lanes for 1024 column groups: 9.4 % of all FP32
// work is recomputation.  Here the bands are joined instead:
//
//   * a cluster of C CTAs x M warps x 32 lanes x 4 columns spans exactly one
//     torus row (cols == 128*M*C), so every lane owns useful columns;
//   * all warps of the cluster share one row segment and march down it in
//     the same skewed wavefront (same tick sequence);
//   * level-0 rows are staged by cp.async into a CTA-wide row buffer (the
//     CTA's 32*M column groups plus one pad entry each side, filled with the
//     ring neighbours' edge columns), so every lane reads its left/right
//     level-0 neighbours from shared memory;
//   * levels 1..K-1: every lane publishes the first and last column (u, v)
//     of each row it produces as one STS.128 into that row's edge slot and
//     reads its neighbours' 8-byte halves when that row is the center row of
//     the level above (two ticks later): one STS.128 + two LDS.64 replace
//     the four SHFLs per row of the wavefront kernel, and warp boundaries
//     cost nothing extra;
//   * once per tick the CTA's first/last lane sends its edge entries (and
//     the next staged row's two edge values) into the ring neighbour CTA's
//     pad entries by st.async, counting the bytes on the receiver's mbarrier
//     (complete_tx): DSMEM over the cluster, no fences; the ring wraps the
//     torus column edge (a one-CTA ring writes its own pads directly);
//   * one mbarrier per tick slot (ring of 3: slot = tick % 3, a compile-time
//     offset in the 3-unrolled tick loop) completes when all 32*M threads of
//     the CTA have arrived (release: after this tick's stores, reads and the
//     cp.async wait for the NEXT level-0 row) and the neighbours' edge bytes
//     have landed.  Tick j waits on the barrier of tick j-2 before its first
//     read (the rows it reads as centers were produced at j-2 / staged by
//     j-2) and on that of tick j-1 before its first store (slot j%3 was last
//     read at tick j-1).  No CTA- or cluster-wide barrier runs in the loop.
//
// Arithmetic is fhn_cell, unchanged, so results are bit-identical to the
// wavefront kernel (and the reference) in strict and fast mode alike.
//
// MEASURED AND REJECTED (profiles/README.md, round 2): bit-exact at every
// shape and M tried, but slower than the wavefront kernel -- 4096^2 744k vs
// 894k, 8192^2 739k vs 955k Mcell-updates/s (M=16, C=2).  ncu: issue active
// 75 % vs 90 % (the 16 coupled warps of an SM idle together whenever the
// slowest one waits: ~10 % of stall samples sit in the mbarrier loops),
// 43x the shared-memory bank conflicts (the 4-byte neighbour reads), and
// ~8 % more instructions per computed cell than the shuffle-based wavefront
// -- more than the 9.4 % of halo work it removes.  A 4-slot ring (one wait
// per tick, two ticks of slack) was slower still (726k).  Kept behind
// RDCNN_ROWRING=1 (off by default) as the measured alternative.
#pragma once

#include "fhn_cluster.cuh"
#include "fhn_stencil.cuh"

namespace rdcnn_dev {

// Edge / barrier slots: 3 (slot = tick % 3, a compile-time offset; stores
// wait for the barrier of tick j-1) or 4 (slot = tick % 4 from uniform
// registers; one wait per tick, on tick j-2: two ticks of slack).
#ifndef RDCNN_RR_SLOTS
#define RDCNN_RR_SLOTS 3
#endif
constexpr int kRrTickSlots = RDCNN_RR_SLOTS;

// Level-0 rows: kept in a 3-row register ring (1) or re-read from the staged
// rows each tick (0: 24 fewer registers, four more LDS.128 per tick).
#ifndef RDCNN_RR_L0REG
#define RDCNN_RR_L0REG 0
#endif

// Shared memory of one row-ring CTA of M warps at K levels: 3 mbarriers,
// the edge slots, the level-0 staging ring.
__host__ __device__ constexpr int rowring_row_bytes(int M) { return (32 * M + 2) * 16; }
__host__ __device__ constexpr int rowring_smem_bytes(int M, int K) {
  return 64 + kRrTickSlots * (K - 1) * rowring_row_bytes(M) + kStage * 2 * rowring_row_bytes(M);
}

__device__ __forceinline__ void sts_v4u(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void lds_v2(uint32_t addr, float& a, float& b) {
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(a), "=f"(b) : "r"(addr) : "memory");
}
// Every thread arrives; `bytes` (non-zero in one thread) is the tick's
// expected DSMEM transaction count.
__device__ __forceinline__ void mbar_arrive_tx(uint32_t mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void stas_v4(uint32_t addr, const Row<4, float>& r, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];\n"
               ::"r"(addr), "f"(r.u[0]), "f"(r.v[0]), "f"(r.u[3]), "f"(r.v[3]), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void sts_row_edges(uint32_t addr, const Row<4, float>& r) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "f"(r.u[0]), "f"(r.v[0]), "f"(r.u[3]),
               "f"(r.v[3])
               : "memory");
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float x) {
  asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(addr), "f"(x) : "memory");
}
__device__ __forceinline__ void stas_f32(uint32_t addr, float x, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(addr),
               "r"(__float_as_uint(x)), "r"(mbar)
               : "memory");
}
// Phase wait, CTA-scope acquire (the barrier and every byte it covers live
// in this CTA's shared memory; no L1 invalidation).
__device__ __forceinline__ void mbar_wait_cta(uint32_t mbar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAITR_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAITR_%=;\n"
      "}\n" ::"r"(mbar), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void lds_v4f(uint32_t addr, float (&x)[4]) {
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]) : "r"(addr)
               : "memory");
}

// One level of one row with the center row's outer neighbours given.
template <int kArith>
__device__ __forceinline__ void level_row_nb(const Row<4, float>& up, const Row<4, float>& c,
                                             const Row<4, float>& dn, Row<4, float>& out, const Params& p,
                                             float neg_eps, float ul, float vl, float ur, float vr) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float u_l = k > 0 ? c.u[k - 1] : ul;
    const float u_r = k < 3 ? c.u[k + 1] : ur;
    const float v_l = k > 0 ? c.v[k - 1] : vl;
    const float v_r = k < 3 ? c.v[k + 1] : vr;
    fhn_cell<float, kArith>(c.u[k], c.v[k], u_r, u_l, dn.u[k], up.u[k], v_r, v_l, dn.v[k], up.v[k], p, neg_eps,
                            out.u[k], out.v[k]);
  }
}

// a.n_bands = C (CTAs per ring), a.n_segs = segments per grid; the grid is
// n_segs x batch clusters of C CTAs (cluster dims (C,1,1)).
template <int K, int M, int kArith, bool kPerGrid>
__global__ void __launch_bounds__(32 * M, 16 / M) fhn_rowring_kernel(const StepArgsT<float> a) {
  static_assert(K >= 2 && K <= 4, "row-ring instances: K in {2, 4}");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr uint32_t kRow = (uint32_t)rowring_row_bytes(M);  // one plane of one CTA row (+2 pads)
  constexpr uint32_t kEdgeTick = (K - 1) * kRow;              // edge entries of one tick slot
  constexpr uint32_t kSlot = 2 * kRow;                        // one staged level-0 row (u, v)
  const int lane = threadIdx.x & 31;
  const int li = int(threadIdx.x);  // lane index within the CTA row
  const int C = a.n_bands;
  const unsigned rank = cluster_ctarank();
  const int cid = int(blockIdx.x) / C;
  const int g = cid / a.n_segs;
  const int seg = cid - g * a.n_segs;

  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t mbar0 = sbase;
  const uint32_t ebase = sbase + 64;
  const uint32_t sring = ebase + kRrTickSlots * kEdgeTick;
  // This lane's entry (index li + 1; pads 0 and 32M+1) in edge and staging rows.
  const uint32_t e_own = ebase + 16u * (uint32_t)(li + 1);
  const uint32_t s_own = 16u * (uint32_t)(li + 1);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < kRrTickSlots; ++q) mbar_init(mbar0 + 8u * q, 32u * M);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // Every CTA's barriers are initialised before any ring neighbour sends.
  cluster_barrier();

  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const unsigned fl = a.flags != nullptr ? *(volatile unsigned*)(a.flags + g) : 0u;
  const bool frozen = fl != 0u && fl != a.tag;

  const Params p = kPerGrid ? a.params[g] : a.shared;
  const float neg_eps = -p.eps;

  const int L = (int)rank * (32 * M) + li;  // this lane's column group
  const size_t goff = (size_t)g * (size_t)a.grid_stride + (size_t)L * 4;
  const float* __restrict__ uin = a.u_in + goff;
  const ptrdiff_t vdelta = a.v_in - a.u_in;
  float* __restrict__ uout = a.u_out + goff;
  const ptrdiff_t vout_delta = a.v_out - a.u_out;
  const size_t pitch = (size_t)a.pitch;

  // CTA-edge lanes.  Once per tick the CTA's first lane sends its edge
  // entries (levels 1..K-1) to the left CTA's pad 32M+1 -- read there as
  // (u0, v0) -- and the last lane sends its to the right CTA's pad 0 -- read
  // as (u3, v3); both also send the matching two level-0 values of the next
  // staged row into the neighbour's staging pad.  Remote addresses are the
  // local ones plus the neighbour's shared::cluster window offset.
  const bool first_lane = li == 0;
  const bool last_lane = li == 32 * M - 1;
  const bool halo_lane = first_lane || last_lane;
  const unsigned nb = first_lane ? (rank == 0 ? (unsigned)C - 1 : rank - 1)
                                 : (rank + 1 == (unsigned)C ? 0u : rank + 1);
  const uint32_t rem = mapa_shared(sbase, nb) - sbase;
  const uint32_t e_pad = first_lane ? 16u * (uint32_t)(32 * M + 1) : 0u;  // target entry (edge and staging rows)
  const uint32_t v_off = first_lane ? 0u : 12u;                           // (u0, v0) or (u3, v3)

  const int r0 = a.row_begin + seg * a.seg_rows;
  const int h = min(a.seg_rows, a.row_end - r0);
  const int n_load = h + 2 * K;
  const int nt = h + 3 * K - 1;

  const int r_first = wrap_index(r0 - K, a.rows);
  const float* su = uin + (size_t)r_first * pitch;
  int rows_left = a.rows - r_first;
  const size_t span = (size_t)a.rows * pitch;
  auto src_next = [&]() {
    su = reinterpret_cast<const float*>(reinterpret_cast<const char*>(su) + a.pitch_b);
    if (__builtin_expect(--rows_left == 0, 0)) {
      su -= span;
      rows_left = a.rows;
    }
  };
  float* du = uout + (size_t)r0 * pitch;

  auto stage = [&](uint32_t slot) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(slot + s_own), "l"(su) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(slot + kRow + s_own), "l"(su + vdelta)
                 : "memory");
  };

#pragma unroll
  for (int d = 0; d < kPrefetch; ++d) {
    if (d < n_load) {
      stage(sring + d * kSlot);
      src_next();
    }
    stage_commit();
  }

  Row<4, float> win[K - 1][3];
#if RDCNN_RR_L0REG
  Row<4, float> l0[3];
#endif
  Finite<float> fin;
  const bool store = !frozen;
  uint32_t half_now = sring, half_other = sring + 3 * kSlot;
  unsigned par = 0;  // phase parity of the current 3-tick group's barriers

  auto tick = [&](auto ph_c, int j) {
    constexpr int ph = decltype(ph_c)::value;
#if RDCNN_RR_SLOTS == 3
    constexpr uint32_t kW = ph * kEdgeTick;              // edge slot of tick j (written)
    constexpr uint32_t kR = ((ph + 1) % 3) * kEdgeTick;  // edge slot of tick j-2 (read)
    constexpr uint32_t kMb = 8u * ph;                     // barrier of tick j
    // The barrier of tick j-2 (slot (ph+1)%3; previous group unless ph == 2)
    // and of tick j-1 (slot (ph+2)%3; previous group when ph == 0).
    const unsigned par2 = ph == 2 ? par : par ^ 1u;
    const unsigned par1 = ph >= 1 ? par : par ^ 1u;
    if (j >= 2) mbar_wait_cta(mbar0 + 8u * ((ph + 1) % 3), par2);
#else
    const uint32_t kW = (uint32_t)(j & 3) * kEdgeTick;
    const uint32_t kR = (uint32_t)((j + 2) & 3) * kEdgeTick;
    const uint32_t kMb = 8u * (uint32_t)(j & 3);
    // Tick j-2's barrier: its rows are in, and slot j%4 (last read at j-2) is free.
    if (j >= 2) mbar_wait_cta(mbar0 + 8u * (uint32_t)((j + 2) & 3), (unsigned)(((j - 2) >> 2) & 1));
#endif
    unsigned sends = 0;  // level rows published this tick (levels 1..K-1)
#pragma unroll
    for (int t = K; t >= 2; --t) {
#if RDCNN_RR_SLOTS == 3
      if (t == K - 1 && j >= 1) mbar_wait_cta(mbar0 + 8u * ((ph + 2) % 3), par1);
#endif
      if (j >= 3 * t - 1 && j - (h + 2 * K - 1) < t) {
        const Row<4, float>& up = win[t - 2][ph];
        const Row<4, float>& ce = win[t - 2][(ph + 1) % 3];
        const Row<4, float>& dn = win[t - 2][(ph + 2) % 3];
        const uint32_t ce_e = e_own + kR + (uint32_t)(t - 2) * kRow;
        float ul, vl, ur, vr;
        lds_v2(ce_e - 8u, ul, vl);   // left neighbour's (u3, v3)
        lds_v2(ce_e + 16u, ur, vr);  // right neighbour's (u0, v0)
        if (t < K) {
          Row<4, float>& o = win[t - 1][ph];
          level_row_nb<kArith>(up, ce, dn, o, p, neg_eps, ul, vl, ur, vr);
          sts_v4u(e_own + kW + (uint32_t)(t - 1) * kRow, o.u[0], o.v[0], o.u[3], o.v[3]);
          ++sends;
        } else {
          Row<4, float> o;
          level_row_nb<kArith>(up, ce, dn, o, p, neg_eps, ul, vl, ur, vr);
          fold_finite<4, float>(fin, o);
          if (store) store_row<4, float>(du, du + vout_delta, 0, o);
          du = reinterpret_cast<float*>(reinterpret_cast<char*>(du) + a.pitch_b);
        }
      }
    }
#if RDCNN_RR_SLOTS == 3
    if constexpr (K == 2) {  // no level-1 row above: the store wait comes here
      if (j >= 1) mbar_wait_cta(mbar0 + 8u * ((ph + 2) % 3), par1);
    }
#endif
    // Stage the row of tick j+3 into the slot of tick j-3 (its last readers,
    // the neighbours of tick j-2, are past the barrier waited on above).
    if (j + kPrefetch < n_load) {
      stage(half_other + ph * kSlot);
      src_next();
    }
    stage_commit();
    // Rows up to j+1 landed (this thread's copies); the arrival below
    // publishes row j+1 to the CTA for tick j+2.
    stage_wait<kPrefetch - 1>();
#if RDCNN_RR_L0REG
    if (j < n_load) {
      const uint32_t rs = half_now + ph * kSlot + s_own;
      lds_v4f(rs, l0[ph].u);
      lds_v4f(rs + kRow, l0[ph].v);
    }
#endif
    const bool l1 = j >= 2 && j < n_load;
    if (l1) {
      // Rows of ticks j-2 (up), j-1 (center), j (down) and the center's
      // outer neighbours.
      const uint32_t cs = (ph >= 1 ? half_now + (ph - 1) * kSlot : half_other + 2 * kSlot) + s_own;
      float ul, vl, ur, vr;
      lds(cs - 4u, ul);
      lds(cs + kRow - 4u, vl);
      lds(cs + 16u, ur);
      lds(cs + kRow + 16u, vr);
      Row<4, float>& o = win[0][ph];
#if RDCNN_RR_L0REG
      level_row_nb<kArith>(l0[(ph + 1) % 3], l0[(ph + 2) % 3], l0[ph], o, p, neg_eps, ul, vl, ur, vr);
#else
      Row<4, float> up0, ce0, dn0;
      const uint32_t us = (ph >= 2 ? half_now + (ph - 2) * kSlot : half_other + (ph + 1) * kSlot) + s_own;
      const uint32_t ds = half_now + ph * kSlot + s_own;
      lds_v4f(us, up0.u);
      lds_v4f(us + kRow, up0.v);
      lds_v4f(cs, ce0.u);
      lds_v4f(cs + kRow, ce0.v);
      lds_v4f(ds, dn0.u);
      lds_v4f(ds + kRow, dn0.v);
      level_row_nb<kArith>(up0, ce0, dn0, o, p, neg_eps, ul, vl, ur, vr);
#endif
      sts_v4u(e_own + kW, o.u[0], o.v[0], o.u[3], o.v[3]);
      ++sends;
    }
    // Row j+1's slot (its pads are the neighbours' edge values of tick j).
    const uint32_t nxt = ph <= 1 ? half_now + (ph + 1) * kSlot : half_other;
    const bool s0 = j + 1 < n_load;
    if (halo_lane) {
      // Ring neighbour sends: the level rows produced this tick, then the
      // next staged row's two edge values.  A one-CTA ring (C == 1) wraps
      // onto itself: plain shared stores, released by the arrival below
      // (st.async needs a cluster of at least two CTAs).
      const uint32_t mb = mbar0 + kMb + rem;
      float eu = 0.0f, ev = 0.0f;
      if (s0) {
        lds(nxt + s_own + v_off, eu);
        lds(nxt + kRow + s_own + v_off, ev);
      }
      if (C > 1) {
        if (l1) stas_v4(ebase + kW + rem + e_pad, win[0][ph], mb);
#pragma unroll
        for (int t = 2; t < K; ++t)
          if (j >= 3 * t - 1 && j - (h + 2 * K - 1) < t)
            stas_v4(ebase + kW + (uint32_t)(t - 1) * kRow + rem + e_pad, win[t - 1][ph], mb);
        if (s0) {
          stas_f32(nxt + e_pad + v_off + rem, eu, mb);
          stas_f32(nxt + kRow + e_pad + v_off + rem, ev, mb);
        }
      } else {
        if (l1) sts_row_edges(ebase + kW + e_pad, win[0][ph]);
#pragma unroll
        for (int t = 2; t < K; ++t)
          if (j >= 3 * t - 1 && j - (h + 2 * K - 1) < t)
            sts_row_edges(ebase + kW + (uint32_t)(t - 1) * kRow + e_pad, win[t - 1][ph]);
        if (s0) {
          sts_f32(nxt + e_pad + v_off, eu);
          sts_f32(nxt + kRow + e_pad + v_off, ev);
        }
      }
    }
    // Done with this tick's stores, reads and row j+1's copy: arrive (thread
    // 0 also expects both ring neighbours' bytes for this tick).
    const unsigned tx = C > 1 ? 2u * (16u * sends + (s0 ? 8u : 0u)) : 0u;
    mbar_arrive_tx(mbar0 + kMb, threadIdx.x == 0 ? tx : 0u);
  };

  for (int j0 = 0; j0 < nt; j0 += 3) {
    tick(Int<0>{}, j0);
    if (j0 + 1 < nt) tick(Int<1>{}, j0 + 1);
    if (j0 + 2 < nt) tick(Int<2>{}, j0 + 2);
    const uint32_t t_half = half_now;
    half_now = half_other;
    half_other = t_half;
    par ^= 1u;
  }
  stage_wait<0>();
  // Every byte the neighbours send lands before the CTA exits: wait on the
  // ticks nt-2 and nt-1, never waited on inside the loop.
  for (int j = max(nt - 2, 0); j < nt; ++j)
    mbar_wait_cta(mbar0 + 8u * (uint32_t)(j % kRrTickSlots), (unsigned)((j / kRrTickSlots) & 1));

  if (!store) fin = Finite<float>{};
  const bool bad = fin.bad_in_warp();
  if (bad && lane == 0 && a.flags != nullptr) atomicCAS(a.flags + g, 0u, a.tag);
}

}  // namespace rdcnn_dev
