// fhn_stencil.cuh -- sm_100a register-wavefront stencil for the coupled u/v
// FitzHugh-Nagumo RD-CNN step (reference proj/include/rdcnn/kernels.hpp:63-72,
// model.hpp:37-56), advancing K time levels per launch, in fp32 (default) or
// fp64 (the reference templates instantiate both, grid.hpp:13-28).
//
// Mapping:
//   * one warp owns a column BAND x row SEGMENT of one grid;
//   * each lane owns W consecutive columns (16 bytes per plane: W=4 fp32,
//     W=2 fp64; W=1 when the column count is not a multiple of that);
//   * the warp marches down the segment in a skewed wavefront, keeping three
//     rows per level in registers and staging the level-0 rows through a
//     per-warp shared-memory ring filled by cp.async;
//   * left/right neighbours come from the adjacent lanes by warp shuffle;
//     the outermost `halo_groups` lanes of a band are halo (their values go
//     stale one column per level and are never stored);
//   * rows wrap on the torus by index arithmetic (periodic mode) or read
//     ghost rows written by the halo exchange (slab mode);
//   * only level-K rows are stored; their finiteness is folded into one word
//     per grid (atomicCAS of the launch tag).  Non-finite values are absorbing
//     and spread one cell per level, so a non-finite value at any level of
//     the block implies a non-finite stored value; the host replays the block
//     one level at a time to recover the exact iteration.
//
// Arithmetic: in strict mode each operation is one IEEE round-to-nearest op
// in the reference order (__fadd_rn/__fmul_rn/__dadd_rn/... are never
// contracted), with subnormals preserved (no -ftz).  x/3 uses a three-op
// corrected reciprocal proven equal to IEEE division on the only domain it
// sees (x = u*u), see div3_rn below and oracle/div3_check.c.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rdcnn_dev {

constexpr unsigned kFull = 0xFFFFFFFFu;

// Gene narrowed once to the working precision, kernel order
// {dt,a,b,eps,c,du,dv} (reference model.hpp:24-32, gene.hpp:39-41).
template <class T>
struct ParamsT {
  T dt, a, b, eps, c, du, dv;
};
using Params = ParamsT<float>;

template <class T>
struct StepArgsT {
  const T* u_in;
  const T* v_in;
  T* u_out;
  T* v_out;
  long long grid_stride;  // elements between consecutive grids (same for in/out)
  int rows;               // lattice rows (periodic) or slab rows (ghosted)
  int cols;               // lattice cols (W divides cols)
  int pitch;              // elements between consecutive rows
  long long pitch_b;      // the same in bytes (kernel-param operand of the pointer steps)
  int periodic;           // 1: rows wrap mod rows; 0: ghost rows present
  int ghost;              // ghosted mode: ghost rows above row 0 in the buffer
  int row_begin, row_end; // output rows computed by this launch
  int seg_rows;           // H: output rows per warp segment
  int n_segs;
  int n_bands;
  int band_groups;        // useful W-groups per band
  int halo_groups;        // halo W-groups each side (0 = full-width wrap)
  int batch;
  ParamsT<T> shared;      // the gene when every grid shares one (kernel-param
                          // space: the FP ops read it as constant-bank operands)
  const ParamsT<T>* params;  // per-grid genes (kPerGrid instances only)
  int params_stride;      // 0: one gene for all grids; 1: one per grid
  unsigned* flags;        // per grid: 0 clean, else tag of the first bad launch
  unsigned tag;           // this launch's tag (launch index + 1)
  // Fused peer halo exchange (kPeer instances, slab mode only).
  // The level-0 rows beyond the slab are read straight from the ring
  // neighbours' INPUT buffers (peer memory: CUDA IPC over NVLink, or the same
  // device); the edge warps signal completion with one release store per
  // block and direction.
  const T* peer_top;      // prev rank's owned row rows_prev (one past its last) in its input buffer
  const T* peer_bot;      // next rank's owned row 0 in its input buffer
  unsigned* edge_count;   // [2] this rank's completion counters: top / bottom edge warps
  unsigned* sig_prev;     // prev rank's "bottom ghosts delivered" word
  unsigned* sig_next;     // next rank's "top ghosts delivered" word
  const unsigned* ready;  // [2] this rank's "top / bottom ghosts delivered" words
  unsigned seq;           // block number: this block's ghosts are in when ready[] >= seq
  int n_top, n_bot;       // warps whose segment touches the top / bottom `ghost` rows
  // Checkpoint tee (kTee instances, the first block of a slab advance): the
  // owned level-0 rows this launch reads are also stored here (same layout
  // as u_in), so the advance's input survives for an exact blow-up replay
  // without a separate device copy.
  T* tee_u;
  // Profiling only (rdcnn_sim_trace_launch / rdcnn_ring_trace_block): per
  // warp {start ns, end ns, smid} (trace_stride 3), plus {ns spent waiting
  // for the neighbours' ready words, bytes staged from peer memory}
  // (trace_stride 5, kPeer instances).
  unsigned long long* trace;
  int trace_stride;
  // TMA tensor-map staging (RDCNN_BULK=2 builds): a 3-D map {cols, rows x
  // batch, 2 planes} of this launch's input buffer with a {128, 1, 2} box --
  // one band row of both planes -- built by the host (cuTensorMapEncodeTiled).
  int tma_ok;
  alignas(64) unsigned char tmap[128];
};

// Per-warp profile of one block (kPeer traces).
struct BlockStats {
  unsigned long long wait_ns = 0;
  unsigned long long peer_bytes = 0;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
using StepArgs = StepArgsT<float>;

// ---------------------------------------------------------------------------
// Per-cell arithmetic.
// ---------------------------------------------------------------------------

// RN(x/3) for every x the kernel can present (x = RN(u*u): +0, positive,
// +inf or NaN).  q0 = RN(x*R), e = x - 3*q0 exactly (FMA), q = RN(q0 + e*R).
// fp32: exhaustively verified over all 2^32 inputs (CPU: oracle/div3_check.c;
// GPU: rdcnn_selftest_div3); the single mismatch is x = -0.0, which u*u never
// produces.  fp64: the same argument (the exact quotient's fraction of an ulp
// is 0, 1/3 or 2/3, never within the FMA's 2^-53-ulp error of a midpoint),
// checked on random and boundary patterns by rdcnn_selftest_div3_f64.
// Non-finite x yields a non-finite q, so blow-up is preserved.
__device__ __forceinline__ float div3_rn(float x) {
  const float R = __uint_as_float(0x3EAAAAABu);  // RN(1/3)
  const float q0 = __fmul_rn(x, R);
  const float e = __fmaf_rn(-q0, 3.0f, x);
  return __fmaf_rn(e, R, q0);
}

__device__ __forceinline__ double div3_rn(double x) {
  const double R = __longlong_as_double(0x3FD5555555555555ll);  // RN(1/3)
  const double q0 = __dmul_rn(x, R);
  const double e = __fma_rn(-q0, 3.0, x);
  return __fma_rn(e, R, q0);
}

// Two-op x/3 for strict fp32 under a gene gate (kStrictDiv2):
//   q2 = RN(x*R + RN(x*C)),  C = RN(1/3 - R) = 0xB22AAAAB.
// Exhaustive over all 2^32 patterns (oracle/div3_check.c div3_two_op_sweep):
// q2 == RN(x/3) for every x >= 0 except x in [2^-125, 2^-123] (where x*C is
// subnormal), and there q and q2 are both <= 2^-124.4; q2 is non-finite iff
// x is.  The kernel uses the quotient only in RN(c - x/3) (model.hpp:39):
// for |c| >= 2^-90 both RN(c - q) and RN(c - q2) equal c on that range (half
// an ulp below |c| is >= 2^-115), so f1 is bit-identical for every x.  The
// host selects this instance only when every gene of the launch has
// |c| >= 2^-90 (rdcnn_cuda.cu arith_for); otherwise div3_rn runs.
__device__ __forceinline__ float div3_rn2(float x) {
  const float R = __uint_as_float(0x3EAAAAABu);  // RN(1/3)
  const float C = __uint_as_float(0xB22AAAABu);  // RN(1/3 - R)
  return __fmaf_rn(x, R, __fmul_rn(x, C));
}
__device__ __forceinline__ double div3_rn2(double x) { return div3_rn(x); }

// Arithmetic instances: strict (reference op order, 3-op x/3), fast
// (FMA-contracted, opt-in), strict with the gated 2-op x/3 (fp32 only).
constexpr int kStrictArith = 0;
constexpr int kFastArith = 1;
constexpr int kStrictDiv2 = 2;
// Strict with the gated 2-op x/3 and a unit v diffusion coefficient (every
// gene of the launch has Dv == 1 after narrowing): RN(1 * lap_v) == lap_v for
// every lap_v (finite, +-0, +-inf; NaN stays NaN), so the Dv*lap_v product of
// model.hpp:55 is the identity and is skipped.  The reference's default gene
// (gene.hpp:19) and every BASELINE workload have Dv = 1.
constexpr int kStrictDiv2U = 3;
// kStrictDiv2U with the v Laplacian's tail fused as on the u plane:
// RN(s - RN(4*vc)) == fma(-4, vc, s) whenever 4*vc is finite, i.e. |vc| <
// 2^126.  For |vc| >= 2^126 the reference's v+ is non-finite at that step
// for EVERY gene (RN(4*vc) = +-inf; Dv*lap_v, f2 + ., dt*., vc + . stay
// non-finite, dt = 0 included: 0*inf = NaN), while the fused form may stay
// finite.  So this instance also folds the magnitude of every level's centre
// v (the value that gets multiplied by 4) and flags the launch when one
// reaches 2^126.  A flag then means exactly what it means for the other
// instances: the reference blows up inside this block (at the first level
// whose centre v is that large, or earlier) -- and without such a centre the
// fused form computes the reference's values bit for bit, so the flag is
// raised iff the reference blows up within the block.  The host's level
// replay (K = 1 launches of this same instance) therefore finds the exact
// iteration unchanged.  Periodic handles only.
constexpr int kStrictDiv2UF = 4;

// Round-to-nearest primitives that the compiler never contracts.
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

// kern::stencil_cell (kernels.hpp:63-72) with reaction_u/v (model.hpp:37-46):
//   lap   = right + left + down + up - 4*c          (down = row i+1)
//   u+    = u + dt*( u*(c - u*u/3) - v + Du*lap_u )
//   v+    = v + dt*( -eps*(u - b*v + a) + Dv*lap_v )
template <class T, int kArith>
__device__ __forceinline__ void fhn_cell(T uc, T vc, T ur, T ul, T ud, T uu, T vr, T vl, T vd,
                                         T vu, const ParamsT<T>& p, T neg_eps, T& un, T& vn) {
  if constexpr (kArith != kFastArith) {
    // RN(s - RN(4*uc)) == RN(s - 4*uc) == fma(-4, uc, s) whenever 4*uc is
    // finite (scaling by 4 is exact).  When 4*uc overflows, |uc| is so large
    // that uc*uc overflows and u+ is non-finite in both forms:
    // the fused form is bit-identical on every finite outcome.  The v plane
    // has no such guard and keeps the separate multiply.
    const T lap_u = fma_rn(T(-4), uc, add_rn(add_rn(add_rn(ur, ul), ud), uu));
    const T lap_v = kArith == kStrictDiv2UF ? fma_rn(T(-4), vc, add_rn(add_rn(add_rn(vr, vl), vd), vu))
                                            : sub_rn(add_rn(add_rn(add_rn(vr, vl), vd), vu), mul_rn(T(4), vc));
    const T uu3 = kArith >= kStrictDiv2 ? div3_rn2(mul_rn(uc, uc)) : div3_rn(mul_rn(uc, uc));
    const T f1 = sub_rn(mul_rn(uc, sub_rn(p.c, uu3)), vc);
    const T f2 = mul_rn(neg_eps, add_rn(sub_rn(uc, mul_rn(p.b, vc)), p.a));
    un = add_rn(uc, mul_rn(p.dt, add_rn(f1, mul_rn(p.du, lap_u))));
    const T dv_lap = kArith >= kStrictDiv2U ? lap_v : mul_rn(p.dv, lap_v);
    vn = add_rn(vc, mul_rn(p.dt, add_rn(f2, dv_lap)));
  } else {
    // Opt-in fast mode: same formula, FMA-contracted and reassociated.
    // Validated statistically, never bit-exact.
    const T lap_u = fma_rn(T(-4), uc, (ur + ul) + (ud + uu));
    const T lap_v = fma_rn(T(-4), vc, (vr + vl) + (vd + vu));
    const T f1 = fma_rn(uc, fma_rn(-uc * uc, T(1) / T(3), p.c), -vc);
    const T f2 = neg_eps * (fma_rn(-p.b, vc, uc) + p.a);
    un = fma_rn(p.dt, fma_rn(p.du, lap_u, f1), uc);
    vn = fma_rn(p.dt, fma_rn(p.dv, lap_v, f2), vc);
  }
}

template <int W, class T>
struct Row {
  T u[W];
  T v[W];
};

// Running "largest |value|" that turns non-finite once any value is inf/NaN
// (reference grid.hpp:58-67 finite_bits).  fp32: sm_100 three-input
// FMNMX3.NAN with |.| operand modifiers, one ALU op per two values.  fp64:
// the high words' magnitudes in an integer max.
template <class T>
struct Finite;

template <>
struct Finite<float> {
  float m = 0.0f;
  __device__ __forceinline__ void add(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(m), "f"(fabsf(a)), "f"(fabsf(b)));
    m = r;
  }
  // m >= 0, so its bit pattern orders like its value; NaN and +inf are the
  // only patterns >= 0x7F800000.
  __device__ __forceinline__ bool bad_in_warp() const {
    return __reduce_max_sync(kFull, __float_as_uint(m)) >= 0x7F800000u;
  }
};

template <>
struct Finite<double> {
  unsigned m = 0u;
  __device__ __forceinline__ void add(double a, double b) {
    m = max(m, max((unsigned)__double2hiint(a) & 0x7FFFFFFFu, (unsigned)__double2hiint(b) & 0x7FFFFFFFu));
  }
  __device__ __forceinline__ bool bad_in_warp() const {
    return __reduce_max_sync(kFull, m) >= 0x7FF00000u;
  }
};

template <int W, class T>
__device__ __forceinline__ void fold_finite(Finite<T>& f, const Row<W, T>& r) {
#pragma unroll
  for (int k = 0; k < W; ++k) f.add(r.u[k], r.v[k]);
}

// kStrictDiv2UF: the largest |v| among a level's centre cells (fp32 only).
template <int W, class T, int kArith>
__device__ __forceinline__ void fold_centre_v(Finite<T>& f, const Row<W, T>& c) {
  if constexpr (kArith == kStrictDiv2UF) {
#pragma unroll
    for (int k = 0; k + 1 < W; k += 2) f.add(c.v[k], c.v[k + 1]);
    if constexpr (W % 2 == 1) f.add(c.v[W - 1], c.v[W - 1]);
  }
}
// Any |v| >= 2^126 (or non-finite) among the folded centres of the warp.
__device__ __forceinline__ bool big_centre_in_warp(const Finite<float>& f) {
  return __reduce_max_sync(kFull, __float_as_uint(f.m)) >= 0x7E800000u;
}

// 16-byte vector store when a lane's group is 16 bytes, else scalar stores.
template <int W, class T>
__device__ __forceinline__ void store_row(T* __restrict__ u, T* __restrict__ v, size_t off,
                                          const Row<W, T>& r) {
  if constexpr (W * sizeof(T) % 16 == 0 && sizeof(T) == 4) {
#pragma unroll
    for (int c = 0; c < W; c += 4) {
      __stcs(reinterpret_cast<float4*>(u + off + c), make_float4(r.u[c], r.u[c + 1], r.u[c + 2], r.u[c + 3]));
      __stcs(reinterpret_cast<float4*>(v + off + c), make_float4(r.v[c], r.v[c + 1], r.v[c + 2], r.v[c + 3]));
    }
  } else if constexpr (W * sizeof(T) == 16 && sizeof(T) == 8) {
    __stcs(reinterpret_cast<double2*>(u + off), make_double2(r.u[0], r.u[1]));
    __stcs(reinterpret_cast<double2*>(v + off), make_double2(r.v[0], r.v[1]));
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      u[off + k] = r.u[k];
      v[off + k] = r.v[k];
    }
  }
}

// One level of one row: out = step(center) given the rows above/below.
// kWrap: the band is the whole row (no halo lanes), so lane 0's left
// neighbour is lane 31 (indexed shuffles with wrap).  Otherwise lanes 0 and
// 31 are halo lanes whose outer values are stale anyway, and shfl.up/down
// with an immediate delta need no lane-index registers.
template <int W, class T, int kArith, bool kWrap>
__device__ __forceinline__ void level_row(const Row<W, T>& up, const Row<W, T>& c,
                                          const Row<W, T>& dn, Row<W, T>& out,
                                          const ParamsT<T>& p, T neg_eps, int lane_l,
                                          int lane_r) {
  T ul, ur, vl, vr;
  if constexpr (kWrap) {
    ul = __shfl_sync(kFull, c.u[W - 1], lane_l);
    ur = __shfl_sync(kFull, c.u[0], lane_r);
    vl = __shfl_sync(kFull, c.v[W - 1], lane_l);
    vr = __shfl_sync(kFull, c.v[0], lane_r);
  } else {
    ul = __shfl_up_sync(kFull, c.u[W - 1], 1);
    ur = __shfl_down_sync(kFull, c.u[0], 1);
    vl = __shfl_up_sync(kFull, c.v[W - 1], 1);
    vr = __shfl_down_sync(kFull, c.v[0], 1);
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const T u_l = k > 0 ? c.u[k - 1] : ul;
    const T u_r = k < W - 1 ? c.u[k + 1] : ur;
    const T v_l = k > 0 ? c.v[k - 1] : vl;
    const T v_r = k < W - 1 ? c.v[k + 1] : vr;
    fhn_cell<T, kArith>(c.u[k], c.v[k], u_r, u_l, dn.u[k], up.u[k], v_r, v_l, dn.v[k], up.v[k],
                       p, neg_eps, out.u[k], out.v[k]);
  }
}

__device__ __forceinline__ int wrap_index(int x, int n) {
  int r = x % n;
  return r < 0 ? r + n : r;
}

// Level-0 rows are staged through a per-warp shared-memory ring with
// cp.async (LDGSTS; 16-byte copies bypass L1): kStage = 6 slots, prefetch
// distance 3 ticks (thousands of cycles at 16 warps/SM).  Each lane copies and later reads back only its
// own W columns of each plane, so no cross-lane synchronisation is needed
// beyond the lane's own cp.async.wait_group.
#ifndef RDCNN_L0REG
#define RDCNN_L0REG 1
#endif
constexpr int kStage = 6;
constexpr int kPrefetch = 3;

template <int W, class T>
__device__ __forceinline__ void stage_row(uint32_t dst, const T* __restrict__ u,
                                          const T* __restrict__ v, size_t off) {
  constexpr int B = int(sizeof(T)) * W;  // bytes per lane per plane
  if constexpr (B % 16 == 0) {
    // 16-byte chunks, chunk-major: chunk c of every lane at c*512 + lane*16,
    // so each LDS.128 of a warp reads 512 contiguous bytes (dst is this
    // lane's chunk-0 address; B == 16 is the plain per-lane layout).
    constexpr int E = 16 / int(sizeof(T));
#pragma unroll
    for (int c = 0; c < B / 16; ++c) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 512 * c), "l"(u + off + E * c) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 32 * B + 512 * c), "l"(v + off + E * c)
                   : "memory");
    }
  } else {
    constexpr int E = int(sizeof(T));
#pragma unroll
    for (int k = 0; k < W; ++k) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(dst + E * k), "l"(u + off + k), "n"(E) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(dst + 32 * B + E * k), "l"(v + off + k), "n"(E) : "memory");
    }
  }
}

__device__ __forceinline__ void stage_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ void lds(uint32_t a, float& x) {
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(x) : "r"(a) : "memory");
}
__device__ __forceinline__ void lds(uint32_t a, double& x) {
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(x) : "r"(a) : "memory");
}

template <int W, class T>
__device__ __forceinline__ void read_staged(uint32_t src, Row<W, T>& r) {
  constexpr int B = int(sizeof(T)) * W;
  if constexpr (B % 16 == 0 && sizeof(T) == 4) {
#pragma unroll
    for (int c = 0; c < W; c += 4) {
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                   : "=f"(r.u[c]), "=f"(r.u[c + 1]), "=f"(r.u[c + 2]), "=f"(r.u[c + 3]) : "r"(src + 128 * c) : "memory");
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                   : "=f"(r.v[c]), "=f"(r.v[c + 1]), "=f"(r.v[c + 2]), "=f"(r.v[c + 3])
                   : "r"(src + 32 * B + 128 * c)
                   : "memory");
    }
  } else if constexpr (B == 16 && sizeof(T) == 8) {
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(r.u[0]), "=d"(r.u[1]) : "r"(src) : "memory");
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(r.v[0]), "=d"(r.v[1]) : "r"(src + 32 * B) : "memory");
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      lds(src + int(sizeof(T)) * k, r.u[k]);
      lds(src + 32 * B + int(sizeof(T)) * k, r.v[k]);
    }
  }
}

// ---- TMA bulk staging (fp32, W = 4) ------------------------------------------
// A warp's band row is 32 lanes x 16 bytes = 512 contiguous bytes per plane
// (two pieces where the band wraps around the torus edge), so lane 0 stages
// it with cp.async.bulk (the TMA engine) and the completion is counted on a
// per-slot mbarrier; every lane waits on the barrier instead of its own
// cp.async group.  -DRDCNN_BULK=2 stages the bands that do not wrap with one
// tensor-map copy (UTMALDG, both planes) per row instead: 8 % slower
// (4096^2 822k vs 893k).  Built with -DRDCNN_BULK=1 only: measured 6 % SLOWER than
// per-lane cp.async (4096^2: 785k vs 833k; batched 128^2: 876k vs 932k) --
// the elected copy, expect_tx and per-slot waits cost more issue slots than
// two LDGSTS per lane in an issue-bound kernel (profiles/README.md).
#ifndef RDCNN_BULK
#define RDCNN_BULK 0
#endif
template <int W, class T>
struct BulkStage {
  static constexpr bool value = RDCNN_BULK && W == 4 && sizeof(T) == 4;
};

// One elected lane: arm the slot's barrier with the row's 1024 bytes and
// issue the bulk copies of both planes.  All operands are warp-uniform
// (derived from blockIdx and kernel parameters), so they live in uniform
// registers and each copy is one UBLKCP.  The slot being recycled was last
// read (LDS) one tick earlier by this same warp and those values have been
// consumed, so no proxy fence is needed for the write-after-read.
__device__ __forceinline__ bool elect_one() {
  unsigned p;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
template <class T>
__device__ __forceinline__ void bulk_stage_row(uint32_t dst, const T* su, ptrdiff_t vdelta, uint32_t bytes_a,
                                               ptrdiff_t d_b, uint32_t bytes_b, uint32_t mbar) {
  if (elect_one()) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 1024;\n" ::"r"(mbar) : "memory");
    bulk_copy(dst, su, bytes_a, mbar);
    bulk_copy(dst + 512u, su + vdelta, bytes_a, mbar);
    if (bytes_b != 0) {
      bulk_copy(dst + bytes_a, su + d_b, bytes_b, mbar);
      bulk_copy(dst + 512u + bytes_a, su + vdelta + d_b, bytes_b, mbar);
    }
  }
  __syncwarp();
}
__device__ __forceinline__ void bulk_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "BW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra BW_%=;\n"
      "}\n" ::"r"(mbar), "r"(parity)
      : "memory");
}

// One band row of both planes by the TMA engine from the tensor map (UTMALDG):
// box {128 columns, 1 row, 2 planes} at column x, stacked row y.
__device__ __forceinline__ void tma_stage_row(uint32_t dst, const void* tmap, int x, int y, uint32_t mbar) {
  if (elect_one()) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 1024;\n" ::"r"(mbar) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(0), "r"(mbar)
        : "memory");
  }
  __syncwarp();
}

// ---- peer ring synchronisation (kPeer) --------------------------------------
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Wait until *p >= seq (wrap-safe).  Every lane polls, so every lane's later
// reads of the ghost rows are ordered after its own acquire.
__device__ __forceinline__ void wait_ready(const unsigned* p, unsigned seq) {
  while ((int)(ld_acquire_sys(p) - seq) < 0) __nanosleep(128);
}
// Called by lane 0 of an edge warp after every lane's peer stores were
// fenced: the last of `n` warps resets the counter and publishes `val`.
__device__ __forceinline__ void edge_done(unsigned* count, int n, unsigned* sig, unsigned val) {
  if (atomicAdd(count, 1u) == unsigned(n - 1)) {
    atomicExch(count, 0u);
    __threadfence_system();
    st_release_sys(sig, val);
  }
}

// Shared memory per CTA of the wavefront kernel (+ the bulk-staging barriers).
template <int W, class T>
constexpr int wavefront_smem_bytes(int warps) {
  return warps * (kStage * 2 * 32 * int(sizeof(T)) * W + (BulkStage<W, T>::value ? 64 : 0));
}

template <int V>
struct Int {
  static constexpr int value = V;
};
template <bool V>
struct Bool {
  static constexpr bool value = V;
};

// One warp per CTA: every per-warp quantity (grid, band, segment, row range,
// tick count) derives from blockIdx and kernel parameters only, so ptxas can
// keep the loop control on the uniform datapath.  The warps of a CTA never
// cooperate, so nothing is lost by not grouping them.
constexpr int kWarpsPerCta = 1;
constexpr int kCtaThreads = 32 * kWarpsPerCta;

// Resident warps per SM the register budget is capped for: 16 warps
// (<= 128 registers) for fp32 K <= 4 and fp64 K <= 2, else 8.
template <int K, class T, int W = 16 / int(sizeof(T))>
struct MinBlocks {
  static constexpr int kWarps = (sizeof(T) * W <= 16 && (sizeof(T) == 4 ? K <= 4 : K <= 2)) ? 16 : 8;
  static constexpr int value = kWarps / kWarpsPerCta;
};

// One K-level block of one warp's band x segment: stage, step, store;
// returns whether a stored value was non-finite (folded over the warp).
// (A persistent variant that looped over blocks, each warp waiting only for
// its 8 neighbours, measured 2.5 % slower than launches + PDL: profiles/.)
template <int K, int W, class T, int kArith, bool kPerGrid, bool kPeer, bool kWrap, bool kTee>
__device__ __forceinline__ bool wavefront_block(const StepArgsT<T>& a, unsigned char* smem_raw, int lane, int wib,
                                                int g, int band, int seg, unsigned frozen,
                                                const T* __restrict__ u_in_b, const T* __restrict__ v_in_b,
                                                T* __restrict__ u_out_b, T* __restrict__ v_out_b,
                                                BlockStats& stats) {
  static_assert(!kTee || (kPeer && RDCNN_L0REG), "the checkpoint tee is a slab (kPeer) feature");
  // Shared gene: read straight from the kernel-parameter bank.  Per-grid
  // genes (sweeps) come from global memory once per warp.
  const ParamsT<T> p = kPerGrid ? a.params[g] : a.shared;
  const T neg_eps = -p.eps;  // reference model.hpp:45 negates eps first

  const int G = a.cols / W;
  const int gl = band * a.band_groups - a.halo_groups + lane;
  const int grp = wrap_index(gl, G);
  // Store the band's useful lanes; gl >= G only when a band overhangs a grid
  // narrower than itself (the wrapped duplicates are not stored twice).
  const bool owner =
      lane >= a.halo_groups && lane < a.halo_groups + a.band_groups && gl < G;
  const int lane_l = (lane + 31) & 31;
  const int lane_r = (lane + 1) & 31;

  const size_t goff = (size_t)g * (size_t)a.grid_stride + (size_t)grp * W;
  const T* __restrict__ uin = u_in_b + goff;
  const T* __restrict__ vin = v_in_b + goff;
  T* __restrict__ uout = u_out_b + goff;
  T* __restrict__ vout = v_out_b + goff;
  const size_t pitch = (size_t)a.pitch;

  const int r0 = a.row_begin + seg * a.seg_rows;
  const int h = min(a.seg_rows, a.row_end - r0);
  const int n_load = h + 2 * K;       // level-0 rows x_0 .. x_{n_load-1}
  const int nt = h + 3 * K - 1;       // ticks until level K has produced h rows

  // Fused exchange: a warp reads the previous (next) rank's last (first)
  // rows iff it produces one of the first (last) `ghost` rows.  Wait until
  // that neighbour's edge warps of the previous block are done -- they wrote
  // those rows.  Our own signal at the end tells the neighbour we are done
  // reading them, so its next write of that buffer (two blocks on) cannot
  // race our reads.
  bool top_edge = false, bot_edge = false;
  if constexpr (kPeer) {
    top_edge = r0 < a.ghost;
    bot_edge = r0 + h > a.rows - a.ghost;
    const bool tracing = a.trace != nullptr && (top_edge || bot_edge);
    const unsigned long long t0 = tracing ? globaltimer() : 0ull;
    if (top_edge) wait_ready(a.ready + 0, a.seq);
    if (bot_edge) wait_ready(a.ready + 1, a.seq);
    if (tracing) {
      stats.wait_ns = globaltimer() - t0;
      // Level-0 rows beyond the slab: rows r0-K .. r0+h+K-1 outside [0, rows).
      const int beyond = max(0, K - r0) + max(0, r0 + h + K - a.rows);
      stats.peer_bytes = (unsigned long long)beyond * 32ull * 2ull * W * sizeof(T);
    }
  }

  // Running source row (wraps on the torus; never in ghosted slabs) and
  // running destination row: pointer increments, no per-tick index math.
  const int r_first = a.periodic ? wrap_index(r0 - K, a.rows) : r0 - K + a.ghost;
  const T* su = uin + (size_t)r_first * pitch;
  const ptrdiff_t vdelta = vin - uin;
  int rows_left = a.periodic ? a.rows - r_first : 0x7FFFFFFF;
  const size_t span = (size_t)a.rows * pitch;
  // kPeer pulls the rows beyond its slab straight from the ring neighbours'
  // input buffers (peer memory): the running source pointer starts in the
  // previous rank's last rows and jumps into this slab -- and from this
  // slab's end into the next rank's first rows -- exactly like the torus
  // wrap jumps, so the tick loop is unchanged.
  ptrdiff_t jump = -(ptrdiff_t)span, jump2 = 0;
  int rows_left2 = a.rows;
  if constexpr (kPeer) {
    auto delta = [](const T* to, const T* from) {
      return (ptrdiff_t)(((intptr_t)to - (intptr_t)from) / (intptr_t)sizeof(T));
    };
    const T* local0 = uin + (size_t)a.ghost * pitch;       // owned row 0 (this lane's columns)
    const T* local_end = local0 + (size_t)a.rows * pitch;  // owned row `rows`
    const T* prev_end = a.peer_top + (size_t)grp * W;      // prev's owned row rows_prev
    const T* next0 = a.peer_bot + (size_t)grp * W;         // next's owned row 0
    const int rf = r0 - K;
    rows_left2 = 0x7FFFFFFF;
    if (rf < 0) {
      su = prev_end + (ptrdiff_t)rf * (ptrdiff_t)pitch;
      rows_left = -rf;
      jump = delta(local0, prev_end);
      rows_left2 = a.rows;
      jump2 = delta(next0, local_end);
    } else {
      su = local0 + (size_t)rf * pitch;
      rows_left = a.rows - rf;
      jump = delta(next0, local_end);
    }
  }
  // The row step adds a kernel-parameter operand (no register, no rescale);
  // the wrap is a rarely taken branch, not predicated selects every tick.
  auto src_next = [&]() {
    su = reinterpret_cast<const T*>(reinterpret_cast<const char*>(su) + a.pitch_b);
    if (__builtin_expect(--rows_left == 0, 0)) {
      if constexpr (kPeer) {
        su += jump;
        rows_left = rows_left2;
        jump = jump2;
        rows_left2 = 0x7FFFFFFF;
      } else {
        su -= span;
        rows_left = a.rows;
      }
    }
  };
  T* du = uout + (size_t)(a.periodic ? r0 : r0 + a.ghost) * pitch;
  const ptrdiff_t vout_delta = vout - uout;
  // Checkpoint tee: the owned rows r0 .. r0+h-1 (level-0 rows of ticks
  // K .. K+h-1) go to the same place in a.tee_u.
  T* dc = nullptr;
  if constexpr (kTee) dc = a.tee_u + (size_t)g * (size_t)a.grid_stride + (size_t)grp * W + (size_t)(r0 + a.ghost) * pitch;

  constexpr uint32_t kLaneBytes = uint32_t(sizeof(T)) * W;
  // A lane's first chunk: lane*16 in the chunk-major layout (16-byte multiples), else lane*kLaneBytes.
  constexpr uint32_t kLaneStride = kLaneBytes % 16 == 0 ? 16u : kLaneBytes;
  constexpr uint32_t kSlot = 2 * 32 * kLaneBytes;  // bytes of one staged row (u,v)
  constexpr bool kBulk = BulkStage<W, T>::value;
  constexpr uint32_t kWarpSmem = kStage * kSlot + (kBulk ? 64u : 0u);
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem_raw) + (uint32_t)wib * kWarpSmem +
                        lane * kLaneStride;
  // Bulk staging works on warp-uniform quantities only: the band row starts
  // at lane 0's column group; a band that wraps the torus edge has a second
  // piece starting at group 0.  Slot s's barrier is at mbar0 + 8*s.
  const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(smem_raw) + (uint32_t)wib * kWarpSmem;
  const uint32_t mbar0 = ring0 + kStage * kSlot;
  uint32_t bytes_a = 32u * kLaneBytes, bytes_b = 0;
  ptrdiff_t d_b = 0;
  const T* ub = nullptr;  // uniform running source row (lane 0's group)
  // Tensor-map staging (RDCNN_BULK=2): bands that do not wrap the torus
  // column edge take one UTMALDG per row; the edge bands keep the two-piece
  // 1-D bulk copies.  y is the stacked row (grid g's row r at g*rows + r).
  bool use_tma = false;
  int tma_x = 0, tma_y = 0;
  if constexpr (kBulk) {
    const int gl0 = band * a.band_groups - a.halo_groups;  // lane 0's column group
    const int grp0 = wrap_index(gl0, G);
    int na = 32;
    if (gl0 < 0) na = -gl0;
    else if (gl0 + 32 > G) na = G - gl0;
    bytes_a = (uint32_t)na * kLaneBytes;
    bytes_b = 32u * kLaneBytes - bytes_a;
    d_b = -(ptrdiff_t)grp0 * W;  // group 0 relative to lane 0's group
    ub = u_in_b + (size_t)g * (size_t)a.grid_stride + (size_t)grp0 * W + (size_t)r_first * pitch;
    use_tma = RDCNN_BULK == 2 && a.tma_ok && bytes_b == 0 && a.periodic;
    tma_x = grp0 * W;
    tma_y = g * a.rows + r_first;
    if (elect_one()) {
#pragma unroll
      for (int q = 0; q < kStage; ++q)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mbar0 + 8u * q) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
  }
  auto stage = [&](uint32_t slot, uint32_t mb) {  // slot: the lane-0 (base) address
    if constexpr (kBulk) {
      if (use_tma) {
        tma_stage_row(slot, a.tmap, tma_x, tma_y, mb);
        ++tma_y;
        if (rows_left == 1) tma_y -= a.rows;  // same wrap point as su (src_next)
      } else {
        bulk_stage_row<T>(slot, ub, vdelta, bytes_a, d_b, bytes_b, mb);
        ub += pitch;
        if (rows_left == 1) ub -= span;  // same wrap point as su (src_next)
      }
    } else {
      stage_row<W, T>(slot + lane * kLaneStride, su, su + vdelta, 0);
    }
  };

  // Prime the staging ring with the rows of ticks 0 .. kPrefetch-1.
#pragma unroll
  for (int d = 0; d < kPrefetch; ++d) {
    if (d < n_load) {
      stage(ring0 + d * kSlot, mbar0 + 8u * d);
      src_next();
    }
    if constexpr (!kBulk) stage_commit();
  }

  Row<W, T> win[K > 1 ? K - 1 : 1][3];
#if RDCNN_L0REG
  Row<W, T> l0[3];
#endif
  Finite<T> fin;
  Finite<T> big;  // kStrictDiv2UF: centre |v| (fold_centre_v)
  const bool store = owner && frozen == 0u;
  // The 6-slot ring is two halves of 3: tick j lives in slot j % 6, i.e.
  // slot ph of the half the current 3-tick group uses; the prefetch of tick
  // j+3 goes to slot ph of the other half.  Both half bases swap once per
  // group, so every slot address is a base plus a compile-time offset.
  // Half bases are warp-uniform; a lane reads its own chunk at + lane_off.
  const uint32_t lane_off = lane * kLaneStride;
  uint32_t half_now = ring0, half_other = ring0 + 3 * kSlot;
  uint32_t mb_now = mbar0, mb_other = mbar0 + 24u;  // their slots' barriers (bulk)
  uint32_t phase_now = 0, phase_other = 0;           // barrier phase of each half's next use

  // One tick.  PH = j % 3 (compile-time ring slot); kSteady = every level is
  // active in this tick, so the validity tests disappear.
  auto tick = [&](auto ph_c, auto steady_c, int j) {
    constexpr int ph = decltype(ph_c)::value;
    constexpr bool kSteady = decltype(steady_c)::value;
    // Levels K..2, top-down: level t reads the level-(t-1) rows of ticks
    // j-3, j-2, j-1 (slots ph, ph+1, ph+2 mod 3), then level t-1 overwrites
    // slot ph with its tick-j row.
#pragma unroll
    for (int t = K; t >= 2; --t) {
      if (kSteady || (j >= 3 * t - 1 && j - (h + 2 * K - 1) < t)) {
        const Row<W, T>& up = win[t - 2][ph];
        const Row<W, T>& ce = win[t - 2][(ph + 1) % 3];
        const Row<W, T>& dn = win[t - 2][(ph + 2) % 3];
        fold_centre_v<W, T, kArith>(big, ce);
        if (t < K) {
          level_row<W, T, kArith, kWrap>(up, ce, dn, win[t - 1][ph], p, neg_eps, lane_l, lane_r);
        } else {
          Row<W, T> o;
          level_row<W, T, kArith, kWrap>(up, ce, dn, o, p, neg_eps, lane_l, lane_r);
          // Folded on every lane (non-storing lanes are cleared at the end),
          // so the store is the only guarded instruction.
          fold_finite<W, T>(fin, o);
          if (store) store_row<W, T>(du, du + vout_delta, 0, o);
          du = reinterpret_cast<T*>(reinterpret_cast<char*>(du) + a.pitch_b);
        }
      }
    }
    // Stage the row of tick j + kPrefetch into the slot of tick j - 3 (an
    // empty group past the end keeps the wait_group accounting uniform).
    if (j + kPrefetch < n_load) {
      stage(half_other + ph * kSlot, mb_other + 8u * ph);
      src_next();
    }
    if constexpr (!kBulk) stage_commit();
    // Level 1 from the level-0 rows of ticks j-2, j-1, j.
    // The row of tick j has landed.  Bulk: every filled slot is waited on
    // its own barrier, ticks 0 and 1 included (per-slot barriers complete in
    // any order, unlike cp.async groups; and no copy may still be in flight
    // when the CTA exits).
    if constexpr (kBulk) {
      if (kSteady || j < n_load) bulk_wait(mb_now + 8u * ph, phase_now);
    }
#if RDCNN_L0REG
    // Level-0 rows kept in a 3-slot register ring: each staged row is read
    // from shared memory once (tick j -> slot j % 3), ticks 0 and 1 included.
    if (kSteady || j < n_load) {
      if constexpr (!kBulk) stage_wait<kPrefetch>();
      read_staged<W, T>(lane_off + half_now + ph * kSlot, l0[ph]);
      if constexpr (kTee) {
        if (j >= K && j < K + h) {
          if (store) store_row<W, T>(dc, dc + vdelta, 0, l0[ph]);
          dc = reinterpret_cast<T*>(reinterpret_cast<char*>(dc) + a.pitch_b);
        }
      }
    }
    if (kSteady || (j >= 2 && j < n_load)) {
      const Row<W, T>& up = l0[(ph + 1) % 3];
      const Row<W, T>& ce = l0[(ph + 2) % 3];
      const Row<W, T>& dn = l0[ph];
#else
    if (kSteady || (j >= 2 && j < n_load)) {
      if constexpr (!kBulk) stage_wait<kPrefetch>();
      Row<W, T> up, ce, dn;
      read_staged<W, T>(lane_off + (ph >= 2 ? half_now + (ph - 2) * kSlot : half_other + (ph + 1) * kSlot), up);
      read_staged<W, T>(lane_off + (ph >= 1 ? half_now + (ph - 1) * kSlot : half_other + 2 * kSlot), ce);
      read_staged<W, T>(lane_off + half_now + ph * kSlot, dn);
#endif
      fold_centre_v<W, T, kArith>(big, ce);
      if constexpr (K == 1) {
        Row<W, T> o;
        level_row<W, T, kArith, kWrap>(up, ce, dn, o, p, neg_eps, lane_l, lane_r);
        fold_finite<W, T>(fin, o);
        if (store) store_row<W, T>(du, du + vout_delta, 0, o);
        du = reinterpret_cast<T*>(reinterpret_cast<char*>(du) + a.pitch_b);
      } else {
        level_row<W, T, kArith, kWrap>(up, ce, dn, win[0][ph], p, neg_eps, lane_l, lane_r);
      }
    }
  };

  // Steady ticks: every level active, j in [3K-1, n_load).
  const int steady_lo = 3 * K - 1, steady_hi = n_load;
  // Only the deepest instance gets a separate steady-state copy of the loop
  // body: for K <= 4 the doubled code costs more in instruction-cache misses
  // than the removed tests save (measured, profiles/README.md).
  constexpr bool kSplit = K >= 8;
  for (int j0 = 0; j0 < nt; j0 += 3) {
    if (kSplit && j0 >= steady_lo && j0 + 3 <= steady_hi) {
      tick(Int<0>{}, Bool<true>{}, j0);
      tick(Int<1>{}, Bool<true>{}, j0 + 1);
      tick(Int<2>{}, Bool<true>{}, j0 + 2);
    } else {
      tick(Int<0>{}, Bool<false>{}, j0);
      if (j0 + 1 < nt) tick(Int<1>{}, Bool<false>{}, j0 + 1);
      if (j0 + 2 < nt) tick(Int<2>{}, Bool<false>{}, j0 + 2);
    }
    const uint32_t t_half = half_now;
    half_now = half_other;
    half_other = t_half;
    const uint32_t t_mb = mb_now;
    mb_now = mb_other;
    mb_other = t_mb;
    const uint32_t t_ph = phase_now ^ 1u;  // the half just consumed is next used one phase on
    phase_now = phase_other;
    phase_other = t_ph;
  }
  if constexpr (!kBulk) stage_wait<0>();

  if constexpr (kPeer) {
    if (top_edge || bot_edge) {
      __threadfence_system();  // this lane's reads of the neighbours' rows are done
      __syncwarp();
      if (lane == 0) {
        if (top_edge) edge_done(a.edge_count + 0, a.n_top, a.sig_prev, a.seq + 1u);
        if (bot_edge) edge_done(a.edge_count + 1, a.n_bot, a.sig_next, a.seq + 1u);
      }
    }
  }

  if (!store) {  // halo lanes and frozen grids never flag
    fin = Finite<T>{};
    big = Finite<T>{};
  }
  if constexpr (kArith == kStrictDiv2UF) {
    if (big_centre_in_warp(big)) return true;
  }
  return fin.bad_in_warp();
}

// K levels per launch, W columns per lane, element type T.
//
// Schedule (a skewed wavefront, levels visited top-down within a tick): at
// tick j the warp has level-0 rows x_0..x_j (x_j = r0 - K + j) and
//   level t computes row x_j - (2t - 1) from the three level-(t-1) rows
//   produced at ticks j-3, j-2, j-1 (level 1: the level-0 rows of ticks
//   j-2, j-1, j, read back from the staging ring).
// Visiting t = K..1 means no level consumes a row produced in the same tick,
// so the K level updates of one tick are independent instruction streams the
// scheduler can interleave, and each level's oldest row slot can be
// overwritten in place once the level above has read it.
//
// Register rotation: level-t rows (t = 1..K-1) live in rings of 3 (tick j ->
// slot j % 3); the tick loop is unrolled by 3 so every slot index is a
// compile-time constant and no register is copied to advance a window.
//
// kWrap: full-width bands (halo_groups == 0, cols == 32*W), see level_row.
//
// kPeer (slab mode): the launch covers every owned row of the slab; warps
// whose segment reaches beyond it first wait for the neighbour's word, then
// stage those rows straight from the neighbour's input buffer (peer memory)
// and publish completion -- the halo exchange is fused into the step.
template <int K, int W, class T, int kArith, bool kPerGrid, bool kPeer = false, bool kWrap = false,
          bool kTee = false>
__global__ void __launch_bounds__(kCtaThreads, MinBlocks<K, T, W>::value)
    fhn_wavefront_kernel(const __grid_constant__ StepArgsT<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = kWarpsPerCta == 1 ? 0 : int(threadIdx.x >> 5);
  const long long warp_id = (long long)blockIdx.x * kWarpsPerCta + wib;
  const long long per_grid = (long long)a.n_segs * a.n_bands;
  if (warp_id >= per_grid * a.batch) return;
  unsigned long long t_start = 0;
  if (a.trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int g = int(warp_id / per_grid);
  const int rem = int(warp_id - (long long)g * per_grid);
  const int band = rem % a.n_bands;
  const int seg = rem / a.n_bands;

  // A grid that already blew up in an earlier launch of this advance stays
  // frozen (no stores), so the input of its first bad launch survives for
  // the host-side replay.  A flag carrying this launch's own tag was raised
  // by a sibling warp (or, in slab mode, by the boundary launch of the same
  // block) and does not freeze.  The flag is only needed at the first store.
  // Programmatic dependent launch: the next launch of the advance may start
  // its CTAs in this one's tail; nothing global is read before the previous
  // launch has completed (no-ops when launched without the PDL attribute).
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const unsigned fl = a.flags != nullptr ? *(volatile unsigned*)(a.flags + g) : 0u;
  const unsigned frozen = fl != 0u && fl != a.tag;

  BlockStats stats;
  const bool bad = wavefront_block<K, W, T, kArith, kPerGrid, kPeer, kWrap, kTee>(
      a, smem_raw, lane, wib, g, band, seg, frozen, a.u_in, a.v_in, a.u_out, a.v_out, stats);

  if (bad && lane == 0 && a.flags != nullptr) atomicCAS(a.flags + g, 0u, a.tag);
  if (a.trace != nullptr && lane == 0) {
    unsigned long long t_end;
    unsigned smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* tr = a.trace + (size_t)a.trace_stride * (size_t)warp_id;
    tr[0] = t_start;
    tr[1] = t_end;
    tr[2] = smid;
    if (a.trace_stride >= 5) {
      tr[3] = stats.wait_ns;
      tr[4] = stats.peer_bytes;
    }
  }

}

}  // namespace rdcnn_dev
