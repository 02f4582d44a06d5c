// rdcnn_cuda.cu -- C-ABI implementation (include/rdcnn_cuda.h): handles,
// launch planning, device-side initial states, blow-up replay, slab mode.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
//        -fmad=false -prec-div=true -ftz=false -shared -Xcompiler -fPIC
// (see __graft_entry__.build()).  Strict arithmetic relies on -ftz=false
// (reference keeps subnormals, SURVEY.md §7 "Denormals").
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <tuple>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <unistd.h>
#include <nccl.h>

#include "analysis.cuh"
#include "fhn_cluster.cuh"
#include "fhn_rowring.cuh"
#include "fhn_stencil.cuh"
#include "rdcnn_cuda.h"

using rdcnn_dev::ParamsT;
using rdcnn_dev::StepArgsT;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define RDCNN_CUDA_TRY(expr)                                                      \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return fail(RDCNN_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));  \
  } while (0)

#define RDCNN_TRY(expr)           \
  do {                            \
    int rc_ = (expr);             \
    if (rc_ != RDCNN_OK) return rc_; \
  } while (0)

constexpr int kThreads = rdcnn_dev::kCtaThreads;  // threads per stencil CTA

// ---------------------------------------------------------------------------
// Kernel dispatch over the compiled instances.
//   fp32: W in {1,4}, K in {1,2,4,8}, strict|fast, shared|per-grid gene
//   fp64: W in {1,2}, K in {1,2,4},   strict,      shared|per-grid gene
// ---------------------------------------------------------------------------

template <class T>
struct Traits;
#ifndef RDCNN_WIDE_F32
// fp32 columns per lane of the wide instances.  8 was measured and rejected:
// 212 registers -> 9 warps/SM, 507k vs 835k Mcell-updates/s at 4096^2.
#define RDCNN_WIDE_F32 4
#endif
template <>
struct Traits<float> {
  static constexpr int kWide = RDCNN_WIDE_F32;
  static constexpr int kMaxLevels = 8;
};
template <>
struct Traits<double> {
  static constexpr int kWide = 2;
  static constexpr int kMaxLevels = 4;
};

int k_index(int k) { return k == 1 ? 0 : k == 2 ? 1 : k == 4 ? 2 : 3; }

template <class T>
struct KernelTable {
  using Fn = void (*)(StepArgsT<T>);
  Fn fn[2][4][5][2][2] = {};        // [wide][k][arith][per_grid][wrap]
  int resident[2][4][5][2][2] = {};
};

template <class T, int W, int KI, int FI, int PI>
void fill_one(KernelTable<T>& t) {
  constexpr int K = 1 << KI;
  if constexpr (K <= Traits<T>::kMaxLevels && (FI == 0 || sizeof(T) == 4))
  {
    t.fn[W > 1][KI][FI][PI][0] = &rdcnn_dev::fhn_wavefront_kernel<K, W, T, FI, PI == 1, false, false>;
    t.fn[W > 1][KI][FI][PI][1] = &rdcnn_dev::fhn_wavefront_kernel<K, W, T, FI, PI == 1, false, true>;
  }
}

template <class T, int W, int KI>
void fill_k(KernelTable<T>& t) {
  fill_one<T, W, KI, 0, 0>(t);
  fill_one<T, W, KI, 0, 1>(t);
  fill_one<T, W, KI, 1, 0>(t);
  fill_one<T, W, KI, 1, 1>(t);
  fill_one<T, W, KI, 2, 0>(t);
  fill_one<T, W, KI, 2, 1>(t);
  fill_one<T, W, KI, 3, 0>(t);
  fill_one<T, W, KI, 3, 1>(t);
  fill_one<T, W, KI, 4, 0>(t);
  fill_one<T, W, KI, 4, 1>(t);
}

template <class T, int W>
void fill_w(KernelTable<T>& t) {
  fill_k<T, W, 0>(t);
  fill_k<T, W, 1>(t);
  fill_k<T, W, 2>(t);
  fill_k<T, W, 3>(t);
}

template <class T>
KernelTable<T>& table() {
  static KernelTable<T> t = [] {
    KernelTable<T> x;
    fill_w<T, 1>(x);
    fill_w<T, Traits<T>::kWide>(x);
    return x;
  }();
  return t;
}

// Dynamic shared memory of one CTA (the level-0 staging rings).
template <class T>
size_t smem_for(int w) {
  return w > 1 ? rdcnn_dev::wavefront_smem_bytes<Traits<T>::kWide, T>(kThreads / 32)
               : rdcnn_dev::wavefront_smem_bytes<1, T>(kThreads / 32);
}

// Resident CTAs per SM of one instance (cached; occupancy is immutable).
template <class T>
int resident_blocks(int k, int w, int arith, bool per_grid, bool wrap) {
  KernelTable<T>& t = table<T>();
  // Handles may launch concurrently from several host threads: the memo is
  // read and written atomically (every writer stores the same value).
  int* slot = &t.resident[w > 1][k_index(k)][arith][per_grid][wrap];
  int r = __atomic_load_n(slot, __ATOMIC_RELAXED);
  if (r == 0) {
    auto fn = t.fn[w > 1][k_index(k)][arith][per_grid][wrap];
    if (!fn || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, fn, kThreads, smem_for<T>(w)) !=
                   cudaSuccess || r < 1)
      r = 1;
    __atomic_store_n(slot, r, __ATOMIC_RELAXED);
  }
  return r;
}

// Programmatic dependent launch (PDL): consecutive stencil launches of an
// advance overlap launch latency and prologue with the previous launch's
// tail; the kernel issues griddepcontrol.wait before its first global read.
// Measured +4 % at 4096^2, K=4 (779k -> 810k).  RDCNN_PDL=0 turns it off.
// Used only for launches that fill the chip (see launch_pdl).
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RDCNN_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// `full`: the launch fills at least 3/4 of the resident warp slots.  A
// smaller launch must not use PDL: the next launch's CTAs would be
// dispatched at once into the many free slots and wait in
// griddepcontrol.wait beside the running warps, slowing them (1024^2, 49 %
// of the slots: 252k with PDL vs 341k without; 1536^2, 94 %: 519k vs 461k).
template <class Args>
cudaError_t launch_pdl(void (*fn)(Args), unsigned blocks, size_t smem, cudaStream_t s, const Args& a,
                       bool full = true) {
  if (!pdl_enabled() || !full) {
    fn<<<dim3(blocks), dim3(kThreads), smem, s>>>(a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, a);
}

// Fused peer-exchange instances (fp32 slabs, shared gene): [wide][k][fast].
struct PeerTable {
  using Fn = void (*)(StepArgsT<float>);
  Fn fn[2][4][4][2][2] = {};  // [wide][k][arith][wrap][tee]
  int resident[2][4][4][2][2] = {};
};

template <int W, int KI, int FI>
void fill_peer_one(PeerTable& t) {
  t.fn[W > 1][KI][FI][0][0] = &rdcnn_dev::fhn_wavefront_kernel<1 << KI, W, float, FI, false, true, false>;
  t.fn[W > 1][KI][FI][1][0] = &rdcnn_dev::fhn_wavefront_kernel<1 << KI, W, float, FI, false, true, true>;
  t.fn[W > 1][KI][FI][0][1] = &rdcnn_dev::fhn_wavefront_kernel<1 << KI, W, float, FI, false, true, false, true>;
  t.fn[W > 1][KI][FI][1][1] = &rdcnn_dev::fhn_wavefront_kernel<1 << KI, W, float, FI, false, true, true, true>;
}

template <int W>
void fill_peer_w(PeerTable& t) {
  fill_peer_one<W, 0, 0>(t); fill_peer_one<W, 0, 1>(t); fill_peer_one<W, 0, 2>(t); fill_peer_one<W, 0, 3>(t);
  fill_peer_one<W, 1, 0>(t); fill_peer_one<W, 1, 1>(t); fill_peer_one<W, 1, 2>(t); fill_peer_one<W, 1, 3>(t);
  fill_peer_one<W, 2, 0>(t); fill_peer_one<W, 2, 1>(t); fill_peer_one<W, 2, 2>(t); fill_peer_one<W, 2, 3>(t);
  fill_peer_one<W, 3, 0>(t); fill_peer_one<W, 3, 1>(t); fill_peer_one<W, 3, 2>(t); fill_peer_one<W, 3, 3>(t);
}

PeerTable& peer_table() {
  static PeerTable t = [] {
    PeerTable x;
    fill_peer_w<1>(x);
    fill_peer_w<4>(x);
    return x;
  }();
  return t;
}

int peer_resident_blocks(int k, int w, int arith, bool wrap, bool tee) {
  PeerTable& t = peer_table();
  int& r = t.resident[w > 1][k_index(k)][arith][wrap][tee];
  if (r == 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, t.fn[w > 1][k_index(k)][arith][wrap][tee], kThreads,
                                                      smem_for<float>(w)) != cudaSuccess || n < 1)
      n = 1;
    r = n;
  }
  return r;
}

template <class T>
cudaError_t launch_stencil(int k, int w, int arith, bool per_grid, bool wrap, const StepArgsT<T>& a,
                           long long warps, cudaStream_t s, bool full) {
  if (warps <= 0) return cudaSuccess;
  if (k != 1 && k != 2 && k != 4 && k != 8) return cudaErrorInvalidValue;
  auto fn = table<T>().fn[w > 1][k_index(k)][arith][per_grid][wrap];
  if (!fn) return cudaErrorInvalidValue;
  const long long blocks = (warps + (kThreads / 32) - 1) / (kThreads / 32);
  return launch_pdl(fn, (unsigned)blocks, smem_for<T>(w), s, a, full);
}

// Band/segment decomposition of one launch.
struct Plan {
  int w = 1, halo = 0, band_groups = 0, n_bands = 0, seg_rows = 0, n_segs = 0;
  long long warps = 0;
};

Plan make_plan(int cols, int w, int k, int batch, int row_begin, int row_end,
               int seg_override, int sm_count, int resident_warps_per_sm) {
  Plan p;
  p.w = w;
  const int G = cols / w;
  if (G == 32) {  // the band is the whole row: shuffles wrap, no halo lanes
    p.halo = 0;
    p.band_groups = 32;
    p.n_bands = 1;
  } else {
    p.halo = (k + w - 1) / w;
    const int useful = 32 - 2 * p.halo;
    p.n_bands = (G + useful - 1) / useful;
    p.band_groups = (G + p.n_bands - 1) / p.n_bands;
  }
  const int nrows = row_end - row_begin;
  if (nrows <= 0) return p;
  int h;
  if (seg_override > 0) {
    h = seg_override;
  } else {
    // One full wave of resident warps (every warp runs start to finish with
    // no tail), but segments of at least 8K rows so the 2K-row wavefront
    // start-up stays a small fraction.
    const long long target = (long long)std::max(sm_count, 1) * std::max(resident_warps_per_sm, 4);
    const long long per_seg = (long long)batch * p.n_bands;
    const long long segs = std::max<long long>(1, (target + per_seg - 1) / per_seg);
    h = (int)std::max<long long>(1, (nrows + segs - 1) / segs);
    // Long segments amortise the 2K-row wavefront start-up; small lattices
    // that cannot fill the chip anyway trade that for more warps.
    const int h_long = std::max(16, 8 * k);
    const long long warps_long = per_seg * ((nrows + h_long - 1) / h_long);
    h = std::max(h, std::min(nrows, warps_long >= target / 2 ? h_long : std::max(4, 2 * k)));
  }
  h = std::min(h, nrows);
  p.seg_rows = h;
  p.n_segs = (nrows + h - 1) / h;
  p.warps = (long long)p.n_segs * p.n_bands * batch;
  // Never spill long segments into a second wave: warps beyond the resident
  // slots start only when a slot frees.  A short last segment (the runt
  // row range, at most a third of h) may overflow -- its warps finish early
  // and the overflow fills their slots (4096^2: 68 x 35 warps, runt 9 rows,
  // measured faster than 67 segments).  Otherwise use floor(slots/per_seg)
  // segments (8192^2: 2415 -> 2346 warps, 763k -> 825k Mcell-updates/s).
  if (seg_override <= 0) {
    const long long slots = (long long)std::max(sm_count, 1) * std::max(resident_warps_per_sm, 4);
    const long long per_seg = (long long)batch * p.n_bands;
    const long long over = p.warps - slots;
    const int h_last = nrows - (p.n_segs - 1) * p.seg_rows;
    if (over > 0 && p.warps < 2 * slots && !(h_last * 3 <= p.seg_rows && over <= per_seg)) {
      const long long segs = slots / per_seg;
      if (segs >= 1) {
        const int h2 = (int)((nrows + segs - 1) / segs);
        p.seg_rows = h2;
        p.n_segs = (nrows + h2 - 1) / h2;
        p.warps = (long long)p.n_segs * per_seg;
      }
    }
  }
  return p;
}

// ---------------------------------------------------------------------------
// Device-side initial states (init.hpp:20-64, rng.hpp:11-39).
// Draw d (0-based) of splitmix64(seed) is mix(seed + (d+1)*golden), so every
// cell's value is computed independently of the others.
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t d) {
  uint64_t z = seed + (d + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void unit_of(uint64_t z, float& x) {
  x = __fmul_rn((float)(z >> 40), 0x1.0p-24f);  // rng.hpp:28, exact
}
__device__ __forceinline__ void unit_of(uint64_t z, double& x) {
  x = __dmul_rn((double)(z >> 11), 0x1.0p-53);  // rng.hpp:25, exact
}

// Writes rows [row_offset, row_offset + local_rows) of a global
// global_rows x cols lattice initialised with typ (1 or 2).
template <class T>
__global__ void init_kernel(T* u, T* v, int pitch, long long grid_stride, int batch,
                            int local_rows, int cols, int global_rows, int row_offset, int typ,
                            uint64_t seed) {
  const long long n = (long long)local_rows * cols;
  const long long gcells = (long long)global_rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * batch;
       idx += (long long)gridDim.x * blockDim.x) {
    const int g = int(idx / n);
    const long long c = idx - (long long)g * n;
    const int li = int(c / cols);
    const int j = int(c - (long long)li * cols);
    const int i = li + row_offset;  // global row
    T uu = T(0), vv = T(0);
    if (typ == 2) {
      const long long cell = (long long)i * cols + j;
      unit_of(splitmix_draw(seed, (uint64_t)cell), uu);
      unit_of(splitmix_draw(seed, (uint64_t)(gcells + cell)), vv);
    } else {
      const int i0 = (global_rows - 11) / 2, j0 = (cols - 11) / 2;  // init.hpp:36-37
      if (i >= i0 && i < i0 + 11 && j >= j0 && j < j0 + 11) {
        const int d = (i - i0) * 11 + (j - j0);
        unit_of(splitmix_draw(seed, (uint64_t)d), uu);
        unit_of(splitmix_draw(seed, (uint64_t)(121 + d)), vv);
      }
    }
    const size_t off = (size_t)g * grid_stride + (size_t)li * pitch + j;
    u[off] = uu;
    v[off] = vv;
  }
}

template <class T>
__global__ void image_kernel(T* u, T* v, int pitch, long long grid_stride, int batch, int rows,
                             int cols, const uint8_t* px, const T* lut) {
  const long long n = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * batch;
       idx += (long long)gridDim.x * blockDim.x) {
    const int g = int(idx / n);
    const long long c = idx - (long long)g * n;
    const int i = int(c / cols);
    const int j = int(c - (long long)i * cols);
    const T x = lut[px[c]];
    const size_t off = (size_t)g * grid_stride + (size_t)i * pitch + j;
    u[off] = x;
    v[off] = x;
  }
}

__global__ void div3_selftest_kernel(int domain, unsigned long long* count, unsigned* first_bad) {
  unsigned long long local = 0;
  unsigned first = 0xFFFFFFFFu;
  const unsigned long long total = 1ull << 32;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       k < total; k += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned bits = (unsigned)k;
    float x = __uint_as_float(bits);
    if (domain == 1) x = __fmul_rn(x, x);
    if (domain == 2) x = __uint_as_float(bits & 0x7FFFFFFFu);
    const float want = __fdiv_rn(x, 3.0f);
    bool ok;
    if (domain == 2) {
      // The gated 2-op quotient inside RN(c - x/3) at the gate boundary
      // c = +-2^-90 and at c = 1 (fhn_stencil.cuh div3_rn2).
      const float q2 = rdcnn_dev::div3_rn2(x);
      ok = true;
      const float cs[3] = {__uint_as_float(0x12800000u), __uint_as_float(0x92800000u), 1.0f};
      for (int j = 0; j < 3; ++j) {
        const float a = __fsub_rn(cs[j], q2), b = __fsub_rn(cs[j], want);
        if (isfinite(a) != isfinite(b) || (isfinite(a) && __float_as_uint(a) != __float_as_uint(b))) ok = false;
      }
    } else {
      const float got = rdcnn_dev::div3_rn(x);
      ok = isfinite(x) ? __float_as_uint(got) == __float_as_uint(want) : !isfinite(got);
    }
    if (!ok) {
      ++local;
      first = min(first, bits);
    }
  }
  if (local) {
    atomicAdd(count, local);
    atomicMin(first_bad, first);
  }
}

// fp64: every exponent (all 2048) x a hashed stream of mantissas, plus the
// same inputs squared (the x = u*u domain), against IEEE __ddiv_rn.
__global__ void div3_selftest_f64_kernel(unsigned long long samples, unsigned long long* count,
                                         unsigned long long* first_bad) {
  unsigned long long local = 0, first = ~0ull;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       k < samples; k += (unsigned long long)gridDim.x * blockDim.x) {
    uint64_t z = splitmix_draw(0x5EEDull, k);
    const uint64_t expo = k & 0x7FFull;                 // sweep every exponent
    uint64_t bits = (z & 0x800FFFFFFFFFFFFFull) | (expo << 52);
    if ((k >> 11) % 7 == 0) bits &= ~0xFFFFFFFFull;     // low mantissa words zero
    if ((k >> 11) % 11 == 0) bits |= 0xFFFFFFFFull;     // ... and all ones
    for (int sq = 0; sq < 2; ++sq) {
      double x = __longlong_as_double((long long)bits);
      if (sq) x = __dmul_rn(x, x);
      const double want = __ddiv_rn(x, 3.0);
      const double got = rdcnn_dev::div3_rn(x);
      bool ok;
      if (isfinite(x))
        ok = __double_as_longlong(got) == __double_as_longlong(want) || (x == 0.0 && got == 0.0);
      else
        ok = !isfinite(got);
      if (!ok) {
        ++local;
        first = min(first, (unsigned long long)bits);
      }
    }
  }
  if (local) {
    atomicAdd(count, local);
    atomicMin(first_bad, first);
  }
}

// NCCL, resolved at run time from whichever libnccl.so.2 the process already
// has (torch's) or the system one, so the library carries no link-time NCCL
// dependency and single-GPU users never load it.
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
    a.send = (decltype(a.send))dlsym(h, "ncclSend");
    a.recv = (decltype(a.recv))dlsym(h, "ncclRecv");
    a.group_start = (decltype(a.group_start))dlsym(h, "ncclGroupStart");
    a.group_end = (decltype(a.group_end))dlsym(h, "ncclGroupEnd");
    a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.send && a.recv && a.group_start &&
           a.group_end && a.error_string;
    return a;
  }();
  return api;
}

#define RDCNN_NCCL_TRY(expr)                                                          \
  do {                                                                                \
    ncclResult_t r_ = (expr);                                                         \
    if (r_ != ncclSuccess)                                                            \
      return fail(RDCNN_ECUDA, "%s failed: %s", #expr, nccl().error_string(r_));     \
  } while (0)

int sm_count_for(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) n = 148;
  return n;
}

}  // namespace

// ---------------------------------------------------------------------------
// Handle.
// ---------------------------------------------------------------------------

struct rdcnn_sim {
  int rows = 0, cols = 0, batch = 1, device = 0, mode = RDCNN_STRICT;
  int elem = 4;           // bytes per value: 4 (fp32) or 8 (fp64)
  bool slab = false;
  int ghost = 0;          // slab mode: ghost rows per side
  int pitch = 0;          // elements between rows
  int plane_off = 0;      // elements from u row start to v row start (slab: cols)
  long long grid_stride = 0;  // elements between grids (periodic planar: rows*cols)
  size_t buf_elems = 0;   // elements per buffer (both planes, all grids)
  void* buf[2] = {nullptr, nullptr};
  int cur = 0;            // front buffer index
  void* d_params = nullptr;   // ParamsT<T>[batch]
  ParamsT<float> h_params_f{};   // the shared gene (params_stride == 0)
  ParamsT<double> h_params_d{};
  int params_stride = 0;
  bool div2_ok = true;      // every gene has |c| >= 2^-90: the 2-op x/3 instance is exact
  bool unit_dv = false;     // every gene has Dv == 1: the Dv*lap_v product is the identity
  bool replaying = false;   // replay_grid: the reference-order instance, so the post-blow-up state is its
  int arith_override = -1;  // RDCNN_DIV3 / tests: force the 3-op (0) or 2-op (2) strict instance
  unsigned* d_flags = nullptr;  // batch words (+1 scratch for replays)
  unsigned* h_flags = nullptr;  // pinned mirror
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0;
  long launches = 0;
  int max_levels = 4;
  int seg_rows = 0;
  bool tma_ok = false;              // RDCNN_BULK=2 builds: tensor maps of both buffers
  alignas(64) unsigned char tmap[2][128];
  int tuned_seg[4] = {0, 0, 0, 0};  // autotuned segment height per K (0: not tuned)
  bool tuned[4] = {false, false, false, false};
  int seg_force = 0;                // set while an autotune candidate runs
  int cluster_mode = 0;       // persistent cluster path: 0 auto, 1 required, -1 off
  long long* d_first_bad = nullptr;  // cluster path result word
  std::map<std::pair<long, int>, cudaGraphExec_t> graphs;  // captured advances by (steps, start buffer)
  int sm_count = 148;
  unsigned slab_tag = 0;
  // slab ring (native multi-GPU path)
  ncclComm_t comm = nullptr;
  int ring_rank = 0, ring_world = 1;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_xchg = nullptr;
  // fused peer ring (rdcnn_slab_attach_peers): peer memory of the ring
  // neighbours, opened from their IPC handles (or taken as is in-process)
  bool p2p = false;
  unsigned* p2p_words = nullptr;    // own: [0] top ready, [1] bottom ready, [2..3] edge counters
  void* peer_buf[2][2] = {};        // [prev, next][buffer]
  unsigned* peer_words[2] = {};     // [prev, next]
  int peer_rows[2] = {0, 0};
  unsigned p2p_seq = 0;             // blocks run since attach (equal on every rank)
  void* ckpt = nullptr;             // slab: a recent advance's input buffer (ghosts included)
  long ckpt_age = -1;               // iterations from the checkpointed state to now (-1: none)
  long ckpt_age_at_call = 0;        // ... to the start of the last advance
  std::vector<void*> ipc_opened;    // cudaIpcCloseMemHandle on destroy
  void* frames = nullptr;   // snapshot store: n_frames x batch u-planes
  int n_frames = 0;
  double* d_stats = nullptr;        // 3*batch doubles (min, max, median) + batch thresholds
  long long* d_counts = nullptr;    // batch counts
  unsigned long long* d_digest = nullptr;  // batch FNV digests (rdcnn_sim_checksums)
  void* d_scratch = nullptr;        // per-call staging (image pixels, normalised frames), grown on demand
  size_t scratch_bytes = 0;

  template <class T>
  T* u_ptr(int b) {
    return static_cast<T*>(buf[b]);
  }
  template <class T>
  T* v_ptr(int b) {
    return slab ? static_cast<T*>(buf[b]) + plane_off
                : static_cast<T*>(buf[b]) + (size_t)rows * cols * batch;
  }
  template <class T>
  const ParamsT<T>& shared_params() const;
};

template <>
const ParamsT<float>& rdcnn_sim::shared_params<float>() const { return h_params_f; }
template <>
const ParamsT<double>& rdcnn_sim::shared_params<double>() const { return h_params_d; }

namespace {

template <class T>
int width_for(const rdcnn_sim* s) {
  // The fp32 wide instances stage rows with cp.async.bulk, which needs every
  // band to wrap the torus edge at most once: at least 32 column groups.
  const bool bulk = rdcnn_dev::BulkStage<Traits<T>::kWide, T>::value;
  return (s->cols % Traits<T>::kWide == 0 && (!bulk || s->cols / Traits<T>::kWide >= 32)) ? Traits<T>::kWide : 1;
}

// Arithmetic instance of a launch: fast mode, or strict with the 2-op x/3
// when every gene of the handle passes its gate (fhn_stencil.cuh div3_rn2)
// -- and without the Dv*lap_v product when every gene also has Dv == 1
// (kStrictDiv2U) -- else strict with the 3-op x/3.  fp64 always takes the
// 3-op strict path.
template <class T>
int arith_for(const rdcnn_sim* s) {
  if (s->mode == RDCNN_FAST) return rdcnn_dev::kFastArith;
  if (sizeof(T) != 4 || !s->div2_ok || s->arith_override == 0) return rdcnn_dev::kStrictArith;
  if (s->arith_override == 2 || !s->unit_dv) return rdcnn_dev::kStrictDiv2;
  // The fused v tail (kStrictDiv2UF) for periodic handles; slabs (their own
  // replay protocol) and RDCNN_DIV3=u keep the separate 4*v_c product.
  if (s->slab || s->replaying || s->arith_override == 3) return rdcnn_dev::kStrictDiv2U;
  return rdcnn_dev::kStrictDiv2UF;
}

// The gate of the 2-op x/3: |c| >= 2^-90 (false for NaN).
template <class T>
bool div2_gate(const ParamsT<T>* p, int n) {
  for (int i = 0; i < n; ++i)
    if (!(std::fabs((double)p[i].c) >= 0x1p-90)) return false;
  return true;
}

// The gate of kStrictDiv2U: Dv == 1 exactly (after narrowing) for every gene.
template <class T>
bool unit_dv_gate(const ParamsT<T>* p, int n) {
  for (int i = 0; i < n; ++i)
    if (!(p[i].dv == T(1))) return false;
  return n > 0;
}

template <class T>
StepArgsT<T> base_args(rdcnn_sim* s, int in_buf, int out_buf) {
  StepArgsT<T> a{};
  a.u_in = s->u_ptr<T>(in_buf);
  a.v_in = s->v_ptr<T>(in_buf);
  a.u_out = s->u_ptr<T>(out_buf);
  a.v_out = s->v_ptr<T>(out_buf);
  a.grid_stride = s->grid_stride;
  a.rows = s->rows;
  a.cols = s->cols;
  a.pitch = s->pitch;
  a.pitch_b = (long long)s->pitch * (long long)sizeof(T);
  a.periodic = s->slab ? 0 : 1;
  a.ghost = s->slab ? s->ghost : 0;
  a.batch = s->batch;
  a.shared = s->shared_params<T>();
  a.params = static_cast<const ParamsT<T>*>(s->d_params);
  a.params_stride = s->params_stride;
  a.flags = s->d_flags;
  a.tma_ok = s->tma_ok ? 1 : 0;
  if (s->tma_ok) std::memcpy(a.tmap, s->tmap[in_buf], sizeof a.tmap);
  return a;
}

// Segment height override for a launch: an autotune candidate, the user's
// seg_rows, or the autotuned height (full periodic launches only).
int seg_for(const rdcnn_sim* s, int k, int row_begin, int row_end) {
  if (s->seg_force > 0) return s->seg_force;
  if (s->seg_rows > 0) return s->seg_rows;
  if (s->slab || row_begin != 0 || row_end != s->rows) return 0;
  return s->tuned_seg[k_index(k)];
}

// ---- row-ring path (fhn_rowring.cuh): a cluster spans a whole torus row ----
// Periodic fp32 lattices whose width is 128*M*C columns (M warps per CTA, C
// CTAs per cluster) can run their K=4 blocks with no halo lanes.  Measured
// slower than the wavefront kernel (4096^2: 744k vs 894k), so it runs only
// with RDCNN_ROWRING=1; RDCNN_RR_M pins M.
struct RowRingTable {
  using Fn = void (*)(StepArgsT<float>);
  Fn fn[4][3][2] = {};             // [M: -,4,8,16][arith][per_grid]
  int max_clusters[4][3][2][17] = {};  // by C (0: not yet queried)
};

template <int MI, int FI>
void fill_rr(RowRingTable& t) {
  t.fn[MI][FI][0] = &rdcnn_dev::fhn_rowring_kernel<4, 2 << MI, FI, false>;
  t.fn[MI][FI][1] = &rdcnn_dev::fhn_rowring_kernel<4, 2 << MI, FI, true>;
}
template <int MI>
void fill_rr_m(RowRingTable& t) {
  fill_rr<MI, 0>(t);
  fill_rr<MI, 1>(t);
  fill_rr<MI, 2>(t);
}

std::mutex g_rr_mu;
RowRingTable& rr_table() {
  static RowRingTable t = [] {
    RowRingTable x;
    fill_rr_m<1>(x);
    fill_rr_m<2>(x);
    fill_rr_m<3>(x);
    return x;
  }();
  return t;
}

// RDCNN_ROWRING=1: use it where it fits; =2: also fail any K=4 launch that
// cannot take it (tests prove the path ran).
int rowring_setting() {
  static const int v = [] {
    const char* e = std::getenv("RDCNN_ROWRING");
    return e && (e[0] == '1' || e[0] == '2') ? e[0] - '0' : 0;
  }();
  return v;
}
bool rowring_enabled() { return rowring_setting() > 0; }

int rowring_forced_m() {
  static const int m = [] {
    const char* e = std::getenv("RDCNN_RR_M");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

struct RRPlan {
  int M = 0, C = 0, seg_rows = 0, n_segs = 0;
  long long clusters = 0;
  size_t smem = 0;
  bool full = false;
  RowRingTable::Fn fn = nullptr;
};

int rr_mi(int m) { return m == 2 ? 0 : m == 4 ? 1 : m == 8 ? 2 : 3; }

// Chooses M, C and the segment plan; false when the launch does not fit the
// row-ring path (the wavefront kernel runs it).
bool rowring_plan(rdcnn_sim* s, int k, int arith, bool per_grid, int batch, int row_begin, int row_end,
                  int seg_override, RRPlan& p) {
  if (!rowring_enabled() || s->slab || s->elem != 4 || k != 4 || s->cols % 128 != 0) return false;
  const int wr = s->cols / 128;  // warps per row = M*C
  static const int kPref[] = {16, 8, 4};
  const int forced = rowring_forced_m();
  int M = 0;
  for (int m : kPref) {
    if (forced && m != forced) continue;
    if (m <= wr && wr % m == 0 && wr / m <= 16) {
      M = m;
      break;
    }
  }
  if (M == 0) return false;
  const int C = wr / M;
  RowRingTable& t = rr_table();
  const int mi = rr_mi(M);
  p.fn = t.fn[mi][arith][per_grid];
  if (!p.fn) return false;
  p.M = M;
  p.C = C;
  p.smem = (size_t)rdcnn_dev::rowring_smem_bytes(M, k);
  int nc;
  {
    std::lock_guard<std::mutex> lock(g_rr_mu);
    int& slot = t.max_clusters[mi][arith][per_grid][C];
    if (slot == 0) {
      if (cudaFuncSetAttribute(p.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess) {
        cudaGetLastError();
        slot = -1;
      } else {
        if (C > 8) cudaFuncSetAttribute(p.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)C);
        cfg.blockDim = dim3(32u * (unsigned)M);
        cfg.dynamicSmemBytes = p.smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, p.fn, &cfg) != cudaSuccess || n < 1) {
          cudaGetLastError();
          n = -1;
        }
        slot = n;
      }
    }
    nc = slot;
  }
  if (nc < 1) return false;
  const int nrows = row_end - row_begin;
  if (nrows <= 0) return false;
  int h;
  if (seg_override > 0) {
    h = seg_override;
  } else {
    // As make_plan: one wave of clusters, segments of at least 8K rows
    // unless the lattice cannot fill the chip anyway.
    const long long segs = std::max<long long>(1, nc / std::max(batch, 1));
    h = (int)std::max<long long>(1, (nrows + segs - 1) / segs);
    const int h_long = std::max(16, 8 * k);
    const long long cl_long = (long long)batch * ((nrows + h_long - 1) / h_long);
    h = std::max(h, std::min(nrows, cl_long >= nc / 2 ? h_long : std::max(4, 2 * k)));
  }
  h = std::min(h, nrows);
  p.seg_rows = h;
  p.n_segs = (nrows + h - 1) / h;
  p.clusters = (long long)p.n_segs * batch;
  if (seg_override <= 0 && p.clusters > nc && p.clusters < 2LL * nc && nc / batch >= 1) {
    const long long segs = nc / batch;
    p.seg_rows = (int)((nrows + segs - 1) / segs);
    p.n_segs = (nrows + p.seg_rows - 1) / p.seg_rows;
    p.clusters = (long long)p.n_segs * batch;
  }
  p.full = 4 * p.clusters >= 3LL * nc;
  return true;
}

cudaError_t launch_rowring(const RRPlan& p, StepArgsT<float> a, cudaStream_t st) {
  a.seg_rows = p.seg_rows;
  a.n_segs = p.n_segs;
  a.n_bands = p.C;
  a.band_groups = 32 * p.M;
  a.halo_groups = 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  int na = 1;
  if (pdl_enabled() && p.full) {
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    na = 2;
  }
  cfg.gridDim = dim3((unsigned)(p.clusters * p.C));
  cfg.blockDim = dim3(32u * (unsigned)p.M);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = (unsigned)na;
  return cudaLaunchKernelEx(&cfg, p.fn, a);
}

template <class T>
cudaError_t launch_range(rdcnn_sim* s, int k, StepArgsT<T> a, int row_begin, int row_end,
                         cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    RRPlan rp;
    if (a.trace == nullptr &&
        rowring_plan(s, k, std::min(arith_for<T>(s), int(rdcnn_dev::kStrictDiv2)), a.params_stride != 0, a.batch, row_begin, row_end,
                     seg_for(s, k, row_begin, row_end), rp)) {
      a.row_begin = row_begin;
      a.row_end = row_end;
      ++s->launches;
      return launch_rowring(rp, a, st);
    }
    if (rowring_setting() == 2 && k == 4 && a.trace == nullptr) return cudaErrorNotSupported;
  }
  const int w = width_for<T>(s);
  const int arith = arith_for<T>(s);
  const bool per_grid = a.params_stride != 0;
  const bool wrap = s->cols / w == 32;  // full-width bands (make_plan: halo 0)
  const int rw = resident_blocks<T>(k, w, arith, per_grid, wrap) * (kThreads / 32);
  Plan p = make_plan(s->cols, w, k, a.batch, row_begin, row_end, seg_for(s, k, row_begin, row_end), s->sm_count, rw);
  if (p.warps == 0) return cudaSuccess;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.seg_rows = p.seg_rows;
  a.n_segs = p.n_segs;
  a.n_bands = p.n_bands;
  a.band_groups = p.band_groups;
  a.halo_groups = p.halo;
  ++s->launches;
  return launch_stencil<T>(k, w, arith, per_grid, wrap, a, p.warps, st,
                           4 * p.warps >= 3LL * rw * s->sm_count);
}

int alloc_common(rdcnn_sim* s) {
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  s->sm_count = sm_count_for(s->device);
  // A/B and tests: RDCNN_DIV3=3 pins the 3-op x/3 strict instance, =2 the
  // gated 2-op one with the Dv*lap_v product kept (still subject to its
  // gate); unset or anything else: automatic.
  if (const char* e = std::getenv("RDCNN_DIV3"))
    s->arith_override = e[0] == '3' ? 0 : e[0] == '2' ? 2 : e[0] == 'u' ? 3 : -1;
  RDCNN_CUDA_TRY(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  RDCNN_CUDA_TRY(cudaEventCreate(&s->ev0));
  RDCNN_CUDA_TRY(cudaEventCreate(&s->ev1));
  for (int b = 0; b < 2; ++b) {
    RDCNN_CUDA_TRY(cudaMalloc(&s->buf[b], s->buf_elems * s->elem));
    RDCNN_CUDA_TRY(cudaMemsetAsync(s->buf[b], 0, s->buf_elems * s->elem, s->stream));
  }
  RDCNN_CUDA_TRY(cudaMalloc(&s->d_params, sizeof(ParamsT<double>) * (size_t)s->batch));
  RDCNN_CUDA_TRY(cudaMalloc(&s->d_flags, sizeof(unsigned) * ((size_t)s->batch + 1)));
  RDCNN_CUDA_TRY(cudaMemsetAsync(s->d_flags, 0, sizeof(unsigned) * ((size_t)s->batch + 1), s->stream));
  RDCNN_CUDA_TRY(cudaMallocHost(&s->h_flags, sizeof(unsigned) * ((size_t)s->batch + 1)));
  // Default gene (gene.hpp:13-24) until set_params is called.
  const double g7[7] = {0.1, -0.3, 1.3, -0.1, 1.0, 0.06, 1.0};
  s->h_params_d = {g7[0], g7[1], g7[2], g7[3], g7[4], g7[5], g7[6]};
  rdcnn_params_f32 pf;
  rdcnn_params_from_gene(g7, &pf);
  std::memcpy(&s->h_params_f, &pf, sizeof pf);
  if (s->elem == 4)
    RDCNN_CUDA_TRY(cudaMemcpyAsync(s->d_params, &s->h_params_f, sizeof s->h_params_f, cudaMemcpyHostToDevice, s->stream));
  else
    RDCNN_CUDA_TRY(cudaMemcpyAsync(s->d_params, &s->h_params_d, sizeof s->h_params_d, cudaMemcpyHostToDevice, s->stream));
  s->params_stride = 0;
  s->unit_dv = true;  // the default gene has Dv = 1
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

void free_all(rdcnn_sim* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (int b = 0; b < 2; ++b)
    if (s->buf[b]) cudaFree(s->buf[b]);
  if (s->d_params) cudaFree(s->d_params);
  if (s->d_flags) cudaFree(s->d_flags);
  if (s->h_flags) cudaFreeHost(s->h_flags);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->comm) nccl().comm_destroy(s->comm);
  if (s->comm_stream) cudaStreamDestroy(s->comm_stream);
  if (s->ev_bnd) cudaEventDestroy(s->ev_bnd);
  if (s->ev_xchg) cudaEventDestroy(s->ev_xchg);
  for (void* p : s->ipc_opened) cudaIpcCloseMemHandle(p);
  if (s->p2p_words) cudaFree(s->p2p_words);
  if (s->d_first_bad) cudaFree(s->d_first_bad);
  for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);
  s->graphs.clear();
  if (s->ckpt) cudaFree(s->ckpt);
  if (s->frames) cudaFree(s->frames);
  if (s->d_stats) cudaFree(s->d_stats);
  if (s->d_counts) cudaFree(s->d_counts);
  if (s->d_digest) cudaFree(s->d_digest);
  if (s->d_scratch) cudaFree(s->d_scratch);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

// Drop a handle's captured graphs (their kernel parameters -- the shared
// gene, the segment plan -- no longer match the handle's).
void drop_graphs(rdcnn_sim* s) {
  for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);
  s->graphs.clear();
}

// Iterations between exact-blow-up checkpoints of slab advances (the first
// advance after the state is set always takes one).  RDCNN_CKPT_INTERVAL
// overrides (tests use 1 and small values).
long ckpt_interval() {
  static const long v = [] {
    const char* e = std::getenv("RDCNN_CKPT_INTERVAL");
    const long x = e ? std::atol(e) : 0;
    return x > 0 ? x : 2048L;
  }();
  return v;
}

// Sequence of block depths an advance of `steps` uses: floor(steps/Kmax)
// blocks of Kmax, then the remainder as descending powers of two.
struct Schedule {
  long full = 0;
  int kmax = 1;
  std::vector<int> tail;
  long count() const { return full + (long)tail.size(); }
  int depth(long n) const { return n < full ? kmax : tail[size_t(n - full)]; }
  long start(long n) const {
    if (n < full) return n * kmax;
    long it = full * kmax;
    for (long t = 0; t < n - full; ++t) it += tail[size_t(t)];
    return it;
  }
};

Schedule make_schedule(long steps, int kmax) {
  Schedule s;
  s.kmax = kmax;
  s.full = steps / kmax;
  long rem = steps - s.full * kmax;
  for (int k = kmax / 2; k >= 1; k /= 2)
    while (rem >= k) {
      s.tail.push_back(k);
      rem -= k;
    }
  return s;
}

// Re-runs one block of grid g level by level from its preserved input to
// find the first non-finite iteration.  Leaves the post-blow-up state in
// buffer `final_buf`.  Returns the 1-based level (1..k) in *level_out.
template <class T>
int replay_grid(rdcnn_sim* s, int g, int in_buf, int k, int final_buf, int* level_out) {
  // Level by level with the reference-order instance (kStrictDiv2U, not the
  // fused-v-tail one): the same first bad level either way (fhn_stencil.cuh
  // kStrictDiv2UF), and the state it leaves is the reference's own
  // post-blow-up state (non-finite exactly where the reference's is).
  struct Guard {
    rdcnn_sim* s;
    ~Guard() { s->replaying = false; }
  } guard{s};
  s->replaying = true;
  unsigned* scratch = s->d_flags + s->batch;
  int a_buf = in_buf;
  const size_t off = (size_t)g * (size_t)s->grid_stride;
  for (int m = 1; m <= k; ++m) {
    RDCNN_CUDA_TRY(cudaMemsetAsync(scratch, 0, sizeof(unsigned), s->stream));
    StepArgsT<T> a = base_args<T>(s, a_buf, a_buf ^ 1);
    a.u_in += off;
    a.v_in += off;
    a.u_out += off;
    a.v_out += off;
    a.batch = 1;
    a.params = static_cast<const ParamsT<T>*>(s->d_params) + (size_t)g * s->params_stride;
    a.flags = scratch;
    a.tag = 1;
    if (s->params_stride != 0) {
      // One grid: run it on the shared-gene instance with its own gene.
      RDCNN_CUDA_TRY(cudaMemcpyAsync(&a.shared, a.params, sizeof(ParamsT<T>), cudaMemcpyDeviceToHost, s->stream));
      RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
      a.params_stride = 0;
    }
    RDCNN_CUDA_TRY(launch_range<T>(s, 1, a, 0, s->rows, s->stream));
    unsigned hv = 0;
    RDCNN_CUDA_TRY(cudaMemcpyAsync(&hv, scratch, sizeof hv, cudaMemcpyDeviceToHost, s->stream));
    RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
    a_buf ^= 1;
    if (hv != 0) {
      if (a_buf != final_buf) {
        const size_t plane = (size_t)s->rows * s->cols * sizeof(T);
        RDCNN_CUDA_TRY(cudaMemcpyAsync(s->u_ptr<T>(final_buf) + off, s->u_ptr<T>(a_buf) + off, plane,
                                       cudaMemcpyDeviceToDevice, s->stream));
        RDCNN_CUDA_TRY(cudaMemcpyAsync(s->v_ptr<T>(final_buf) + off, s->v_ptr<T>(a_buf) + off, plane,
                                       cudaMemcpyDeviceToDevice, s->stream));
        RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
      }
      *level_out = m;
      return RDCNN_OK;
    }
  }
  return fail(RDCNN_ECUDA, "blow-up flagged for grid %d but not reproduced by replay", g);
}

// ---- persistent cluster path (small single lattices, fhn_cluster.cuh) -------

struct ClusterPlan {
  int C = 0, R = 0, W = 0, RW = 0;
  size_t smem = 0;
};

using ClusterFn = void (*)(rdcnn_dev::ClusterArgs);

// Arithmetic instance of the cluster kernel: fast, strict with the 2-op x/3
// and the unit-Dv product skipped when both gates hold, else the 3-op strict
// instance (kStrictDiv2 alone is not instantiated here: fewer kernels).
int cluster_arith(const rdcnn_sim* s) {
  const int a = arith_for<float>(s);
  return a == rdcnn_dev::kStrictDiv2 ? rdcnn_dev::kStrictArith
         : a == rdcnn_dev::kStrictDiv2UF ? rdcnn_dev::kStrictDiv2U  // per-step exact stop of its own
                                         : a;
}

template <int W, int RW>
ClusterFn cluster_fn_wr(int arith) {
  return arith == rdcnn_dev::kFastArith      ? &rdcnn_dev::fhn_cluster_kernel<W, RW, rdcnn_dev::kFastArith>
         : arith == rdcnn_dev::kStrictDiv2U ? &rdcnn_dev::fhn_cluster_kernel<W, RW, rdcnn_dev::kStrictDiv2U>
                                            : &rdcnn_dev::fhn_cluster_kernel<W, RW, rdcnn_dev::kStrictArith>;
}

ClusterFn cluster_fn(int w, int rw, int arith) {
  if (w == 4) return rw == 1 ? cluster_fn_wr<4, 1>(arith) : rw == 2 ? cluster_fn_wr<4, 2>(arith) : cluster_fn_wr<4, 4>(arith);
  return rw == 1 ? cluster_fn_wr<8, 1>(arith) : rw == 2 ? cluster_fn_wr<8, 2>(arith) : cluster_fn_wr<8, 4>(arith);
}

int cluster_max_warps(int rw) { return (rw >= 4 ? 256 : 512) / 32; }

// Rows per warp to try, best first (RDCNN_CLUSTER_RW pins one for tuning).
std::vector<int> cluster_rw_order() {
  if (const char* e = std::getenv("RDCNN_CLUSTER_RW")) {
    const int r = std::atoi(e);
    if (r == 1 || r == 2 || r == 4) return {r};
  }
  return {4, 2, 1};
}

// One cluster of C CTAs, each R = nw*RW rows (nw warps of RW rows), W =
// cols/32 columns per lane (4 or 8), the most CTAs per RW: every launchable
// plan, one per rows-per-warp candidate.  Empty when the shape does not fit
// or the device cannot host the cluster (then the wavefront kernel runs).
std::vector<ClusterPlan> cluster_plans(rdcnn_sim* s) {
  std::vector<ClusterPlan> plans;
  if (s->slab || s->batch != 1 || s->elem != 4 || s->params_stride != 0 || s->cluster_mode < 0) return plans;
  if (s->cols % 128 != 0) return plans;
  const int w = s->cols / 32;
  if (w != 4 && w != 8) return plans;
  const int arith = cluster_arith(s);
  for (int rw : cluster_rw_order()) {
    int C = 0;
    for (int c = rdcnn_dev::kClusterMax; c >= 1; --c)
      if (s->rows % c == 0 && (s->rows / c) % rw == 0 && s->rows / c / rw <= cluster_max_warps(rw)) {
        C = c;
        break;
      }
    if (C == 0) continue;
    ClusterPlan p;
    p.C = C;
    p.R = s->rows / C;
    p.W = w;
    p.RW = rw;
    p.smem = (size_t)(w == 4 ? rdcnn_dev::cluster_smem_bytes<4>(p.R) : rdcnn_dev::cluster_smem_bytes<8>(p.R));
    if (p.smem > 200 * 1024) continue;
    static int checked[2][5][4][rdcnn_dev::kClusterMax + 1] = {};  // 1 ok, -1 not launchable
    static std::mutex checked_mu;  // handles may plan concurrently from several host threads
    std::lock_guard<std::mutex> lock(checked_mu);
    int& ok = checked[w == 8][rw][arith][C];
    if (ok == 0) {
      ClusterFn fn = cluster_fn(w, rw, arith);
      ok = -1;
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)C);
        cfg.blockDim = dim3(32u * (unsigned)cluster_max_warps(rw));
        cfg.dynamicSmemBytes = 200 * 1024;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n >= 1) ok = 1;
      }
      cudaGetLastError();
    }
    if (ok != 1) continue;
    plans.push_back(p);
  }
  return plans;
}

int cluster_advance(rdcnn_sim* s, const ClusterPlan& pl, long steps, long* first_bad, bool* fell_back) {
  *fell_back = false;
  if (!s->d_first_bad) RDCNN_CUDA_TRY(cudaMalloc(&s->d_first_bad, sizeof(long long)));
  rdcnn_dev::ClusterArgs a{};
  a.u_in = s->u_ptr<float>(s->cur);
  a.v_in = s->v_ptr<float>(s->cur);
  a.u_out = s->u_ptr<float>(s->cur ^ 1);
  a.v_out = s->v_ptr<float>(s->cur ^ 1);
  a.rows = s->rows;
  a.cols = s->cols;
  a.R = pl.R;
  a.steps = steps;
  a.p = s->h_params_f;
  a.first_bad = s->d_first_bad;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pl.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)pl.C);
  cfg.blockDim = dim3(32u * (unsigned)(pl.R / pl.RW));
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ClusterFn fn = cluster_fn(pl.W, pl.RW, cluster_arith(s));
  RDCNN_CUDA_TRY(cudaMemsetAsync(s->d_first_bad, 0xFF, sizeof(long long), s->stream));
  RDCNN_CUDA_TRY(cudaEventRecord(s->ev0, s->stream));
  {
    const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
    if (e != cudaSuccess) {
      // The 16-CTA cluster could not be placed right now (e.g. SMs held by
      // another context).  In automatic mode the wavefront path takes over;
      // the state is untouched (the launch did not happen).
      cudaGetLastError();
      if (s->cluster_mode == 0) {
        *fell_back = true;
        return RDCNN_OK;
      }
      return fail(RDCNN_ECUDA, "cluster launch failed: %s", cudaGetErrorString(e));
    }
  }
  RDCNN_CUDA_TRY(cudaEventRecord(s->ev1, s->stream));
  long long fb = 0;
  RDCNN_CUDA_TRY(cudaMemcpyAsync(&fb, s->d_first_bad, sizeof fb, cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  float ms = 0;
  RDCNN_CUDA_TRY(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  s->last_ms = ms;
  s->launches = 1;
  if (fb > 0 && fb <= steps) {
    // Re-run exactly fb steps from the untouched input (cur): the output is
    // the state right after the first non-finite step.
    a.steps = fb;
    RDCNN_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, a));
    RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->launches = 2;
  } else {
    fb = 0;
  }
  s->cur ^= 1;
  if (first_bad) first_bad[0] = (long)fb;
  if (fb) return fail(RDCNN_EBLOWUP, "blow-up: non-finite state");
  return RDCNN_OK;
}

// Autotuned segment height for lattices that cannot fill the chip.  Their
// launches are latency-bound and the best height depends on how the warps
// spread over the SMs' schedulers (512^2: 6 rows run 25 % faster than the
// plan's 8), which no simple model captures.  Segmentation never changes
// the arithmetic, so the first long advance times a few candidate heights on
// its OWN first blocks (3 blocks each, CUDA events) and keeps the fastest
// per level count; no extra work is done.  An explicit seg_rows disables it.
// The result is kept process-wide per launch shape, so later handles of the
// same shape (bench reps, sweep chunks, per-call step handles) reuse it.
using TuneKey = std::tuple<int, int, int, int, int, int, int, int>;  // device, rows, cols, batch, elem, mode, per-grid, K
std::mutex g_tune_mu;
std::map<TuneKey, int> g_tune_cache;

template <class T>
int autotune_segments(rdcnn_sim* s, const Schedule& sched, long* n_io) {
  const int k = sched.kmax;
  const int ki = k_index(k);
  static const bool off = [] {
    const char* e = std::getenv("RDCNN_AUTOTUNE");
    return e && e[0] == '0';
  }();
  if (off || s->slab || s->seg_rows > 0 || s->tuned[ki]) return RDCNN_OK;
  const int w = width_for<T>(s);
  const bool per_grid = s->params_stride != 0, wrap = s->cols / w == 32;
  const int rw = resident_blocks<T>(k, w, arith_for<T>(s), per_grid, wrap) * (kThreads / 32);
  const Plan p0 = make_plan(s->cols, w, k, s->batch, 0, s->rows, 0, s->sm_count, rw);
  if (4 * p0.warps >= 3LL * rw * s->sm_count) {  // fills the chip: the plan is right
    s->tuned[ki] = true;
    return RDCNN_OK;
  }
  const TuneKey key{s->device, s->rows, s->cols, s->batch, s->elem, s->mode, int(per_grid), k};
  {
    std::lock_guard<std::mutex> lock(g_tune_mu);
    const auto it = g_tune_cache.find(key);
    if (it != g_tune_cache.end()) {
      s->tuned_seg[ki] = it->second;
      s->tuned[ki] = true;
      return RDCNN_OK;
    }
  }
  static const int kCand[] = {0, 3, 4, 5, 6, 8, 10, 12, 16, 24};
  constexpr int kReps = 3;
  std::vector<int> cand;
  for (int h : kCand)
    if (h <= s->rows) cand.push_back(h);
  if (sched.full < (long)(cand.size() * kReps) + 8) return RDCNN_OK;  // too short to tune on
  std::vector<cudaEvent_t> ev(cand.size() + 1);
  for (auto& e : ev) RDCNN_CUDA_TRY(cudaEventCreate(&e));
  long n = *n_io;
  for (size_t c = 0; c < cand.size(); ++c) {
    s->seg_force = cand[c];  // 0: the default plan
    RDCNN_CUDA_TRY(cudaEventRecord(ev[c], s->stream));
    for (int r = 0; r < kReps; ++r, ++n) {
      StepArgsT<T> a = base_args<T>(s, s->cur, s->cur ^ 1);
      a.tag = (unsigned)(n + 1);
      const int saved = s->tuned_seg[ki];
      s->tuned_seg[ki] = 0;
      const cudaError_t e = launch_range<T>(s, k, a, 0, s->rows, s->stream);
      s->tuned_seg[ki] = saved;
      if (e != cudaSuccess) {
        s->seg_force = 0;
        return fail(RDCNN_ECUDA, "autotune launch failed: %s", cudaGetErrorString(e));
      }
      s->cur ^= 1;
    }
  }
  s->seg_force = 0;
  RDCNN_CUDA_TRY(cudaEventRecord(ev.back(), s->stream));
  RDCNN_CUDA_TRY(cudaEventSynchronize(ev.back()));
  float best = 1e30f;
  int best_h = 0;
  for (size_t c = 0; c < cand.size(); ++c) {
    float ms = 0;
    RDCNN_CUDA_TRY(cudaEventElapsedTime(&ms, ev[c], ev[c + 1]));
    if (ms < best * 0.98f) {  // prefer the default plan unless clearly faster
      best = ms;
      best_h = cand[c];
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  s->tuned_seg[ki] = best_h;
  s->tuned[ki] = true;
  drop_graphs(s);  // any earlier capture used the untuned plan
  {
    std::lock_guard<std::mutex> lock(g_tune_mu);
    g_tune_cache.emplace(key, best_h);
  }
  *n_io = n;
  return RDCNN_OK;
}

// CUDA graphs for the per-launch path: the launch loop of an advance is
// captured once (its PDL edges become programmatic graph edges) and replayed
// on later advances of the same length.  Measured: 512^2 128k -> 153-166k,
// 1024^2 341k -> 402k, 2048^2 637k -> 649k, 4096^2 835k -> 840k
// Mcell-updates/s, bit-identical.  Used for launches that do not fill the
// chip (latency-bound lattices, where the gain is); chip-filling ones gain
// < 1 %, less than a capture costs a short-lived handle (a sweep's).
// RDCNN_GRAPH=0 turns it off.
bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RDCNN_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class T>
int advance_launches(rdcnn_sim* s, long steps, long* first_bad) {
  s->launches = 0;
  if (first_bad)
    for (int g = 0; g < s->batch; ++g) first_bad[g] = 0;
  RDCNN_CUDA_TRY(cudaMemsetAsync(s->d_flags, 0, sizeof(unsigned) * (size_t)s->batch, s->stream));
  const Schedule sched = make_schedule(steps, s->max_levels);
  const int cur0 = s->cur;
  RDCNN_CUDA_TRY(cudaEventRecord(s->ev0, s->stream));
  const long nl = sched.count();
  long n = 0;
  RDCNN_TRY(autotune_segments<T>(s, sched, &n));
  bool graph = graphs_enabled() && n == 0 && nl >= 8;
  if (graph) {  // only for launches that leave warp slots empty (same rule as the autotuner)
    const int k = sched.kmax, w = width_for<T>(s);
    const bool per_grid = s->params_stride != 0, wrap = s->cols / w == 32;
    const int rw = resident_blocks<T>(k, w, arith_for<T>(s), per_grid, wrap) * (kThreads / 32);
    const Plan p0 = make_plan(s->cols, w, k, s->batch, 0, s->rows, 0, s->sm_count, rw);
    graph = 4 * p0.warps < 3LL * rw * s->sm_count;
  }
  if (graph) {
    const std::pair<long, int> key{steps, cur0};
    auto it = s->graphs.find(key);
    if (it == s->graphs.end()) {
      if (s->graphs.size() >= 8) drop_graphs(s);  // bounded: a few advance lengths per handle
      // Capture; on any failure end the capture and take the direct path.
      cudaError_t ce = cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal);
      int cur = s->cur;
      for (long m = 0; m < nl && ce == cudaSuccess; ++m) {
        StepArgsT<T> a = base_args<T>(s, cur, cur ^ 1);
        a.tag = (unsigned)(m + 1);
        ce = launch_range<T>(s, sched.depth(m), a, 0, s->rows, s->stream);
        cur ^= 1;
      }
      cudaGraph_t g = nullptr;
      const cudaError_t ee = cudaStreamEndCapture(s->stream, &g);
      cudaGraphExec_t ge = nullptr;
      if (ce == cudaSuccess && ee == cudaSuccess) ce = cudaGraphInstantiate(&ge, g, 0);
      if (g) cudaGraphDestroy(g);
      if (ce == cudaSuccess && ee == cudaSuccess) {
        it = s->graphs.emplace(key, ge).first;
      } else {
        cudaGetLastError();
        graph = false;
      }
      s->launches = 0;
      RDCNN_CUDA_TRY(cudaEventRecord(s->ev0, s->stream));  // time the replay, not the capture
    }
    if (graph) {
      RDCNN_CUDA_TRY(cudaGraphLaunch(it->second, s->stream));
      s->launches = nl;  // the graph's kernel nodes
      if (nl & 1) s->cur ^= 1;
      n = nl;
    }
  }
  for (; n < nl; ++n) {
    StepArgsT<T> a = base_args<T>(s, s->cur, s->cur ^ 1);
    a.tag = (unsigned)(n + 1);
    RDCNN_CUDA_TRY(launch_range<T>(s, sched.depth(n), a, 0, s->rows, s->stream));
    s->cur ^= 1;
  }
  RDCNN_CUDA_TRY(cudaEventRecord(s->ev1, s->stream));
  RDCNN_CUDA_TRY(cudaMemcpyAsync(s->h_flags, s->d_flags, sizeof(unsigned) * (size_t)s->batch,
                                 cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  float ms = 0;
  RDCNN_CUDA_TRY(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  s->last_ms = ms;
  bool any = false;
  for (int g = 0; g < s->batch; ++g) {
    const unsigned tag = s->h_flags[g];
    if (tag == 0) continue;
    any = true;
    const long n = (long)tag - 1;
    const int in_buf = cur0 ^ int(n & 1);
    int level = 0;
    RDCNN_TRY(replay_grid<T>(s, g, in_buf, sched.depth(n), s->cur, &level));
    if (first_bad) first_bad[g] = sched.start(n) + level;
  }
  if (any) return fail(RDCNN_EBLOWUP, "blow-up: non-finite state");
  return RDCNN_OK;
}

// Rows per warp of the cluster kernel: more rows per warp amortise the
// per-step exchange, more warps hide latency, and the best trade depends on
// the shape (256^2: RW=4 72k vs RW=1 61k Mcell-updates/s; 128^2: RW=1 41k
// vs RW=4 32k).  So the first long advance of a shape runs kTrial steps on
// each candidate -- real progress of the advance, timed by its CUDA events
// -- and the fastest is kept process-wide; later advances use it directly.
using ClusterKey = std::tuple<int, int, int, int>;  // device, rows, cols, mode
std::mutex g_cluster_mu;
std::map<ClusterKey, int> g_cluster_rw;

int cluster_advance_tuned(rdcnn_sim* s, const std::vector<ClusterPlan>& plans, long steps, long* first_bad,
                          bool* fell_back) {
  constexpr long kTrial = 128;
  const ClusterKey key{s->device, s->rows, s->cols, s->mode};
  int rw = 0;
  {
    std::lock_guard<std::mutex> lock(g_cluster_mu);
    const auto it = g_cluster_rw.find(key);
    if (it != g_cluster_rw.end()) rw = it->second;
  }
  auto plan_of = [&](int r) {
    for (const ClusterPlan& p : plans)
      if (p.RW == r) return p;
    return plans[0];
  };
  if (rw != 0 || plans.size() == 1 || steps < (long)(plans.size() + 1) * kTrial)
    return cluster_advance(s, rw ? plan_of(rw) : plans[0], steps, first_bad, fell_back);

  long done = 0, launches = 0;
  double ms = 0;
  float best = 1e30f;
  int best_rw = plans[0].RW;
  bool all_ran = true;
  for (const ClusterPlan& p : plans) {
    long fb = 0;
    const int rc = cluster_advance(s, p, kTrial, &fb, fell_back);
    if (*fell_back) {  // this candidate could not be placed right now
      *fell_back = false;
      all_ran = false;
      continue;
    }
    ms += s->last_ms;
    launches += s->launches;
    if (rc != RDCNN_OK) {  // blow-up inside a trial: exact, and the advance ends there
      if (rc == RDCNN_EBLOWUP && first_bad) first_bad[0] = done + fb;
      s->last_ms = ms;
      s->launches = launches;
      return rc;
    }
    done += kTrial;
    if (s->last_ms < best) {
      best = s->last_ms;
      best_rw = p.RW;
    }
  }
  if (done == 0) {  // no candidate could be placed: the wavefront path runs the whole advance
    *fell_back = true;
    return RDCNN_OK;
  }
  if (all_ran) {
    std::lock_guard<std::mutex> lock(g_cluster_mu);
    g_cluster_rw.emplace(key, best_rw);
  }
  long fb = 0;
  int rc = cluster_advance(s, plan_of(best_rw), steps - done, &fb, fell_back);
  if (*fell_back) {  // finish on the wavefront path
    *fell_back = false;
    rc = advance_launches<float>(s, steps - done, &fb);
  }
  s->last_ms += ms;
  s->launches += launches;
  if (first_bad) first_bad[0] = fb ? done + fb : 0;
  return rc;
}

template <class T>
int advance_impl(rdcnn_sim* s, long steps, long* first_bad) {
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  if constexpr (sizeof(T) == 4) {
    const std::vector<ClusterPlan> plans = steps > 0 ? cluster_plans(s) : std::vector<ClusterPlan>{};
    if (!plans.empty()) {
      bool fell_back = false;
      const int rc = cluster_advance_tuned(s, plans, steps, first_bad, &fell_back);
      if (!fell_back) return rc;
    }
    if (s->cluster_mode > 0) return fail(RDCNN_EINVAL, "persistent cluster path required but %dx%d (batch %d) does not fit it",
                                         s->rows, s->cols, s->batch);
  }
  return advance_launches<T>(s, steps, first_bad);
}

// Device-to-host copies into pageable memory that was never written (a
// fresh numpy/malloc buffer) spend most of their time in the page faults of
// the single copying thread: 268 MB took 55-66 ms against 13 ms into touched
// pages (tools/download_timing.py).  Large pageable destinations are
// therefore faulted in first by several threads (one store per page; the
// copy overwrites every byte anyway).  Pinned destinations are left alone.
void prefault_pageable(void* dst, size_t bytes) {
  if (bytes < (32u << 20)) return;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, dst) == cudaSuccess && at.type != cudaMemoryTypeUnregistered) return;
  cudaGetLastError();
  const long page = sysconf(_SC_PAGESIZE) > 0 ? sysconf(_SC_PAGESIZE) : 4096;
  const unsigned hw = std::thread::hardware_concurrency();
  const unsigned nt = std::max(1u, std::min(16u, hw ? hw : 1u));
  const size_t slice = (bytes / nt + (size_t)page - 1) / (size_t)page * (size_t)page;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) {
    const size_t lo = (size_t)t * slice;
    if (lo >= bytes) break;
    const size_t hi = std::min(bytes, lo + slice);
    th.emplace_back([=] {
      volatile char* p = static_cast<char*>(dst);
      for (size_t i = lo; i < hi; i += (size_t)page) p[i] = 0;
    });
  }
  for (auto& t : th) t.join();
}

int copy_state(rdcnn_sim* s, void* u, void* v, bool upload) {
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  if (upload) s->ckpt_age = -1;  // the checkpoint no longer precedes the state
  const size_t e = (size_t)s->elem;
  char* du = static_cast<char*>(s->buf[s->cur]);
  char* dv = du + (s->slab ? (size_t)s->plane_off * e : (size_t)s->rows * s->cols * s->batch * e);
  if (!s->slab) {
    const size_t bytes = (size_t)s->rows * s->cols * s->batch * e;
    const cudaMemcpyKind kind = upload ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    if (!upload) {
      prefault_pageable(u, bytes);
      prefault_pageable(v, bytes);
    }
    RDCNN_CUDA_TRY(cudaMemcpyAsync(upload ? (void*)du : u, upload ? u : (void*)du, bytes, kind, s->stream));
    RDCNN_CUDA_TRY(cudaMemcpyAsync(upload ? (void*)dv : v, upload ? v : (void*)dv, bytes, kind, s->stream));
  } else {
    // Slab phases run on caller streams: drain them before touching the state.
    RDCNN_CUDA_TRY(cudaDeviceSynchronize());
    const size_t row0 = (size_t)s->ghost * s->pitch * e;
    const size_t dpitch = (size_t)s->pitch * e, w = (size_t)s->cols * e;
    if (upload) {
      RDCNN_CUDA_TRY(cudaMemcpy2DAsync(du + row0, dpitch, u, w, w, s->rows, cudaMemcpyHostToDevice, s->stream));
      RDCNN_CUDA_TRY(cudaMemcpy2DAsync(dv + row0, dpitch, v, w, w, s->rows, cudaMemcpyHostToDevice, s->stream));
    } else {
      prefault_pageable(u, w * (size_t)s->rows);
      prefault_pageable(v, w * (size_t)s->rows);
      RDCNN_CUDA_TRY(cudaMemcpy2DAsync(u, w, du + row0, dpitch, w, s->rows, cudaMemcpyDeviceToHost, s->stream));
      RDCNN_CUDA_TRY(cudaMemcpy2DAsync(v, w, dv + row0, dpitch, w, s->rows, cudaMemcpyDeviceToHost, s->stream));
    }
  }
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

// Tensor maps of the two state buffers for TMA staging (RDCNN_BULK=2
// builds): {cols, rows x batch, 2 planes} fp32 with a {128, 1, 2} box, i.e.
// one 32-lane band row of both planes.  Periodic fp32 handles whose rows
// hold at least one band; the driver entry point is resolved at run time.
int make_tensor_maps(rdcnn_sim* s) {
  if (s->slab || s->cols % 4 != 0 || s->cols < 128) return RDCNN_OK;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return fail(RDCNN_ECUDA, "cuTensorMapEncodeTiled unavailable");
  for (int b = 0; b < 2; ++b) {
    const cuuint64_t dims[3] = {(cuuint64_t)s->cols, (cuuint64_t)s->rows * (cuuint64_t)s->batch, 2};
    const cuuint64_t strides[2] = {(cuuint64_t)s->pitch * 4,
                                   (cuuint64_t)((char*)s->v_ptr<float>(b) - (char*)s->u_ptr<float>(b))};
    const cuuint32_t box[3] = {128, 1, 2};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap* m = reinterpret_cast<CUtensorMap*>(s->tmap[b]);
    const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, s->u_ptr<float>(b), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(RDCNN_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  }
  s->tma_ok = true;
  return RDCNN_OK;
}

int create_impl(int rows, int cols, int batch, int device, int mode, int elem, rdcnn_sim_t* out) {
  if (!out) return fail(RDCNN_EINVAL, "null output handle");
  *out = nullptr;
  if (rows < 3 || cols < 3) return fail(RDCNN_EINVAL, "grid must be at least 3x3, got %dx%d", rows, cols);
  if (batch < 1) return fail(RDCNN_EINVAL, "batch must be >= 1, got %d", batch);
  if (mode != RDCNN_STRICT && mode != RDCNN_FAST) return fail(RDCNN_EINVAL, "unknown mode %d", mode);
  if (elem != 4 && elem != 8) return fail(RDCNN_EINVAL, "element size must be 4 or 8 bytes, got %d", elem);
  if (elem == 8 && mode == RDCNN_FAST) return fail(RDCNN_EINVAL, "fast mode is fp32 only");
  auto* s = new (std::nothrow) rdcnn_sim();
  if (!s) return fail(RDCNN_EINVAL, "out of host memory");
  s->rows = rows;
  s->cols = cols;
  s->batch = batch;
  s->device = device;
  s->mode = mode;
  s->elem = elem;
  s->pitch = cols;
  s->grid_stride = (long long)rows * cols;
  s->buf_elems = (size_t)rows * cols * batch * 2;
  s->max_levels = 4;
  int rc = alloc_common(s);
  if (rc == RDCNN_OK && RDCNN_BULK == 2 && elem == 4) rc = make_tensor_maps(s);
  if (rc != RDCNN_OK) {
    std::string msg = g_last_error;
    free_all(s);
    g_last_error = msg;
    return rc;
  }
  *out = s;
  return RDCNN_OK;
}

template <class T>
int init_impl(rdcnn_sim* s, int typ, uint64_t seed, int global_rows, int row_offset) {
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  const size_t row0 = s->slab ? (size_t)s->ghost * s->pitch : 0;
  init_kernel<T><<<4 * s->sm_count, 256, 0, s->stream>>>(
      s->u_ptr<T>(s->cur) + row0, s->v_ptr<T>(s->cur) + row0, s->pitch, s->grid_stride,
      s->slab ? 1 : s->batch, s->rows, s->cols, global_rows, row_offset, typ, seed);
  RDCNN_CUDA_TRY(cudaGetLastError());
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->ckpt_age = -1;  // the checkpoint no longer precedes the state
  return RDCNN_OK;
}

// Device staging kept with the handle (stream-ordered malloc/free per call
// made short calls' wall time vary by two orders of magnitude).  The caller
// synchronises the handle's stream before returning, so the next call may
// reuse the bytes.
int scratch(rdcnn_sim* s, size_t bytes, void** out) {
  if (s->scratch_bytes < bytes) {
    if (s->d_scratch) RDCNN_CUDA_TRY(cudaFree(s->d_scratch));
    s->d_scratch = nullptr;
    s->scratch_bytes = 0;
    RDCNN_CUDA_TRY(cudaMalloc(&s->d_scratch, bytes));
    s->scratch_bytes = bytes;
  }
  *out = s->d_scratch;
  return RDCNN_OK;
}

template <class T>
int image_impl(rdcnn_sim* s, const uint8_t* px, double ka) {
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  T lut[256];
  const T k = (T)ka;
  for (int p = 0; p < 256; ++p) lut[p] = k * (T)(p / 255.0);  // init.hpp:58, image.hpp:283
  const size_t n = (size_t)s->rows * s->cols;
  void* buf = nullptr;
  const size_t lut_off = (n + 255) / 256 * 256;
  RDCNN_TRY(scratch(s, lut_off + sizeof lut, &buf));
  uint8_t* d_px = static_cast<uint8_t*>(buf);
  T* d_lut = reinterpret_cast<T*>(static_cast<uint8_t*>(buf) + lut_off);
  RDCNN_CUDA_TRY(cudaMemcpyAsync(d_px, px, n, cudaMemcpyHostToDevice, s->stream));
  RDCNN_CUDA_TRY(cudaMemcpyAsync(d_lut, lut, sizeof lut, cudaMemcpyHostToDevice, s->stream));
  image_kernel<T><<<4 * s->sm_count, 256, 0, s->stream>>>(s->u_ptr<T>(s->cur), s->v_ptr<T>(s->cur),
                                                           s->pitch, s->grid_stride, s->batch,
                                                           s->rows, s->cols, d_px, d_lut);
  RDCNN_CUDA_TRY(cudaGetLastError());
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

template <class T>
int set_params_impl(rdcnn_sim* s, const ParamsT<T>* p, int n) {
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  RDCNN_CUDA_TRY(cudaMemcpyAsync(s->d_params, p, sizeof(ParamsT<T>) * (size_t)n, cudaMemcpyHostToDevice, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  // Captured launches carry the shared gene (and the arithmetic instance it
  // selects) by value: they survive only an identical shared gene.
  const bool same = n == 1 && s->params_stride == 0 &&
                    std::memcmp(&s->shared_params<T>(), p, sizeof(ParamsT<T>)) == 0;
  s->params_stride = (n == 1) ? 0 : 1;
  s->div2_ok = div2_gate<T>(p, n);
  s->unit_dv = unit_dv_gate<T>(p, n);
  if (n == 1) {
    if constexpr (sizeof(T) == 4) s->h_params_f = *p;
    else s->h_params_d = *p;
  }
  if (!same) drop_graphs(s);
  return RDCNN_OK;
}

template <class T>
int slab_step_impl(rdcnn_sim* s, int k, cudaStream_t st, bool boundary) {
  StepArgsT<T> a = base_args<T>(s, s->cur, s->cur ^ 1);
  if (boundary) ++s->slab_tag;
  a.tag = s->slab_tag;
  const int gh = s->ghost;
  if (boundary) {
    RDCNN_CUDA_TRY(launch_range<T>(s, k, a, 0, gh, st));
    RDCNN_CUDA_TRY(launch_range<T>(s, k, a, s->rows - gh, s->rows, st));
  } else {
    RDCNN_CUDA_TRY(launch_range<T>(s, k, a, gh, s->rows - gh, st));
  }
  return RDCNN_OK;
}

// One block of the fused peer ring (rdcnn_slab_attach_peers): every owned row
// in ONE launch of the kPeer instance, which also stores the edge rows into
// the neighbours' ghost rows of the output buffer and signals them.  Stream
// order alone covers the local dependencies (block n+1 reads what block n
// wrote); the cross-rank ones are the in-kernel ready words.
// The band/segment plan of one fused peer-ring block (every owned row).
Plan peer_plan(rdcnn_sim* s, int k, bool tee) {
  const int w = width_for<float>(s);
  const bool wrap = s->cols / w == 32;
  const int rw = peer_resident_blocks(k, w, arith_for<float>(s), wrap, tee) * (kThreads / 32);
  return make_plan(s->cols, w, k, 1, 0, s->rows, s->seg_rows, s->sm_count, rw);
}

int peer_block(rdcnn_sim* s, int k, unsigned tag, cudaStream_t st, float* tee = nullptr,
               unsigned long long* trace = nullptr) {
  StepArgsT<float> a = base_args<float>(s, s->cur, s->cur ^ 1);
  a.tag = tag;
  a.tee_u = tee;
  a.trace = trace;
  a.trace_stride = 5;
  const int ib = s->cur;  // the neighbours' INPUT buffers (all ranks run the same blocks)
  const size_t pitch = (size_t)s->pitch;
  a.peer_top = static_cast<const float*>(s->peer_buf[0][ib]) + (size_t)(s->ghost + s->peer_rows[0]) * pitch;
  a.peer_bot = static_cast<const float*>(s->peer_buf[1][ib]) + (size_t)s->ghost * pitch;
  a.edge_count = s->p2p_words + 2;
  a.sig_prev = s->peer_words[0] + 1;
  a.sig_next = s->peer_words[1] + 0;
  a.ready = s->p2p_words;
  a.seq = s->p2p_seq;
  const int w = width_for<float>(s);
  const int arith = arith_for<float>(s);
  const bool wrap = s->cols / w == 32;
  const int rw = peer_resident_blocks(k, w, arith, wrap, tee != nullptr) * (kThreads / 32);
  const Plan p = peer_plan(s, k, tee != nullptr);
  a.row_begin = 0;
  a.row_end = s->rows;
  a.seg_rows = p.seg_rows;
  a.n_segs = p.n_segs;
  a.n_bands = p.n_bands;
  a.band_groups = p.band_groups;
  a.halo_groups = p.halo;
  const int h = p.seg_rows, S = s->rows, g = s->ghost;
  a.n_top = p.n_bands * std::min(p.n_segs, (g + h - 1) / h);  // segments with r0 < g
  a.n_bot = p.n_bands * (p.n_segs - (S - g) / h);             // segments with r0 + h > S - g
  auto fn = peer_table().fn[w > 1][k_index(k)][arith][wrap][tee != nullptr];
  RDCNN_CUDA_TRY(launch_pdl(fn, (unsigned)p.warps, smem_for<float>(w), st, a, 4 * p.warps >= 3LL * rw * s->sm_count));
  ++s->launches;
  ++s->p2p_seq;
  s->cur ^= 1;
  return RDCNN_OK;
}

int need_elem(rdcnn_sim* s, int elem) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (s->elem != elem)
    return fail(RDCNN_EINVAL, "handle holds fp%d values; this entry point is fp%d", 8 * s->elem, 8 * elem);
  return RDCNN_OK;
}

template <class T>
void host_unit(uint64_t& st, T& x) {
  uint64_t z = (st += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  if constexpr (sizeof(T) == 4) x = (float)(z >> 40) * 0x1.0p-24f;
  else x = (double)(z >> 11) * 0x1.0p-53;
}

template <class T>
int host_full_random(int rows, int cols, uint64_t seed, T* u, T* v) {
  if (rows < 3 || cols < 3 || !u || !v) return fail(RDCNN_EINVAL, "bad arguments");
  uint64_t st = seed;
  const size_t n = (size_t)rows * cols;
  for (size_t k = 0; k < n; ++k) host_unit(st, u[k]);
  for (size_t k = 0; k < n; ++k) host_unit(st, v[k]);
  return RDCNN_OK;
}

template <class T>
int host_center_square(int rows, int cols, uint64_t seed, T* u, T* v) {
  if (rows < 11 || cols < 11 || !u || !v)
    return fail(RDCNN_EINVAL, "typ=1 needs a grid of at least 11x11, got %dx%d", rows, cols);
  const size_t n = (size_t)rows * cols;
  std::fill(u, u + n, T(0));
  std::fill(v, v + n, T(0));
  const int i0 = (rows - 11) / 2, j0 = (cols - 11) / 2;
  uint64_t st = seed;
  for (T* plane : {u, v})
    for (int i = i0; i < i0 + 11; ++i)
      for (int j = j0; j < j0 + 11; ++j) host_unit(st, plane[(size_t)i * cols + j]);
  return RDCNN_OK;
}

// normalize_frame / normalize_frame_fixed (frame.hpp:28-66): lround of
// (x - lo) * (255 / (hi - lo)) in double, clamped to 0..255; 128 when hi <= lo.
template <class T>
__global__ void normalize_kernel(const T* __restrict__ x, long long n, double lo, double hi,
                                 uint8_t* __restrict__ out) {
  const bool flat = !(hi > lo);
  const double scale = flat ? 0.0 : 255.0 / (hi - lo);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (flat) {
      out[i] = 128;
    } else {
      long long p = llround(__dmul_rn(__dsub_rn((double)x[i], lo), scale));
      out[i] = (uint8_t)(p < 0 ? 0 : (p > 255 ? 255 : p));
    }
  }
}

// Whole-device min/max of one plane for normalize_frame (frame.hpp:28-44):
// values are exact in double, so the order of the reduction does not matter;
// each block folds its grid-stride share with shuffles and one atomic pair on
// order-preserving 64-bit keys of the doubles.
__device__ __forceinline__ unsigned long long order_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double key_value(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double x;
  std::memcpy(&x, &b, sizeof x);
  return x;
}

template <class T>
__global__ void minmax_kernel(const T* __restrict__ x, long long n, unsigned long long* __restrict__ keys) {
  double mn = INFINITY, mx = -INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = (double)x[i];
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(keys, order_key(mn));
    atomicMax(keys + 1, order_key(mx));
  }
}

template <class T>
int normalize_impl(rdcnn_sim* s, const void* src_dev, double lo, double hi, uint8_t* out);

template <class T>
int normalize_auto_impl(rdcnn_sim* s, const void* src_dev, uint8_t* out, double* lo_out, double* hi_out) {
  const long long n = (long long)s->rows * s->cols;
  void* buf = nullptr;
  const size_t key_off = ((size_t)n + 255) / 256 * 256;
  RDCNN_TRY(scratch(s, key_off + 2 * sizeof(unsigned long long), &buf));
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(static_cast<char*>(buf) + key_off);
  const unsigned long long init[2] = {~0ull, 0ull};
  RDCNN_CUDA_TRY(cudaMemcpyAsync(keys, init, sizeof init, cudaMemcpyHostToDevice, s->stream));
  minmax_kernel<T><<<4 * s->sm_count, 256, 0, s->stream>>>(static_cast<const T*>(src_dev), n, keys);
  RDCNN_CUDA_TRY(cudaGetLastError());
  unsigned long long k[2];
  RDCNN_CUDA_TRY(cudaMemcpyAsync(k, keys, sizeof k, cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  const double lo = key_value(k[0]), hi = key_value(k[1]);
  if (lo_out) *lo_out = lo;
  if (hi_out) *hi_out = hi;
  return normalize_impl<T>(s, src_dev, lo, hi, out);
}

template <class T>
int frame_stats_impl(rdcnn_sim* s, int slot, double* mn, double* mx, double* med) {
  const long long n = (long long)s->rows * s->cols;
  const T* base = static_cast<const T*>(s->frames) + (size_t)slot * s->batch * n;
  double* d = s->d_stats;
  rdcnn_dev::frame_stats_kernel<T><<<s->batch, rdcnn_dev::kStatThreads, 0, s->stream>>>(
      base, n, d, d + s->batch, d + 2 * s->batch);
  RDCNN_CUDA_TRY(cudaGetLastError());
  const size_t b = sizeof(double) * (size_t)s->batch;
  RDCNN_CUDA_TRY(cudaMemcpyAsync(mn, d, b, cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaMemcpyAsync(mx, d + s->batch, b, cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaMemcpyAsync(med, d + 2 * s->batch, b, cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

template <class T>
int frame_active_impl(rdcnn_sim* s, int slot, const double* med, const double* thr, long long* counts) {
  const long long n = (long long)s->rows * s->cols;
  const T* base = static_cast<const T*>(s->frames) + (size_t)slot * s->batch * n;
  double* d = s->d_stats;
  const size_t b = sizeof(double) * (size_t)s->batch;
  RDCNN_CUDA_TRY(cudaMemcpyAsync(d + 2 * s->batch, med, b, cudaMemcpyHostToDevice, s->stream));
  RDCNN_CUDA_TRY(cudaMemcpyAsync(d + 3 * s->batch, thr, b, cudaMemcpyHostToDevice, s->stream));
  rdcnn_dev::frame_active_kernel<T><<<s->batch, rdcnn_dev::kStatThreads, 0, s->stream>>>(
      base, n, d + 2 * s->batch, d + 3 * s->batch, s->d_counts);
  RDCNN_CUDA_TRY(cudaGetLastError());
  RDCNN_CUDA_TRY(cudaMemcpyAsync(counts, s->d_counts, sizeof(long long) * (size_t)s->batch,
                                 cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

template <class T>
int normalize_impl(rdcnn_sim* s, const void* src_dev, double lo, double hi, uint8_t* out) {
  const long long n = (long long)s->rows * s->cols;
  void* buf = nullptr;
  RDCNN_TRY(scratch(s, (size_t)n, &buf));
  uint8_t* d_out = static_cast<uint8_t*>(buf);
  normalize_kernel<T><<<4 * s->sm_count, 256, 0, s->stream>>>(static_cast<const T*>(src_dev), n, lo, hi, d_out);
  RDCNN_CUDA_TRY(cudaGetLastError());
  RDCNN_CUDA_TRY(cudaMemcpyAsync(out, d_out, (size_t)n, cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

// checksum / fnv1a (grid.hpp:100-126) of every grid of a batch on the device:
// one thread per grid, FNV-1a 64 over the raw bytes of its u plane then its v
// plane -- sequential within a grid, independent across grids.  The hash is
// a dependent chain (XOR, multiply) per byte, so the loads are software-
// pipelined kDepth x 16 bytes ahead: the next chunk is in flight while the
// current one is hashed (the 4096-grid cfg4 digest: 85 ms -> a few ms).
constexpr int kFnvDepth = 8;

__device__ __forceinline__ unsigned long long fnv_word(unsigned long long h, unsigned w) {
#pragma unroll
  for (int k = 0; k < 4; ++k) h = (h ^ ((w >> (8 * k)) & 0xFFu)) * 0x100000001b3ull;
  return h;
}

__global__ void fnv_batch_kernel(const unsigned char* __restrict__ u, const unsigned char* __restrict__ v,
                                 size_t plane_bytes, size_t grid_stride_bytes, int batch,
                                 unsigned long long* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= batch) return;
  unsigned long long h = 0xcbf29ce484222325ull;
  const size_t n16 = plane_bytes / 16;  // the caller guarantees plane_bytes % 16 == 0
  for (const unsigned char* plane : {u, v}) {
    const uint4* p = reinterpret_cast<const uint4*>(plane + (size_t)g * grid_stride_bytes);
    uint4 cur[kFnvDepth];
#pragma unroll
    for (int k = 0; k < kFnvDepth; ++k) cur[k] = (size_t)k < n16 ? __ldcs(p + k) : make_uint4(0, 0, 0, 0);
    for (size_t i = 0; i < n16; i += kFnvDepth) {
      uint4 nxt[kFnvDepth];
#pragma unroll
      for (int k = 0; k < kFnvDepth; ++k)
        nxt[k] = i + kFnvDepth + k < n16 ? __ldcs(p + i + kFnvDepth + k) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < kFnvDepth; ++k) {
        if (i + k < n16) {
          h = fnv_word(h, cur[k].x);
          h = fnv_word(h, cur[k].y);
          h = fnv_word(h, cur[k].z);
          h = fnv_word(h, cur[k].w);
        }
      }
#pragma unroll
      for (int k = 0; k < kFnvDepth; ++k) cur[k] = nxt[k];
    }
  }
  out[g] = h;
}

uint64_t fnv_planes(const void* u, const void* v, size_t bytes) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (const void* plane : {u, v}) {
    const unsigned char* p = static_cast<const unsigned char*>(plane);
    for (size_t i = 0; i < bytes; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  }
  return h;
}

}  // namespace

// ---------------------------------------------------------------------------
// Exported C-ABI.
// ---------------------------------------------------------------------------

extern "C" {

int rdcnn_abi_version(void) { return RDCNN_ABI_VERSION; }

const char* rdcnn_last_error(void) { return g_last_error.c_str(); }

int rdcnn_device_count(int* n) {
  if (!n) return fail(RDCNN_EINVAL, "null output");
  RDCNN_CUDA_TRY(cudaGetDeviceCount(n));
  return RDCNN_OK;
}

void rdcnn_params_from_gene(const double g[7], rdcnn_params_f32* out) {
  // model.hpp:24-32: T(g.x) for each field, kernel order.
  out->dt = (float)g[0];
  out->a = (float)g[1];
  out->b = (float)g[2];
  out->eps = (float)g[3];
  out->c = (float)g[4];
  out->du = (float)g[5];
  out->dv = (float)g[6];
}

int rdcnn_sim_create(int rows, int cols, int batch, int device, int mode, rdcnn_sim_t* out) {
  return create_impl(rows, cols, batch, device, mode, 4, out);
}

int rdcnn_sim_create_f64(int rows, int cols, int batch, int device, rdcnn_sim_t* out) {
  return create_impl(rows, cols, batch, device, RDCNN_STRICT, 8, out);
}

int rdcnn_sim_precision(rdcnn_sim_t s, int* bytes) {
  if (!s || !bytes) return fail(RDCNN_EINVAL, "null argument");
  *bytes = s->elem;
  return RDCNN_OK;
}

int rdcnn_slab_create(int rows, int cols, int ghost, int device, int mode, rdcnn_sim_t* out) {
  if (!out) return fail(RDCNN_EINVAL, "null output handle");
  *out = nullptr;
  if (cols < 3 || rows < 1) return fail(RDCNN_EINVAL, "bad slab shape %dx%d", rows, cols);
  if (ghost != 1 && ghost != 2 && ghost != 4 && ghost != 8)
    return fail(RDCNN_EINVAL, "ghost depth must be 1, 2, 4 or 8, got %d", ghost);
  if (rows < 2 * ghost) return fail(RDCNN_EINVAL, "slab rows %d < 2*ghost %d", rows, 2 * ghost);
  if (mode != RDCNN_STRICT && mode != RDCNN_FAST) return fail(RDCNN_EINVAL, "unknown mode %d", mode);
  auto* s = new (std::nothrow) rdcnn_sim();
  if (!s) return fail(RDCNN_EINVAL, "out of host memory");
  s->rows = rows;
  s->cols = cols;
  s->batch = 1;
  s->device = device;
  s->mode = mode;
  s->elem = 4;
  s->slab = true;
  s->ghost = ghost;
  s->pitch = 2 * cols;
  s->plane_off = cols;
  s->grid_stride = 0;
  s->buf_elems = (size_t)(rows + 2 * ghost) * 2 * cols;
  s->max_levels = ghost;
  int rc = alloc_common(s);
  if (rc != RDCNN_OK) {
    std::string msg = g_last_error;
    free_all(s);
    g_last_error = msg;
    return rc;
  }
  *out = s;  // buf[b] points at the first ghost row; owned row 0 is `ghost` rows below
  return RDCNN_OK;
}

void rdcnn_sim_destroy(rdcnn_sim_t s) { free_all(s); }

int rdcnn_sim_set_params(rdcnn_sim_t s, const rdcnn_params_f32* p, int n) {
  RDCNN_TRY(need_elem(s, 4));
  if (!p) return fail(RDCNN_EINVAL, "null argument");
  if (n != 1 && n != s->batch) return fail(RDCNN_EINVAL, "params count %d must be 1 or batch %d", n, s->batch);
  static_assert(sizeof(ParamsT<float>) == sizeof(rdcnn_params_f32), "layout");
  return set_params_impl<float>(s, reinterpret_cast<const ParamsT<float>*>(p), n);
}

int rdcnn_sim_set_params_f64(rdcnn_sim_t s, const rdcnn_params_f64* p, int n) {
  RDCNN_TRY(need_elem(s, 8));
  if (!p) return fail(RDCNN_EINVAL, "null argument");
  if (n != 1 && n != s->batch) return fail(RDCNN_EINVAL, "params count %d must be 1 or batch %d", n, s->batch);
  static_assert(sizeof(ParamsT<double>) == sizeof(rdcnn_params_f64), "layout");
  return set_params_impl<double>(s, reinterpret_cast<const ParamsT<double>*>(p), n);
}

int rdcnn_sim_set_tuning(rdcnn_sim_t s, int max_levels, int seg_rows) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (max_levels != 1 && max_levels != 2 && max_levels != 4 && max_levels != 8)
    return fail(RDCNN_EINVAL, "max_levels must be 1, 2, 4 or 8, got %d", max_levels);
  if (s->elem == 8 && max_levels > Traits<double>::kMaxLevels)
    return fail(RDCNN_EINVAL, "fp64 handles fuse at most %d levels", Traits<double>::kMaxLevels);
  if (s->slab && max_levels > s->ghost)
    return fail(RDCNN_EINVAL, "max_levels %d exceeds slab ghost depth %d", max_levels, s->ghost);
  if (seg_rows < 0) return fail(RDCNN_EINVAL, "seg_rows must be >= 0");
  s->max_levels = max_levels;
  s->seg_rows = seg_rows;
  for (int i = 0; i < 4; ++i) {
    s->tuned[i] = false;
    s->tuned_seg[i] = 0;
  }
  drop_graphs(s);
  return RDCNN_OK;
}

int rdcnn_sim_trace_launch(rdcnn_sim_t s, int levels, unsigned long long* host_trace, long long cap,
                           long long* n_warps) {
  if (!s || !host_trace || !n_warps || s->slab) return fail(RDCNN_EINVAL, "bad argument");
  if (levels != 1 && levels != 2 && levels != 4 && levels != 8) return fail(RDCNN_EINVAL, "bad levels");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  const int w = s->elem == 4 ? width_for<float>(s) : width_for<double>(s);
  const bool per_grid = s->params_stride != 0;
  const bool wrap = s->cols / w == 32;
  const int rw = (s->elem == 4 ? resident_blocks<float>(levels, w, arith_for<float>(s), per_grid, wrap)
                               : resident_blocks<double>(levels, w, arith_for<double>(s), per_grid, wrap)) * (kThreads / 32);
  const Plan p = make_plan(s->cols, w, levels, s->batch, 0, s->rows, seg_for(s, levels, 0, s->rows), s->sm_count, rw);
  *n_warps = p.warps;
  if (p.warps > cap) return fail(RDCNN_EINVAL, "trace needs %lld entries", (long long)p.warps);
  unsigned long long* d = nullptr;
  RDCNN_CUDA_TRY(cudaMalloc(&d, sizeof(unsigned long long) * 3 * (size_t)p.warps));
  int rc = RDCNN_OK;
  if (s->elem == 4) {
    StepArgsT<float> a = base_args<float>(s, s->cur, s->cur ^ 1);
    a.trace = d;
    a.trace_stride = 3;
    a.tag = 1;
    rc = launch_range<float>(s, levels, a, 0, s->rows, s->stream) == cudaSuccess ? RDCNN_OK : RDCNN_ECUDA;
  } else {
    StepArgsT<double> a = base_args<double>(s, s->cur, s->cur ^ 1);
    a.trace = d;
    a.trace_stride = 3;
    a.tag = 1;
    rc = launch_range<double>(s, levels, a, 0, s->rows, s->stream) == cudaSuccess ? RDCNN_OK : RDCNN_ECUDA;
  }
  if (rc == RDCNN_OK) {
    s->cur ^= 1;
    RDCNN_CUDA_TRY(cudaMemcpyAsync(host_trace, d, sizeof(unsigned long long) * 3 * (size_t)p.warps,
                                   cudaMemcpyDeviceToHost, s->stream));
    RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  }
  cudaFree(d);
  if (rc != RDCNN_OK) return fail(rc, "trace launch failed");
  return RDCNN_OK;
}

int rdcnn_sim_set_persistent(rdcnn_sim_t s, int mode) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (mode < -1 || mode > 1) return fail(RDCNN_EINVAL, "mode must be -1, 0 or 1, got %d", mode);
  s->cluster_mode = mode;
  return RDCNN_OK;
}

int rdcnn_sim_upload(rdcnn_sim_t s, const float* u, const float* v) {
  RDCNN_TRY(need_elem(s, 4));
  if (!u || !v) return fail(RDCNN_EINVAL, "null argument");
  return copy_state(s, const_cast<float*>(u), const_cast<float*>(v), true);
}

int rdcnn_sim_download(rdcnn_sim_t s, float* u, float* v) {
  RDCNN_TRY(need_elem(s, 4));
  if (!u || !v) return fail(RDCNN_EINVAL, "null argument");
  return copy_state(s, u, v, false);
}

int rdcnn_sim_upload_f64(rdcnn_sim_t s, const double* u, const double* v) {
  RDCNN_TRY(need_elem(s, 8));
  if (!u || !v) return fail(RDCNN_EINVAL, "null argument");
  return copy_state(s, const_cast<double*>(u), const_cast<double*>(v), true);
}

int rdcnn_sim_download_f64(rdcnn_sim_t s, double* u, double* v) {
  RDCNN_TRY(need_elem(s, 8));
  if (!u || !v) return fail(RDCNN_EINVAL, "null argument");
  return copy_state(s, u, v, false);
}

int rdcnn_sim_init(rdcnn_sim_t s, int typ, uint64_t seed) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (typ != 1 && typ != 2) return fail(RDCNN_EINVAL, "typ must be 1 or 2 (3 = rdcnn_sim_init_image)");
  if (s->slab) return fail(RDCNN_EINVAL, "slab handles initialise through rdcnn_slab_init");
  if (typ == 1 && (s->rows < 11 || s->cols < 11))
    return fail(RDCNN_EINVAL, "typ=1 needs a grid of at least 11x11, got %dx%d", s->rows, s->cols);
  return s->elem == 4 ? init_impl<float>(s, typ, seed, s->rows, 0) : init_impl<double>(s, typ, seed, s->rows, 0);
}

int rdcnn_slab_init(rdcnn_sim_t s, int typ, uint64_t seed, int global_rows, int row_offset) {
  if (!s || !s->slab) return fail(RDCNN_EINVAL, "not a slab handle");
  if (typ != 1 && typ != 2) return fail(RDCNN_EINVAL, "typ must be 1 or 2");
  if (typ == 1 && (global_rows < 11 || s->cols < 11))
    return fail(RDCNN_EINVAL, "typ=1 needs a grid of at least 11x11");
  if (row_offset < 0 || row_offset + s->rows > global_rows)
    return fail(RDCNN_EINVAL, "slab rows [%d,%d) outside the %d-row lattice", row_offset,
                row_offset + s->rows, global_rows);
  return init_impl<float>(s, typ, seed, global_rows, row_offset);
}

int rdcnn_sim_init_image(rdcnn_sim_t s, const uint8_t* px, double ka) {
  if (!s || !px) return fail(RDCNN_EINVAL, "null argument");
  if (s->slab) return fail(RDCNN_EINVAL, "image init is for periodic handles");
  return s->elem == 4 ? image_impl<float>(s, px, ka) : image_impl<double>(s, px, ka);
}

int rdcnn_sim_advance(rdcnn_sim_t s, long steps, long* first_bad) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (s->slab) return fail(RDCNN_EINVAL, "slab handles advance through rdcnn_slab_step_*");
  if (steps < 0) return fail(RDCNN_EINVAL, "steps must be >= 0, got %ld", steps);
  return s->elem == 4 ? advance_impl<float>(s, steps, first_bad) : advance_impl<double>(s, steps, first_bad);
}

int rdcnn_sim_elapsed_ms(rdcnn_sim_t s, double* ms) {
  if (!s || !ms) return fail(RDCNN_EINVAL, "null argument");
  *ms = s->last_ms;
  return RDCNN_OK;
}

int rdcnn_sim_launch_count(rdcnn_sim_t s, long* n) {
  if (!s || !n) return fail(RDCNN_EINVAL, "null argument");
  *n = s->launches;
  return RDCNN_OK;
}

int rdcnn_sim_stream(rdcnn_sim_t s, void** stream) {
  if (!s || !stream) return fail(RDCNN_EINVAL, "null argument");
  *stream = (void*)s->stream;
  return RDCNN_OK;
}

int rdcnn_sim_device_state(rdcnn_sim_t s, void** u, void** v) {
  if (!s || !u || !v) return fail(RDCNN_EINVAL, "null argument");
  const size_t e = (size_t)s->elem;
  char* base = static_cast<char*>(s->buf[s->cur]);
  const size_t row0 = s->slab ? (size_t)s->ghost * s->pitch * e : 0;
  *u = base + row0;
  *v = base + row0 + (s->slab ? (size_t)s->plane_off * e : (size_t)s->rows * s->cols * s->batch * e);
  return RDCNN_OK;
}

// ---- slab phases -----------------------------------------------------------

static int slab_step(rdcnn_sim_t s, int k, void* stream, bool boundary) {
  if (!s || !s->slab) return fail(RDCNN_EINVAL, "not a slab handle");
  if (k != 1 && k != 2 && k != 4 && k != 8) return fail(RDCNN_EINVAL, "k must be 1, 2, 4 or 8");
  if (k > s->ghost) return fail(RDCNN_EINVAL, "k=%d exceeds ghost depth %d", k, s->ghost);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  // The stream is taken literally: 0 is the legacy default stream (what
  // torch.cuda.current_stream() reports by default), not the handle's stream.
  return slab_step_impl<float>(s, k, (cudaStream_t)stream, boundary);
}

int rdcnn_slab_step_boundary(rdcnn_sim_t s, int k, void* stream) { return slab_step(s, k, stream, true); }
int rdcnn_slab_step_interior(rdcnn_sim_t s, int k, void* stream) { return slab_step(s, k, stream, false); }

int rdcnn_slab_swap(rdcnn_sim_t s) {
  if (!s || !s->slab) return fail(RDCNN_EINVAL, "not a slab handle");
  s->cur ^= 1;
  return RDCNN_OK;
}

int rdcnn_slab_rows_ptr(rdcnn_sim_t s, int which, float** first_row, float** first_ghost) {
  if (!s || !s->slab || !first_row || !first_ghost) return fail(RDCNN_EINVAL, "bad argument");
  if (which != 0 && which != 1) return fail(RDCNN_EINVAL, "which must be 0 (front) or 1 (back)");
  const int b = which == 0 ? s->cur : s->cur ^ 1;
  *first_ghost = s->u_ptr<float>(b);
  *first_row = s->u_ptr<float>(b) + (size_t)s->ghost * s->pitch;
  return RDCNN_OK;
}

int rdcnn_slab_poll_blowup(rdcnn_sim_t s, int* bad, unsigned* tag) {
  if (!s || !bad) return fail(RDCNN_EINVAL, "null argument");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  unsigned hv = 0;
  RDCNN_CUDA_TRY(cudaDeviceSynchronize());
  RDCNN_CUDA_TRY(cudaMemcpy(&hv, s->d_flags, sizeof hv, cudaMemcpyDeviceToHost));
  *bad = hv != 0;
  if (tag) *tag = hv;
  return RDCNN_OK;
}

// ---- native slab ring: NCCL transport (boundary launch, NCCL send/recv of the
// ghost rows on a comm stream overlapped with the interior launch) ----------

int rdcnn_nccl_unique_id(uint8_t id[128]) {
  if (!id) return fail(RDCNN_EINVAL, "null argument");
  if (!nccl().ok) return fail(RDCNN_ECUDA, "libnccl.so.2 not loadable");
  ncclUniqueId uid;
  RDCNN_NCCL_TRY(nccl().get_unique_id(&uid));
  std::memcpy(id, &uid, sizeof uid);
  return RDCNN_OK;
}

int rdcnn_slab_attach_ring(rdcnn_sim_t s, const uint8_t id[128], int rank, int world) {
  if (!s || !s->slab) return fail(RDCNN_EINVAL, "not a slab handle");
  if (world < 1 || rank < 0 || rank >= world) return fail(RDCNN_EINVAL, "bad rank %d / world %d", rank, world);
  if (s->comm_stream) return fail(RDCNN_EINVAL, "ring already attached");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  RDCNN_CUDA_TRY(cudaStreamCreateWithFlags(&s->comm_stream, cudaStreamNonBlocking));
  RDCNN_CUDA_TRY(cudaEventCreateWithFlags(&s->ev_bnd, cudaEventDisableTiming));
  RDCNN_CUDA_TRY(cudaEventCreateWithFlags(&s->ev_xchg, cudaEventDisableTiming));
  s->ring_rank = rank;
  s->ring_world = world;
  if (world > 1) {
    if (!id) return fail(RDCNN_EINVAL, "null NCCL id");
    if (!nccl().ok) return fail(RDCNN_ECUDA, "libnccl.so.2 not loadable");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    RDCNN_NCCL_TRY(nccl().comm_init_rank(&s->comm, world, uid, rank));
  }
  return RDCNN_OK;
}

// The ring exchange of buffer `b`: its first `ghost` owned rows go to the
// previous rank (its bottom ghosts), its last `ghost` rows to the next rank
// (its top ghosts).  Issue order matches paper_2102_10340_b200/slab.py
// exchange_ops (tested with gloo): send last -> next, send first -> prev,
// recv top <- prev, recv bottom <- next, so sends and receives between one
// pair pair up in order even when prev == next (world 2).  World 1 closes the
// ring on itself: the torus row wrap is two device copies.
static int ring_exchange(rdcnn_sim* s, int b, cudaStream_t st) {
  float* base = s->u_ptr<float>(b);  // first top-ghost row
  const size_t row = (size_t)s->pitch, g = (size_t)s->ghost, S = (size_t)s->rows;
  float* first = base + g * row;
  float* last = base + S * row;  // owned rows [S-g, S)
  float* top = base;
  float* bottom = base + (g + S) * row;
  const size_t count = g * row;
  if (s->ring_world == 1) {
    RDCNN_CUDA_TRY(cudaMemcpyAsync(top, last, count * sizeof(float), cudaMemcpyDeviceToDevice, st));
    RDCNN_CUDA_TRY(cudaMemcpyAsync(bottom, first, count * sizeof(float), cudaMemcpyDeviceToDevice, st));
    return RDCNN_OK;
  }
  const int prev = (s->ring_rank + s->ring_world - 1) % s->ring_world;
  const int next = (s->ring_rank + 1) % s->ring_world;
  RDCNN_NCCL_TRY(nccl().group_start());
  RDCNN_NCCL_TRY(nccl().send(last, count, ncclFloat32, next, s->comm, st));
  RDCNN_NCCL_TRY(nccl().send(first, count, ncclFloat32, prev, s->comm, st));
  RDCNN_NCCL_TRY(nccl().recv(top, count, ncclFloat32, prev, s->comm, st));
  RDCNN_NCCL_TRY(nccl().recv(bottom, count, ncclFloat32, next, s->comm, st));
  RDCNN_NCCL_TRY(nccl().group_end());
  return RDCNN_OK;
}

// ---- fused peer ring ----------------------------------------------------------

int rdcnn_slab_peer_export(rdcnn_sim_t s, rdcnn_slab_peer_desc* out) {
  if (!s || !s->slab || !out) return fail(RDCNN_EINVAL, "not a slab handle");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  if (!s->p2p_words) {
    RDCNN_CUDA_TRY(cudaMalloc(&s->p2p_words, 4 * sizeof(unsigned)));
    RDCNN_CUDA_TRY(cudaMemset(s->p2p_words, 0, 4 * sizeof(unsigned)));
  }
  std::memset(out, 0, sizeof *out);
  void* mem[3] = {s->buf[0], s->buf[1], s->p2p_words};
  out->ipc_ok = 1;
  for (int m = 0; m < 3; ++m) {
    out->ptr[m] = (uint64_t)(uintptr_t)mem[m];
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, mem[m]) == cudaSuccess) {
      std::memcpy(out->ipc[m], &h, sizeof h);
    } else {
      cudaGetLastError();  // in-process rings do not need IPC
      out->ipc_ok = 0;
    }
  }
  out->pid = (int64_t)getpid();
  out->device = s->device;
  out->rows = s->rows;
  out->cols = s->cols;
  out->ghost = s->ghost;
  return RDCNN_OK;
}

static int open_peer(rdcnn_sim* s, const rdcnn_slab_peer_desc* d, void* mem[3]) {
  if (d->pid == (int64_t)getpid()) {  // same process: the pointers are valid as they are
    for (int m = 0; m < 3; ++m) mem[m] = (void*)(uintptr_t)d->ptr[m];
    if (d->device != s->device) {
      cudaError_t e = cudaDeviceEnablePeerAccess(d->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else RDCNN_CUDA_TRY(e);
    }
    return RDCNN_OK;
  }
  if (!d->ipc_ok) return fail(RDCNN_ECUDA, "peer slab (pid %lld) could not export IPC handles", (long long)d->pid);
  for (int m = 0; m < 3; ++m) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, d->ipc[m], sizeof h);
    RDCNN_CUDA_TRY(cudaIpcOpenMemHandle(&mem[m], h, cudaIpcMemLazyEnablePeerAccess));
    s->ipc_opened.push_back(mem[m]);
  }
  return RDCNN_OK;
}

int rdcnn_slab_attach_peers(rdcnn_sim_t s, int rank, int world, const rdcnn_slab_peer_desc* prev,
                            const rdcnn_slab_peer_desc* next) {
  if (!s || !s->slab || !prev || !next) return fail(RDCNN_EINVAL, "bad argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(RDCNN_EINVAL, "bad rank %d / world %d", rank, world);
  if (s->p2p || s->comm_stream) return fail(RDCNN_EINVAL, "ring already attached");
  if (!s->p2p_words) return fail(RDCNN_EINVAL, "export this slab (rdcnn_slab_peer_export) before attaching");
  for (const rdcnn_slab_peer_desc* d : {prev, next})
    if (d->cols != s->cols || d->ghost != s->ghost)
      return fail(RDCNN_EINVAL, "peer slab %dx%d ghost %d does not match %dx%d ghost %d", d->rows, d->cols,
                  d->ghost, s->rows, s->cols, s->ghost);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  void* mp[3];
  void* mn[3];
  RDCNN_TRY(open_peer(s, prev, mp));
  if (std::memcmp(prev, next, sizeof *prev) == 0) {  // world <= 2: one neighbour on both sides
    std::memcpy(mn, mp, sizeof mp);
  } else {
    RDCNN_TRY(open_peer(s, next, mn));
  }
  for (int b = 0; b < 2; ++b) {
    s->peer_buf[0][b] = mp[b];
    s->peer_buf[1][b] = mn[b];
  }
  s->peer_words[0] = static_cast<unsigned*>(mp[2]);
  s->peer_words[1] = static_cast<unsigned*>(mn[2]);
  s->peer_rows[0] = prev->rows;
  s->peer_rows[1] = next->rows;
  s->ring_rank = rank;
  s->ring_world = world;
  s->p2p = true;
  s->p2p_seq = 0;
  RDCNN_CUDA_TRY(cudaMemset(s->p2p_words, 0, 4 * sizeof(unsigned)));
  return RDCNN_OK;
}

int rdcnn_slab_step_fused(rdcnn_sim_t s, int k, void* stream) {
  if (!s || !s->slab || !s->p2p) return fail(RDCNN_EINVAL, "peer ring not attached");
  if (k != 1 && k != 2 && k != 4 && k != 8) return fail(RDCNN_EINVAL, "k must be 1, 2, 4 or 8");
  if (k > s->ghost) return fail(RDCNN_EINVAL, "k=%d exceeds ghost depth %d", k, s->ghost);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  return peer_block(s, k, s->p2p_seq + 1, stream ? (cudaStream_t)stream : s->stream);
}

int rdcnn_slab_fill_ghosts(rdcnn_sim_t s) {
  if (!s || !s->slab || (!s->comm_stream && !s->p2p)) return fail(RDCNN_EINVAL, "slab ring not attached");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  if (s->p2p) {
    // The peer ring reads the neighbours' rows in place: nothing to copy.
    // The state must be complete before any neighbour's first block reads
    // it; the caller barriers the ranks after this returns.
    RDCNN_CUDA_TRY(cudaDeviceSynchronize());
    return RDCNN_OK;
  }
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  RDCNN_TRY(ring_exchange(s, s->cur, s->comm_stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->comm_stream));
  return RDCNN_OK;
}

// Per block of k <= ghost levels: boundary rows (they read the ghosts) on the
// compute stream; the ring exchange of those rows on the comm stream, which
// waits only for the boundary launch; the interior on the compute stream at
// the same time; then the compute stream waits for the exchange and the
// buffers swap.  No host synchronisation inside the loop.
int rdcnn_slab_advance(rdcnn_sim_t s, long steps, long* first_bad) {
  if (!s || !s->slab || (!s->comm_stream && !s->p2p)) return fail(RDCNN_EINVAL, "slab ring not attached");
  if (steps < 0) return fail(RDCNN_EINVAL, "steps must be >= 0");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  if (first_bad) *first_bad = 0;
  s->launches = 0;
  s->slab_tag = 0;
  RDCNN_CUDA_TRY(cudaMemsetAsync(s->d_flags, 0, sizeof(unsigned), s->stream));
  const Schedule sched = make_schedule(steps, s->max_levels);
  // A state that precedes this advance, for an exact blow-up replay
  // (rdcnn_slab_checkpoint_age): refreshed on the first advance after the
  // state was set and then every ckpt_interval() iterations.  The fused peer
  // ring tees it from its first block's level-0 reads (no extra pass over
  // HBM); the NCCL ring copies it.
  const bool take = s->ckpt && steps > 0 && (s->ckpt_age < 0 || s->ckpt_age >= ckpt_interval());
  if (take) s->ckpt_age = 0;
  s->ckpt_age_at_call = s->ckpt_age;
  if (take && !s->p2p)
    RDCNN_CUDA_TRY(cudaMemcpyAsync(s->ckpt, s->buf[s->cur], s->buf_elems * s->elem, cudaMemcpyDeviceToDevice,
                                   s->stream));
  RDCNN_CUDA_TRY(cudaEventRecord(s->ev0, s->stream));
  for (long n = 0; n < sched.count() && s->p2p; ++n)
    RDCNN_TRY(peer_block(s, sched.depth(n), (unsigned)(n + 1), s->stream,
                         n == 0 && take ? static_cast<float*>(s->ckpt) : nullptr));
  for (long n = 0; n < sched.count() && !s->p2p; ++n) {
    const int k = sched.depth(n);
    RDCNN_TRY(slab_step_impl<float>(s, k, s->stream, true));
    RDCNN_CUDA_TRY(cudaEventRecord(s->ev_bnd, s->stream));
    RDCNN_CUDA_TRY(cudaStreamWaitEvent(s->comm_stream, s->ev_bnd, 0));
    RDCNN_TRY(ring_exchange(s, s->cur ^ 1, s->comm_stream));
    RDCNN_TRY(slab_step_impl<float>(s, k, s->stream, false));
    RDCNN_CUDA_TRY(cudaEventRecord(s->ev_xchg, s->comm_stream));
    RDCNN_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->ev_xchg, 0));
    s->cur ^= 1;
  }
  RDCNN_CUDA_TRY(cudaEventRecord(s->ev1, s->stream));
  if (s->ckpt_age >= 0) s->ckpt_age += steps;
  unsigned tag = 0;
  RDCNN_CUDA_TRY(cudaMemcpyAsync(s->h_flags, s->d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  tag = s->h_flags[0];
  float ms = 0;
  RDCNN_CUDA_TRY(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  s->last_ms = ms;
  if (tag != 0) {
    // Block granularity: a slab cannot replay alone (its neighbours moved on),
    // so the report is the first iteration of the first bad block.
    if (first_bad) *first_bad = sched.start((long)tag - 1) + 1;
    return fail(RDCNN_EBLOWUP, "blow-up: non-finite state in block %u", tag);
  }
  return RDCNN_OK;
}

int rdcnn_slab_checkpoint_enable(rdcnn_sim_t s, int on) {
  if (!s || !s->slab) return fail(RDCNN_EINVAL, "not a slab handle");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  if (on && !s->ckpt) RDCNN_CUDA_TRY(cudaMalloc(&s->ckpt, s->buf_elems * s->elem));
  if (!on && s->ckpt) {
    RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
    RDCNN_CUDA_TRY(cudaFree(s->ckpt));
    s->ckpt = nullptr;
  }
  return RDCNN_OK;
}

int rdcnn_slab_restore(rdcnn_sim_t s) {
  if (!s || !s->slab) return fail(RDCNN_EINVAL, "not a slab handle");
  if (!s->ckpt) return fail(RDCNN_EINVAL, "no checkpoint (rdcnn_slab_checkpoint_enable)");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  RDCNN_CUDA_TRY(cudaDeviceSynchronize());
  if (s->ckpt_age < 0) return fail(RDCNN_EINVAL, "the checkpoint does not precede the current state");
  RDCNN_CUDA_TRY(cudaMemcpyAsync(s->buf[s->cur], s->ckpt, s->buf_elems * s->elem, cudaMemcpyDeviceToDevice,
                                 s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->ckpt_age = 0;
  return RDCNN_OK;
}

int rdcnn_slab_checkpoint_age(rdcnn_sim_t s, long* age) {
  if (!s || !s->slab || !age) return fail(RDCNN_EINVAL, "not a slab handle");
  *age = s->ckpt_age_at_call;
  return RDCNN_OK;
}

// ---- snapshot store and analysis (sweep.hpp:48-112, frame.hpp:28-66) ------

int rdcnn_sim_checksums(rdcnn_sim_t s, uint64_t* out) {
  if (!s || !out) return fail(RDCNN_EINVAL, "null argument");
  if (s->slab) return fail(RDCNN_EINVAL, "not a periodic handle");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  const size_t plane = (size_t)s->rows * s->cols * s->elem;
  // FNV-1a is sequential within a grid: one device thread per grid only pays
  // for batches.  Few grids, or unaligned shapes: hash on the host.
  if (s->batch < 32 || plane % 16 != 0 || (size_t)s->grid_stride * s->elem % 16 != 0) {
    std::vector<unsigned char> hu(plane * s->batch), hv(plane * s->batch);
    RDCNN_TRY(copy_state(s, hu.data(), hv.data(), false));
    for (int g = 0; g < s->batch; ++g) out[g] = fnv_planes(hu.data() + g * plane, hv.data() + g * plane, plane);
    return RDCNN_OK;
  }
  // The digest words live with the handle: a stream-ordered malloc/free per
  // call made this call's wall time vary from 3 to 140 ms.
  if (!s->d_digest) RDCNN_CUDA_TRY(cudaMalloc(&s->d_digest, sizeof(unsigned long long) * (size_t)s->batch));
  unsigned long long* d = s->d_digest;
  const unsigned char* u = static_cast<const unsigned char*>(s->buf[s->cur]);
  const unsigned char* v = u + plane * s->batch;
  fnv_batch_kernel<<<(s->batch + 31) / 32, 32, 0, s->stream>>>(u, v, plane, (size_t)s->grid_stride * s->elem,
                                                                  s->batch, d);
  RDCNN_CUDA_TRY(cudaGetLastError());
  RDCNN_CUDA_TRY(cudaMemcpyAsync(out, d, sizeof(unsigned long long) * (size_t)s->batch, cudaMemcpyDeviceToHost,
                                 s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

int rdcnn_sim_frames_reserve(rdcnn_sim_t s, int nframes) {
  if (!s || s->slab) return fail(RDCNN_EINVAL, "not a periodic handle");
  if (nframes < 1) return fail(RDCNN_EINVAL, "nframes must be >= 1");
  if (s->frames && s->n_frames == nframes) return RDCNN_OK;  // already reserved (reused handles)
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  if (s->frames) RDCNN_CUDA_TRY(cudaFree(s->frames));
  s->frames = nullptr;
  s->n_frames = 0;
  const size_t bytes = (size_t)nframes * s->batch * s->rows * s->cols * s->elem;
  RDCNN_CUDA_TRY(cudaMalloc(&s->frames, bytes));
  if (!s->d_stats) RDCNN_CUDA_TRY(cudaMalloc(&s->d_stats, sizeof(double) * 4 * (size_t)s->batch));
  if (!s->d_counts) RDCNN_CUDA_TRY(cudaMalloc(&s->d_counts, sizeof(long long) * (size_t)s->batch));
  s->n_frames = nframes;
  return RDCNN_OK;
}

static int frame_slot_ok(rdcnn_sim_t s, int slot) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (slot < 0 || slot >= s->n_frames)
    return fail(RDCNN_EINVAL, "frame slot %d outside [0,%d) (rdcnn_sim_frames_reserve)", slot, s->n_frames);
  return RDCNN_OK;
}

int rdcnn_sim_frame_capture(rdcnn_sim_t s, int slot) {
  RDCNN_TRY(frame_slot_ok(s, slot));
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  const size_t bytes = (size_t)s->batch * s->rows * s->cols * s->elem;
  RDCNN_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(s->frames) + (size_t)slot * bytes, s->buf[s->cur],
                                 bytes, cudaMemcpyDeviceToDevice, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

int rdcnn_sim_frame_download(rdcnn_sim_t s, int slot, void* u) {
  RDCNN_TRY(frame_slot_ok(s, slot));
  if (!u) return fail(RDCNN_EINVAL, "null argument");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  const size_t bytes = (size_t)s->batch * s->rows * s->cols * s->elem;
  prefault_pageable(u, bytes);
  RDCNN_CUDA_TRY(cudaMemcpyAsync(u, static_cast<char*>(s->frames) + (size_t)slot * bytes, bytes, cudaMemcpyDeviceToHost,
                                 s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

int rdcnn_sim_frame_stats(rdcnn_sim_t s, int slot, double* mins, double* maxs, double* medians) {
  RDCNN_TRY(frame_slot_ok(s, slot));
  if (!mins || !maxs || !medians) return fail(RDCNN_EINVAL, "null argument");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  return s->elem == 4 ? frame_stats_impl<float>(s, slot, mins, maxs, medians)
                      : frame_stats_impl<double>(s, slot, mins, maxs, medians);
}

int rdcnn_sim_frame_active(rdcnn_sim_t s, int slot, const double* medians, const double* thresholds,
                           long long* counts) {
  RDCNN_TRY(frame_slot_ok(s, slot));
  if (!medians || !thresholds || !counts) return fail(RDCNN_EINVAL, "null argument");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  return s->elem == 4 ? frame_active_impl<float>(s, slot, medians, thresholds, counts)
                      : frame_active_impl<double>(s, slot, medians, thresholds, counts);
}

int rdcnn_sim_frame_normalize(rdcnn_sim_t s, int slot, int grid, double lo, double hi, uint8_t* out) {
  if (!s || !out) return fail(RDCNN_EINVAL, "null argument");
  if (grid < 0 || grid >= s->batch) return fail(RDCNN_EINVAL, "grid %d outside the batch", grid);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  const size_t plane = (size_t)s->rows * s->cols * s->elem;
  const void* src;
  if (slot < 0) {  // the current state's u plane
    if (s->slab) return fail(RDCNN_EINVAL, "not a periodic handle");
    src = static_cast<const char*>(s->buf[s->cur]) + (size_t)grid * plane;
  } else {
    RDCNN_TRY(frame_slot_ok(s, slot));
    src = static_cast<const char*>(s->frames) + ((size_t)slot * s->batch + grid) * plane;
  }
  return s->elem == 4 ? normalize_impl<float>(s, src, lo, hi, out) : normalize_impl<double>(s, src, lo, hi, out);
}

int rdcnn_sim_frame_normalize_auto(rdcnn_sim_t s, int slot, int grid, uint8_t* out, double* lo, double* hi) {
  if (!s || !out) return fail(RDCNN_EINVAL, "null argument");
  if (grid < 0 || grid >= s->batch) return fail(RDCNN_EINVAL, "grid %d outside the batch", grid);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  const size_t plane = (size_t)s->rows * s->cols * s->elem;
  const void* src;
  if (slot < 0) {
    if (s->slab) return fail(RDCNN_EINVAL, "not a periodic handle");
    src = static_cast<const char*>(s->buf[s->cur]) + (size_t)grid * plane;
  } else {
    RDCNN_TRY(frame_slot_ok(s, slot));
    src = static_cast<const char*>(s->frames) + ((size_t)slot * s->batch + grid) * plane;
  }
  return s->elem == 4 ? normalize_auto_impl<float>(s, src, out, lo, hi)
                      : normalize_auto_impl<double>(s, src, out, lo, hi);
}

// ---- host helpers ------------------------------------------------------------

int rdcnn_init_full_random_host(int rows, int cols, uint64_t seed, float* u, float* v) {
  return host_full_random<float>(rows, cols, seed, u, v);
}
int rdcnn_init_center_square_host(int rows, int cols, uint64_t seed, float* u, float* v) {
  return host_center_square<float>(rows, cols, seed, u, v);
}
int rdcnn_init_full_random_host_f64(int rows, int cols, uint64_t seed, double* u, double* v) {
  return host_full_random<double>(rows, cols, seed, u, v);
}
int rdcnn_init_center_square_host_f64(int rows, int cols, uint64_t seed, double* u, double* v) {
  return host_center_square<double>(rows, cols, seed, u, v);
}

uint64_t rdcnn_checksum_f32(const float* u, const float* v, size_t cells) {
  return fnv_planes(u, v, cells * sizeof(float));
}
uint64_t rdcnn_checksum_f64(const double* u, const double* v, size_t cells) {
  return fnv_planes(u, v, cells * sizeof(double));
}

int rdcnn_selftest_div3(int device, int domain, uint64_t* mismatches, uint32_t* first_bad) {
  if (!mismatches || !first_bad || domain < 0 || domain > 2)
    return fail(RDCNN_EINVAL, "bad arguments");
  RDCNN_CUDA_TRY(cudaSetDevice(device));
  unsigned long long* d_count = nullptr;
  unsigned* d_first = nullptr;
  RDCNN_CUDA_TRY(cudaMalloc(&d_count, sizeof *d_count));
  RDCNN_CUDA_TRY(cudaMalloc(&d_first, sizeof *d_first));
  RDCNN_CUDA_TRY(cudaMemset(d_count, 0, sizeof *d_count));
  RDCNN_CUDA_TRY(cudaMemset(d_first, 0xFF, sizeof *d_first));
  div3_selftest_kernel<<<sm_count_for(device) * 8, 256>>>(domain, d_count, d_first);
  RDCNN_CUDA_TRY(cudaGetLastError());
  unsigned long long c = 0;
  unsigned f = 0;
  RDCNN_CUDA_TRY(cudaMemcpy(&c, d_count, sizeof c, cudaMemcpyDeviceToHost));
  RDCNN_CUDA_TRY(cudaMemcpy(&f, d_first, sizeof f, cudaMemcpyDeviceToHost));
  cudaFree(d_count);
  cudaFree(d_first);
  *mismatches = c;
  *first_bad = f;
  return RDCNN_OK;
}

int rdcnn_selftest_div3_f64(int device, uint64_t samples, uint64_t* mismatches, uint64_t* first_bad) {
  if (!mismatches || !first_bad) return fail(RDCNN_EINVAL, "bad arguments");
  RDCNN_CUDA_TRY(cudaSetDevice(device));
  unsigned long long *d_count = nullptr, *d_first = nullptr;
  RDCNN_CUDA_TRY(cudaMalloc(&d_count, sizeof *d_count));
  RDCNN_CUDA_TRY(cudaMalloc(&d_first, sizeof *d_first));
  RDCNN_CUDA_TRY(cudaMemset(d_count, 0, sizeof *d_count));
  RDCNN_CUDA_TRY(cudaMemset(d_first, 0xFF, sizeof *d_first));
  div3_selftest_f64_kernel<<<sm_count_for(device) * 8, 256>>>(samples, d_count, d_first);
  RDCNN_CUDA_TRY(cudaGetLastError());
  unsigned long long c = 0, f = 0;
  RDCNN_CUDA_TRY(cudaMemcpy(&c, d_count, sizeof c, cudaMemcpyDeviceToHost));
  RDCNN_CUDA_TRY(cudaMemcpy(&f, d_first, sizeof f, cudaMemcpyDeviceToHost));
  cudaFree(d_count);
  cudaFree(d_first);
  *mismatches = c;
  *first_bad = f;
  return RDCNN_OK;
}

}  // extern "C"

#include "ring.cuh"
