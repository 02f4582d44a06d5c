// rdcnn_cuda.cu -- C-ABI implementation (include/rdcnn_cuda.h): handles,
// launch planning, device-side initial states, blow-up replay, slab mode.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
//        -fmad=false -prec-div=true -ftz=false -shared -Xcompiler -fPIC
// (see __graft_entry__.build()).  Strict arithmetic relies on -ftz=false
// (reference keeps subnormals, SURVEY.md §7 "Denormals").
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "fhn_stencil.cuh"
#include "rdcnn_cuda.h"

using rdcnn_dev::Params;
using rdcnn_dev::StepArgs;

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

constexpr int kThreads = 128;  // 4 warps per CTA

// ---------------------------------------------------------------------------
// Kernel dispatch over the compiled (K, W, mode) instances.
// ---------------------------------------------------------------------------

using KernelFn = void (*)(StepArgs);

// Every compiled instance: [W=1|4][K=1,2,4,8][strict|fast][shared|per-grid gene].
template <int W, int KI, int FI, int PI>
constexpr KernelFn instance() {
  constexpr int K = 1 << KI;
  return &rdcnn_dev::fhn_wavefront_kernel<K, W, FI == 1, PI == 1>;
}

struct KernelTable {
  KernelFn fn[2][4][2][2];
  int resident[2][4][2][2];
};

template <int W, int KI, int FI, int PI>
void fill_one(KernelTable& t) {
  t.fn[W == 4][KI][FI][PI] = instance<W, KI, FI, PI>();
  t.resident[W == 4][KI][FI][PI] = 0;
}

template <int W, int KI>
void fill_k(KernelTable& t) {
  fill_one<W, KI, 0, 0>(t);
  fill_one<W, KI, 0, 1>(t);
  fill_one<W, KI, 1, 0>(t);
  fill_one<W, KI, 1, 1>(t);
}

KernelTable make_table() {
  KernelTable t{};
  fill_k<1, 0>(t); fill_k<1, 1>(t); fill_k<1, 2>(t); fill_k<1, 3>(t);
  fill_k<4, 0>(t); fill_k<4, 1>(t); fill_k<4, 2>(t); fill_k<4, 3>(t);
  return t;
}

KernelTable& table() {
  static KernelTable t = make_table();
  return t;
}

int k_index(int k) { return k == 1 ? 0 : k == 2 ? 1 : k == 4 ? 2 : 3; }

// Dynamic shared memory of one CTA (the level-0 staging rings).
size_t smem_for(int w) {
  return w == 4 ? rdcnn_dev::wavefront_smem_bytes<4>(kThreads / 32)
                : rdcnn_dev::wavefront_smem_bytes<1>(kThreads / 32);
}

// Resident CTAs per SM of one instance (cached; occupancy is immutable).
int resident_blocks(int k, int w, bool fast, bool per_grid) {
  KernelTable& t = table();
  int& r = t.resident[w == 4][k_index(k)][fast][per_grid];
  if (r == 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, t.fn[w == 4][k_index(k)][fast][per_grid],
                                                      kThreads, smem_for(w)) != cudaSuccess || n < 1)
      n = 1;
    r = n;
  }
  return r;
}

cudaError_t launch_stencil(int k, int w, bool fast, bool per_grid, const StepArgs& a,
                           long long warps, cudaStream_t s) {
  if (warps <= 0) return cudaSuccess;
  if (k != 1 && k != 2 && k != 4 && k != 8) return cudaErrorInvalidValue;
  const long long blocks = (warps + (kThreads / 32) - 1) / (kThreads / 32);
  KernelFn fn = table().fn[w == 4][k_index(k)][fast][per_grid];
  fn<<<dim3((unsigned)blocks), dim3(kThreads), smem_for(w), s>>>(a);
  return cudaGetLastError();
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

__device__ __forceinline__ float unit_f32(uint64_t z) {
  return __fmul_rn((float)(z >> 40), 0x1.0p-24f);  // rng.hpp:28, exact
}

// Writes rows [row_offset, row_offset + local_rows) of a global
// global_rows x cols lattice initialised with typ (1 or 2).
__global__ void init_kernel(float* u, float* v, int pitch, long long grid_stride,
                            int batch, int local_rows, int cols, int global_rows,
                            int row_offset, int typ, uint64_t seed) {
  const long long n = (long long)local_rows * cols;
  const long long gcells = (long long)global_rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * batch;
       idx += (long long)gridDim.x * blockDim.x) {
    const int g = int(idx / n);
    const long long c = idx - (long long)g * n;
    const int li = int(c / cols);
    const int j = int(c - (long long)li * cols);
    const int i = li + row_offset;  // global row
    float uu = 0.0f, vv = 0.0f;
    if (typ == 2) {
      const long long cell = (long long)i * cols + j;
      uu = unit_f32(splitmix_draw(seed, (uint64_t)cell));
      vv = unit_f32(splitmix_draw(seed, (uint64_t)(gcells + cell)));
    } else {
      const int i0 = (global_rows - 11) / 2, j0 = (cols - 11) / 2;  // init.hpp:36-37
      if (i >= i0 && i < i0 + 11 && j >= j0 && j < j0 + 11) {
        const int d = (i - i0) * 11 + (j - j0);
        uu = unit_f32(splitmix_draw(seed, (uint64_t)d));
        vv = unit_f32(splitmix_draw(seed, (uint64_t)(121 + d)));
      }
    }
    const size_t off = (size_t)g * grid_stride + (size_t)li * pitch + j;
    u[off] = uu;
    v[off] = vv;
  }
}

__global__ void image_kernel(float* u, float* v, int pitch, long long grid_stride,
                             int batch, int rows, int cols, const uint8_t* px,
                             const float* lut) {
  const long long n = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * batch;
       idx += (long long)gridDim.x * blockDim.x) {
    const int g = int(idx / n);
    const long long c = idx - (long long)g * n;
    const int i = int(c / cols);
    const int j = int(c - (long long)i * cols);
    const float x = lut[px[c]];
    const size_t off = (size_t)g * grid_stride + (size_t)i * pitch + j;
    u[off] = x;
    v[off] = x;
  }
}

__global__ void div3_selftest_kernel(int domain, unsigned long long* count,
                                     unsigned* first_bad) {
  unsigned long long local = 0;
  unsigned first = 0xFFFFFFFFu;
  const unsigned long long total = 1ull << 32;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       k < total; k += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned bits = (unsigned)k;
    float x = __uint_as_float(bits);
    if (domain == 1) x = __fmul_rn(x, x);
    const float want = __fdiv_rn(x, 3.0f);
    const float got = rdcnn_dev::div3_rn(x);
    bool ok;
    if (isfinite(x))
      ok = __float_as_uint(got) == __float_as_uint(want);
    else
      ok = !isfinite(got);
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
  bool slab = false;
  int ghost = 0;          // slab mode: ghost rows per side
  int pitch = 0;          // floats between rows
  int plane_off = 0;      // floats from u row start to v row start (slab: cols)
  long long grid_stride = 0;  // floats between grids (periodic planar: rows*cols)
  size_t buf_floats = 0;  // floats per buffer (both planes, all grids)
  float* buf[2] = {nullptr, nullptr};
  int cur = 0;            // front buffer index
  Params* d_params = nullptr;
  Params h_params{};      // the shared gene (params_stride == 0)
  int params_stride = 0;
  unsigned* d_flags = nullptr;  // batch words (+1 scratch for replays)
  unsigned* h_flags = nullptr;  // pinned mirror
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0;
  long launches = 0;
  int max_levels = 4;
  int seg_rows = 0;
  int sm_count = 148;
  unsigned slab_tag = 0;

  float* u_ptr(int b) { return buf[b]; }
  float* v_ptr(int b) { return slab ? buf[b] + plane_off : buf[b] + (size_t)rows * cols * batch; }
};

namespace {

int width_for(const rdcnn_sim* s) { return (s->cols % 4 == 0) ? 4 : 1; }

// Periodic handles: planar layout, u planes of all grids then v planes.
StepArgs base_args(const rdcnn_sim* s, int in_buf, int out_buf) {
  StepArgs a{};
  rdcnn_sim* m = const_cast<rdcnn_sim*>(s);
  a.u_in = m->u_ptr(in_buf);
  a.v_in = m->v_ptr(in_buf);
  a.u_out = m->u_ptr(out_buf);
  a.v_out = m->v_ptr(out_buf);
  a.grid_stride = s->grid_stride;
  a.rows = s->rows;
  a.cols = s->cols;
  a.pitch = s->pitch;
  a.periodic = s->slab ? 0 : 1;
  a.ghost = s->slab ? s->ghost : 0;
  a.batch = s->batch;
  a.shared = s->h_params;
  a.params = s->d_params;
  a.params_stride = s->params_stride;
  a.flags = s->d_flags;
  return a;
}

cudaError_t launch_range(rdcnn_sim* s, int k, StepArgs a, int row_begin, int row_end,
                         cudaStream_t st) {
  const int w = width_for(s);
  const bool fast = s->mode == RDCNN_FAST;
  const bool per_grid = a.params_stride != 0;
  const int rw = resident_blocks(k, w, fast, per_grid) * (kThreads / 32);
  Plan p = make_plan(s->cols, w, k, a.batch, row_begin, row_end, s->seg_rows, s->sm_count, rw);
  if (p.warps == 0) return cudaSuccess;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.seg_rows = p.seg_rows;
  a.n_segs = p.n_segs;
  a.n_bands = p.n_bands;
  a.band_groups = p.band_groups;
  a.halo_groups = p.halo;
  ++s->launches;
  return launch_stencil(k, w, fast, per_grid, a, p.warps, st);
}

int alloc_common(rdcnn_sim* s) {
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  s->sm_count = sm_count_for(s->device);
  RDCNN_CUDA_TRY(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  RDCNN_CUDA_TRY(cudaEventCreate(&s->ev0));
  RDCNN_CUDA_TRY(cudaEventCreate(&s->ev1));
  for (int b = 0; b < 2; ++b) {
    RDCNN_CUDA_TRY(cudaMalloc(&s->buf[b], s->buf_floats * sizeof(float)));
    RDCNN_CUDA_TRY(cudaMemsetAsync(s->buf[b], 0, s->buf_floats * sizeof(float), s->stream));
  }
  RDCNN_CUDA_TRY(cudaMalloc(&s->d_params, sizeof(Params) * (size_t)s->batch));
  RDCNN_CUDA_TRY(cudaMalloc(&s->d_flags, sizeof(unsigned) * ((size_t)s->batch + 1)));
  RDCNN_CUDA_TRY(cudaMemsetAsync(s->d_flags, 0, sizeof(unsigned) * ((size_t)s->batch + 1), s->stream));
  RDCNN_CUDA_TRY(cudaMallocHost(&s->h_flags, sizeof(unsigned) * ((size_t)s->batch + 1)));
  // Default gene (gene.hpp:13-24) until set_params is called.
  double g7[7] = {0.1, -0.3, 1.3, -0.1, 1.0, 0.06, 1.0};
  rdcnn_params_f32 p;
  rdcnn_params_from_gene(g7, &p);
  RDCNN_CUDA_TRY(cudaMemcpyAsync(s->d_params, &p, sizeof(Params), cudaMemcpyHostToDevice, s->stream));
  std::memcpy(&s->h_params, &p, sizeof(Params));
  s->params_stride = 0;
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
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
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
// buffer `final_buf`.  Returns the 1-based level (1..k) or a negative error.
int replay_grid(rdcnn_sim* s, int g, int in_buf, int k, int final_buf, int* level_out) {
  unsigned* scratch = s->d_flags + s->batch;
  int a_buf = in_buf;
  for (int m = 1; m <= k; ++m) {
    RDCNN_CUDA_TRY(cudaMemsetAsync(scratch, 0, sizeof(unsigned), s->stream));
    StepArgs a = base_args(s, a_buf, a_buf ^ 1);
    const size_t off = (size_t)g * (size_t)s->grid_stride;
    a.u_in += off;
    a.v_in += off;
    a.u_out += off;
    a.v_out += off;
    a.batch = 1;
    a.params = s->d_params + (size_t)g * s->params_stride;
    a.flags = scratch;
    if (s->params_stride != 0) {
      // One grid: run it on the shared-gene instance with its own gene.
      RDCNN_CUDA_TRY(cudaMemcpyAsync(&a.shared, a.params, sizeof(Params), cudaMemcpyDeviceToHost, s->stream));
      RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
      a.params_stride = 0;
    }
    a.tag = 1;
    RDCNN_CUDA_TRY(launch_range(s, 1, a, 0, s->rows, s->stream));
    unsigned hv = 0;
    RDCNN_CUDA_TRY(cudaMemcpyAsync(&hv, scratch, sizeof hv, cudaMemcpyDeviceToHost, s->stream));
    RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
    a_buf ^= 1;
    if (hv != 0) {
      if (a_buf != final_buf) {
        const size_t plane = (size_t)s->rows * s->cols;
        RDCNN_CUDA_TRY(cudaMemcpyAsync(s->u_ptr(final_buf) + off, s->u_ptr(a_buf) + off,
                                       plane * sizeof(float), cudaMemcpyDeviceToDevice, s->stream));
        RDCNN_CUDA_TRY(cudaMemcpyAsync(s->v_ptr(final_buf) + off, s->v_ptr(a_buf) + off,
                                       plane * sizeof(float), cudaMemcpyDeviceToDevice, s->stream));
        RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
      }
      *level_out = m;
      return RDCNN_OK;
    }
  }
  return fail(RDCNN_ECUDA, "blow-up flagged for grid %d but not reproduced by replay", g);
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
  if (!out) return fail(RDCNN_EINVAL, "null output handle");
  *out = nullptr;
  if (rows < 3 || cols < 3)
    return fail(RDCNN_EINVAL, "grid must be at least 3x3, got %dx%d", rows, cols);
  if (batch < 1) return fail(RDCNN_EINVAL, "batch must be >= 1, got %d", batch);
  if (mode != RDCNN_STRICT && mode != RDCNN_FAST) return fail(RDCNN_EINVAL, "unknown mode %d", mode);
  auto* s = new (std::nothrow) rdcnn_sim();
  if (!s) return fail(RDCNN_EINVAL, "out of host memory");
  s->rows = rows;
  s->cols = cols;
  s->batch = batch;
  s->device = device;
  s->mode = mode;
  s->pitch = cols;
  s->grid_stride = (long long)rows * cols;
  s->buf_floats = (size_t)rows * cols * batch * 2;
  int rc = alloc_common(s);
  if (rc != RDCNN_OK) {
    std::string msg = g_last_error;
    free_all(s);
    g_last_error = msg;
    return rc;
  }
  *out = s;
  return RDCNN_OK;
}

int rdcnn_slab_create(int rows, int cols, int ghost, int device, int mode, rdcnn_sim_t* out) {
  if (!out) return fail(RDCNN_EINVAL, "null output handle");
  *out = nullptr;
  if (cols < 3 || rows < 1) return fail(RDCNN_EINVAL, "bad slab shape %dx%d", rows, cols);
  if (ghost != 1 && ghost != 2 && ghost != 4 && ghost != 8)
    return fail(RDCNN_EINVAL, "ghost depth must be 1, 2, 4 or 8, got %d", ghost);
  if (rows < 2 * ghost) return fail(RDCNN_EINVAL, "slab rows %d < 2*ghost %d", rows, 2 * ghost);
  auto* s = new (std::nothrow) rdcnn_sim();
  if (!s) return fail(RDCNN_EINVAL, "out of host memory");
  s->rows = rows;
  s->cols = cols;
  s->batch = 1;
  s->device = device;
  s->mode = mode;
  s->slab = true;
  s->ghost = ghost;
  s->pitch = 2 * cols;
  s->plane_off = cols;
  s->grid_stride = 0;
  s->buf_floats = (size_t)(rows + 2 * ghost) * 2 * cols;
  s->max_levels = ghost;
  int rc = alloc_common(s);
  if (rc != RDCNN_OK) {
    std::string msg = g_last_error;
    free_all(s);
    g_last_error = msg;
    return rc;
  }
  // buf[b] points at the first ghost row; owned row 0 is `ghost` rows below.
  *out = s;
  return RDCNN_OK;
}

void rdcnn_sim_destroy(rdcnn_sim_t s) { free_all(s); }

int rdcnn_sim_set_params(rdcnn_sim_t s, const rdcnn_params_f32* p, int n) {
  if (!s || !p) return fail(RDCNN_EINVAL, "null argument");
  if (n != 1 && n != s->batch) return fail(RDCNN_EINVAL, "params count %d must be 1 or batch %d", n, s->batch);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  static_assert(sizeof(Params) == sizeof(rdcnn_params_f32), "layout");
  RDCNN_CUDA_TRY(cudaMemcpyAsync(s->d_params, p, sizeof(Params) * (size_t)n, cudaMemcpyHostToDevice, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->params_stride = (n == 1) ? 0 : 1;
  if (n == 1) std::memcpy(&s->h_params, p, sizeof(Params));
  return RDCNN_OK;
}

int rdcnn_sim_set_tuning(rdcnn_sim_t s, int max_levels, int seg_rows) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (max_levels != 1 && max_levels != 2 && max_levels != 4 && max_levels != 8)
    return fail(RDCNN_EINVAL, "max_levels must be 1, 2, 4 or 8, got %d", max_levels);
  if (s->slab && max_levels > s->ghost)
    return fail(RDCNN_EINVAL, "max_levels %d exceeds slab ghost depth %d", max_levels, s->ghost);
  if (seg_rows < 0) return fail(RDCNN_EINVAL, "seg_rows must be >= 0");
  s->max_levels = max_levels;
  s->seg_rows = seg_rows;
  return RDCNN_OK;
}

int rdcnn_sim_upload(rdcnn_sim_t s, const float* u, const float* v) {
  if (!s || !u || !v) return fail(RDCNN_EINVAL, "null argument");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  // Slab phases run on caller streams: drain them before touching the state.
  if (s->slab) RDCNN_CUDA_TRY(cudaDeviceSynchronize());
  const size_t plane = (size_t)s->rows * s->cols;
  if (!s->slab) {
    RDCNN_CUDA_TRY(cudaMemcpyAsync(s->u_ptr(s->cur), u, plane * s->batch * sizeof(float), cudaMemcpyHostToDevice, s->stream));
    RDCNN_CUDA_TRY(cudaMemcpyAsync(s->v_ptr(s->cur), v, plane * s->batch * sizeof(float), cudaMemcpyHostToDevice, s->stream));
  } else {
    const size_t row0 = (size_t)s->ghost * s->pitch;
    const size_t dpitch = (size_t)s->pitch * sizeof(float), w = (size_t)s->cols * sizeof(float);
    RDCNN_CUDA_TRY(cudaMemcpy2DAsync(s->u_ptr(s->cur) + row0, dpitch, u, w, w, s->rows, cudaMemcpyHostToDevice, s->stream));
    RDCNN_CUDA_TRY(cudaMemcpy2DAsync(s->v_ptr(s->cur) + row0, dpitch, v, w, w, s->rows, cudaMemcpyHostToDevice, s->stream));
  }
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

int rdcnn_sim_download(rdcnn_sim_t s, float* u, float* v) {
  if (!s || !u || !v) return fail(RDCNN_EINVAL, "null argument");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  if (s->slab) RDCNN_CUDA_TRY(cudaDeviceSynchronize());
  const size_t plane = (size_t)s->rows * s->cols;
  if (!s->slab) {
    RDCNN_CUDA_TRY(cudaMemcpyAsync(u, s->u_ptr(s->cur), plane * s->batch * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
    RDCNN_CUDA_TRY(cudaMemcpyAsync(v, s->v_ptr(s->cur), plane * s->batch * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
  } else {
    const size_t row0 = (size_t)s->ghost * s->pitch;
    const size_t spitch = (size_t)s->pitch * sizeof(float), w = (size_t)s->cols * sizeof(float);
    RDCNN_CUDA_TRY(cudaMemcpy2DAsync(u, w, s->u_ptr(s->cur) + row0, spitch, w, s->rows, cudaMemcpyDeviceToHost, s->stream));
    RDCNN_CUDA_TRY(cudaMemcpy2DAsync(v, w, s->v_ptr(s->cur) + row0, spitch, w, s->rows, cudaMemcpyDeviceToHost, s->stream));
  }
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

int rdcnn_sim_init(rdcnn_sim_t s, int typ, uint64_t seed) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (typ != 1 && typ != 2) return fail(RDCNN_EINVAL, "typ must be 1 or 2 (3 = rdcnn_sim_init_image)");
  if (s->slab) return fail(RDCNN_EINVAL, "slab handles initialise through rdcnn_slab_init");
  if (typ == 1 && (s->rows < 11 || s->cols < 11))
    return fail(RDCNN_EINVAL, "typ=1 needs a grid of at least 11x11, got %dx%d", s->rows, s->cols);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  init_kernel<<<4 * s->sm_count, 256, 0, s->stream>>>(s->u_ptr(s->cur), s->v_ptr(s->cur), s->pitch,
                                                       s->grid_stride, s->batch, s->rows, s->cols,
                                                       s->rows, 0, typ, seed);
  RDCNN_CUDA_TRY(cudaGetLastError());
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

// Slab of a global_rows x cols torus starting at global row row_offset.
int rdcnn_slab_init(rdcnn_sim_t s, int typ, uint64_t seed, int global_rows, int row_offset) {
  if (!s || !s->slab) return fail(RDCNN_EINVAL, "not a slab handle");
  if (typ != 1 && typ != 2) return fail(RDCNN_EINVAL, "typ must be 1 or 2");
  if (typ == 1 && (global_rows < 11 || s->cols < 11))
    return fail(RDCNN_EINVAL, "typ=1 needs a grid of at least 11x11");
  if (row_offset < 0 || row_offset + s->rows > global_rows)
    return fail(RDCNN_EINVAL, "slab rows [%d,%d) outside the %d-row lattice", row_offset,
                row_offset + s->rows, global_rows);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  const size_t row0 = (size_t)s->ghost * s->pitch;
  init_kernel<<<4 * s->sm_count, 256, 0, s->stream>>>(s->u_ptr(s->cur) + row0, s->v_ptr(s->cur) + row0,
                                                       s->pitch, 0, 1, s->rows, s->cols, global_rows,
                                                       row_offset, typ, seed);
  RDCNN_CUDA_TRY(cudaGetLastError());
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

int rdcnn_sim_init_image(rdcnn_sim_t s, const uint8_t* px, double ka) {
  if (!s || !px) return fail(RDCNN_EINVAL, "null argument");
  if (s->slab) return fail(RDCNN_EINVAL, "image init is for periodic handles");
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  float lut[256];
  const float k = (float)ka;
  for (int p = 0; p < 256; ++p) lut[p] = k * (float)(p / 255.0);  // init.hpp:58, image.hpp:283
  const size_t n = (size_t)s->rows * s->cols;
  uint8_t* d_px = nullptr;
  float* d_lut = nullptr;
  RDCNN_CUDA_TRY(cudaMallocAsync(&d_px, n, s->stream));
  RDCNN_CUDA_TRY(cudaMallocAsync(&d_lut, sizeof lut, s->stream));
  RDCNN_CUDA_TRY(cudaMemcpyAsync(d_px, px, n, cudaMemcpyHostToDevice, s->stream));
  RDCNN_CUDA_TRY(cudaMemcpyAsync(d_lut, lut, sizeof lut, cudaMemcpyHostToDevice, s->stream));
  image_kernel<<<4 * s->sm_count, 256, 0, s->stream>>>(s->u_ptr(s->cur), s->v_ptr(s->cur), s->pitch,
                                                        s->grid_stride, s->batch, s->rows, s->cols,
                                                        d_px, d_lut);
  RDCNN_CUDA_TRY(cudaGetLastError());
  RDCNN_CUDA_TRY(cudaFreeAsync(d_px, s->stream));
  RDCNN_CUDA_TRY(cudaFreeAsync(d_lut, s->stream));
  RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RDCNN_OK;
}

int rdcnn_sim_advance(rdcnn_sim_t s, long steps, long* first_bad) {
  if (!s) return fail(RDCNN_EINVAL, "null handle");
  if (s->slab) return fail(RDCNN_EINVAL, "slab handles advance through rdcnn_slab_step_*");
  if (steps < 0) return fail(RDCNN_EINVAL, "steps must be >= 0, got %ld", steps);
  RDCNN_CUDA_TRY(cudaSetDevice(s->device));
  s->launches = 0;
  if (first_bad)
    for (int g = 0; g < s->batch; ++g) first_bad[g] = 0;
  RDCNN_CUDA_TRY(cudaMemsetAsync(s->d_flags, 0, sizeof(unsigned) * (size_t)s->batch, s->stream));
  const Schedule sched = make_schedule(steps, s->max_levels);
  const int cur0 = s->cur;
  RDCNN_CUDA_TRY(cudaEventRecord(s->ev0, s->stream));
  const long nl = sched.count();
  for (long n = 0; n < nl; ++n) {
    StepArgs a = base_args(s, s->cur, s->cur ^ 1);
    a.tag = (unsigned)(n + 1);
    RDCNN_CUDA_TRY(launch_range(s, sched.depth(n), a, 0, s->rows, s->stream));
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
    int rc = replay_grid(s, g, in_buf, sched.depth(n), s->cur, &level);
    if (rc != RDCNN_OK) return rc;
    if (first_bad) first_bad[g] = sched.start(n) + level;
  }
  if (any) return fail(RDCNN_EBLOWUP, "blow-up: non-finite state");
  return RDCNN_OK;
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

int rdcnn_sim_device_state(rdcnn_sim_t s, float** u, float** v) {
  if (!s || !u || !v) return fail(RDCNN_EINVAL, "null argument");
  const size_t row0 = s->slab ? (size_t)s->ghost * s->pitch : 0;
  *u = s->u_ptr(s->cur) + row0;
  *v = s->v_ptr(s->cur) + row0;
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
  cudaStream_t st = (cudaStream_t)stream;
  StepArgs a = base_args(s, s->cur, s->cur ^ 1);
  if (boundary) ++s->slab_tag;
  a.tag = s->slab_tag;
  const int gh = s->ghost;
  if (boundary) {
    RDCNN_CUDA_TRY(launch_range(s, k, a, 0, gh, st));
    RDCNN_CUDA_TRY(launch_range(s, k, a, s->rows - gh, s->rows, st));
  } else {
    RDCNN_CUDA_TRY(launch_range(s, k, a, gh, s->rows - gh, st));
  }
  return RDCNN_OK;
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
  *first_ghost = s->buf[b];
  *first_row = s->buf[b] + (size_t)s->ghost * s->pitch;
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

// ---- host helpers ------------------------------------------------------------

static uint64_t host_mix(uint64_t& st) {
  uint64_t z = (st += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static float host_unit(uint64_t& st) { return (float)(host_mix(st) >> 40) * 0x1.0p-24f; }

int rdcnn_init_full_random_host(int rows, int cols, uint64_t seed, float* u, float* v) {
  if (rows < 3 || cols < 3 || !u || !v) return fail(RDCNN_EINVAL, "bad arguments");
  uint64_t st = seed;
  const size_t n = (size_t)rows * cols;
  for (size_t k = 0; k < n; ++k) u[k] = host_unit(st);
  for (size_t k = 0; k < n; ++k) v[k] = host_unit(st);
  return RDCNN_OK;
}

int rdcnn_init_center_square_host(int rows, int cols, uint64_t seed, float* u, float* v) {
  if (rows < 11 || cols < 11 || !u || !v)
    return fail(RDCNN_EINVAL, "typ=1 needs a grid of at least 11x11, got %dx%d", rows, cols);
  const size_t n = (size_t)rows * cols;
  std::memset(u, 0, n * sizeof(float));
  std::memset(v, 0, n * sizeof(float));
  const int i0 = (rows - 11) / 2, j0 = (cols - 11) / 2;
  uint64_t st = seed;
  for (int i = i0; i < i0 + 11; ++i)
    for (int j = j0; j < j0 + 11; ++j) u[(size_t)i * cols + j] = host_unit(st);
  for (int i = i0; i < i0 + 11; ++i)
    for (int j = j0; j < j0 + 11; ++j) v[(size_t)i * cols + j] = host_unit(st);
  return RDCNN_OK;
}

uint64_t rdcnn_checksum_f32(const float* u, const float* v, size_t cells) {
  uint64_t h = 0xcbf29ce484222325ull;
  const unsigned char* planes[2] = {reinterpret_cast<const unsigned char*>(u),
                                    reinterpret_cast<const unsigned char*>(v)};
  for (const unsigned char* p : planes)
    for (size_t i = 0; i < cells * sizeof(float); ++i) {
      h ^= p[i];
      h *= 0x100000001b3ull;
    }
  return h;
}

int rdcnn_selftest_div3(int device, int domain, uint64_t* mismatches, uint32_t* first_bad) {
  if (!mismatches || !first_bad || (domain != 0 && domain != 1))
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

}  // extern "C"
