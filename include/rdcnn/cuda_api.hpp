// cuda_api.hpp -- source-compatible C++ API of the reference's time-stepping
// path (proj/include/rdcnn/*.hpp), implemented over the C-ABI in
// include/rdcnn_cuda.h.  Host code written against the reference keeps its
// types and calls (Gene, GridState, StepBuffers, step, run, run_timed,
// init_*, checksum, make_backend) and selects the B200 kernels with
// make_backend("cuda").  Link with -lrdcnn_cuda.
//
// Reference interface -> here:
//   gene.hpp:13-85        Gene, gene_valid, gene_to_vector, vector_to_gene,
//                         gene_field, stability_advisory
//   grid.hpp:13-126       Precision, GridState, finite check, cyclic_shift,
//                         fnv1a, checksum, checksum_hex
//   rng.hpp:11-39         SeededRng
//   model.hpp:13-86       CellModel, FhnParams, make_params, reaction_u/v,
//                         cell_update, FhnModel (host scalar utilities)
//   backend.hpp:12-50     BackendKind (+Cuda), Backend, make_backend
//   kernels.hpp:22-259    StepBuffers, step
//   config.hpp:20-95      InitMode, RunConfig, validate_config
//   init.hpp:20-82        init_full_random, init_center_square,
//                         init_from_image, initial_state (no file I/O)
//   engine.hpp:15-106     ScheduleError, BlowUpError, SnapshotBuffer,
//                         RunOutput, run, run_timed
//   bench.hpp:21-251      Throughput, throughput, BenchRecord, BenchCellError,
//                         bench_suite, emit_csv, emit_table, emit_json
//   sweep.hpp:16-326      Regime, ClassifierConfig, growth_curve,
//                         classify_outcome, SweepSpec, SweepCell, SweepResult,
//                         sweep_grid (batched on the device; no PNG panel)
//   config.hpp:102-106    format_double
//
// Behavioural contract: identical to the reference for the cuda backend
// (bit-exact states in strict mode; BlowUpError at the same iteration;
// step() swaps and returns false on a non-finite result).  The reference's
// CPU backends are not re-implemented: selecting one throws
// std::invalid_argument (there is no silent fallback).  The CUDA kernels are
// FitzHugh-Nagumo in fp32 (strict or fast) and fp64 (strict); other
// CellModels run on a generic device stencil from nvcc-compiled callers
// (rdcnn/cuda_model.cuh) and throw from host-compiled ones.
#pragma once

#if defined(__CUDACC__)
#include "rdcnn/cuda_model.cuh"
#endif

#include <algorithm>
#include <array>
#include <charconv>
#include <chrono>
#include <cmath>
#include <concepts>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "rdcnn_cuda.h"

namespace rdcnn {

// ===========================================================================
// Parameters
// ===========================================================================

struct Gene {
  double a = -0.3;
  double b = 1.3;
  double eps = -0.1;
  double c = 1.0;
  double Du = 0.06;
  double Dv = 1.0;
  double dt = 0.1;
  double ka = 1.0;  // image-input scaling, init only
  bool operator==(const Gene&) const = default;
};

inline bool gene_finite(const Gene& g) {
  for (double x : {g.a, g.b, g.eps, g.c, g.Du, g.Dv, g.dt, g.ka})
    if (!std::isfinite(x)) return false;
  return true;
}

inline bool gene_valid(const Gene& g) {
  return gene_finite(g) && g.dt >= 0.0 && g.Du >= 0.0 && g.Dv >= 0.0;
}

// Kernel order {dt, a, b, eps, c, Du, Dv}; ka excluded.
inline std::array<double, 7> gene_to_vector(const Gene& g) {
  return {g.dt, g.a, g.b, g.eps, g.c, g.Du, g.Dv};
}

inline Gene vector_to_gene(const std::array<double, 7>& p, double ka = 1.0) {
  return Gene{p[1], p[2], p[3], p[4], p[5], p[6], p[0], ka};
}

inline bool stability_advisory(const Gene& g) { return g.dt * std::fmax(g.Du, g.Dv) > 0.25; }

inline double& gene_field(Gene& g, const std::string& name) {
  static const std::pair<const char*, double Gene::*> fields[] = {
      {"a", &Gene::a},   {"b", &Gene::b},   {"eps", &Gene::eps}, {"c", &Gene::c},
      {"du", &Gene::Du}, {"dv", &Gene::Dv}, {"dt", &Gene::dt},   {"ka", &Gene::ka}};
  for (const auto& [n, m] : fields)
    if (name == n) return g.*m;
  throw std::invalid_argument("unknown gene field: " + name);
}

inline double gene_field(const Gene& g, const std::string& name) {
  return gene_field(const_cast<Gene&>(g), name);
}

inline bool is_gene_field(const std::string& name) {
  Gene g;
  try {
    (void)gene_field(g, name);
    return true;
  } catch (const std::invalid_argument&) {
    return false;
  }
}

// ===========================================================================
// Lattice state and digest
// ===========================================================================

enum class Precision { Single, Double };

inline const char* precision_name(Precision p) { return p == Precision::Single ? "single" : "double"; }

inline Precision parse_precision(const std::string& s) {
  if (s == "single") return Precision::Single;
  if (s == "double") return Precision::Double;
  throw std::invalid_argument("unknown precision: " + s);
}

template <class T>
constexpr Precision precision_of() {
  return sizeof(T) == 4 ? Precision::Single : Precision::Double;
}

template <class T>
struct GridState {
  static_assert(std::is_floating_point_v<T>);
  int rows = 0;
  int cols = 0;
  std::vector<T> u;
  std::vector<T> v;

  GridState() = default;
  GridState(int nn, int nm) : rows(nn), cols(nm) {
    if (nn < 3 || nm < 3) throw std::invalid_argument("grid must be at least 3x3");
    u.assign(size_t(nn) * nm, T(0));
    v.assign(size_t(nn) * nm, T(0));
  }
  size_t cells() const { return size_t(rows) * cols; }
  T& at_u(int i, int j) { return u[size_t(i) * cols + j]; }
  T at_u(int i, int j) const { return u[size_t(i) * cols + j]; }
  T& at_v(int i, int j) { return v[size_t(i) * cols + j]; }
  T at_v(int i, int j) const { return v[size_t(i) * cols + j]; }
  bool operator==(const GridState&) const = default;
};

namespace detail {
template <class T>
inline bool finite_bits(T x) {
  if constexpr (sizeof(T) == 4) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    return (b & 0x7F800000u) != 0x7F800000u;
  } else {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    return (b & 0x7FF0000000000000ull) != 0x7FF0000000000000ull;
  }
}
}  // namespace detail

template <class T>
bool all_finite(std::span<const T> xs) {
  return std::all_of(xs.begin(), xs.end(), [](T x) { return detail::finite_bits(x); });
}

template <class T>
bool all_finite(const GridState<T>& s) {
  return all_finite(std::span<const T>(s.u)) && all_finite(std::span<const T>(s.v));
}

template <class T>
GridState<T> cyclic_shift(const GridState<T>& s, int di, int dj) {
  GridState<T> out(s.rows, s.cols);
  for (int i = 0; i < s.rows; ++i) {
    const int si = ((i - di) % s.rows + s.rows) % s.rows;
    for (int j = 0; j < s.cols; ++j) {
      const int sj = ((j - dj) % s.cols + s.cols) % s.cols;
      out.at_u(i, j) = s.at_u(si, sj);
      out.at_v(i, j) = s.at_v(si, sj);
    }
  }
  return out;
}

inline uint64_t fnv1a(const void* data, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  return h;
}

template <class T>
uint64_t checksum(const GridState<T>& s) {
  return fnv1a(s.v.data(), s.v.size() * sizeof(T), fnv1a(s.u.data(), s.u.size() * sizeof(T)));
}

inline std::string checksum_hex(uint64_t x) {
  static const char* digits = "0123456789abcdef";
  std::string out(16, '0');
  for (int k = 15; k >= 0; --k, x >>= 4) out[size_t(k)] = digits[x & 0xF];
  return out;
}

// ===========================================================================
// RNG and initial states
// ===========================================================================

class SeededRng {
 public:
  explicit SeededRng(uint64_t seed) : s_(seed) {}
  uint64_t next_u64() {
    uint64_t z = (s_ += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double next_double() { return double(next_u64() >> 11) * 0x1.0p-53; }
  float next_float() { return float(next_u64() >> 40) * 0x1.0p-24f; }
  template <class T>
  T next_unit() {
    if constexpr (sizeof(T) == 4) return next_float();
    else return next_double();
  }

 private:
  uint64_t s_;
};

struct GridTooSmall : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ImageTooSmall : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

inline constexpr int kSeedSquare = 11;

template <class T>
GridState<T> init_full_random(int nn, int nm, uint64_t seed) {
  GridState<T> s(nn, nm);
  SeededRng rng(seed);
  for (T& x : s.u) x = rng.next_unit<T>();
  for (T& x : s.v) x = rng.next_unit<T>();
  return s;
}

template <class T>
GridState<T> init_center_square(int nn, int nm, uint64_t seed) {
  if (nn < kSeedSquare || nm < kSeedSquare)
    throw GridTooSmall("typ=1 needs a grid of at least 11x11, got " + std::to_string(nn) + "x" +
                       std::to_string(nm));
  GridState<T> s(nn, nm);
  SeededRng rng(seed);
  const int i0 = (nn - kSeedSquare) / 2, j0 = (nm - kSeedSquare) / 2;
  for (T* plane : {s.u.data(), s.v.data()})
    for (int i = i0; i < i0 + kSeedSquare; ++i)
      for (int j = j0; j < j0 + kSeedSquare; ++j) plane[size_t(i) * nm + j] = rng.next_unit<T>();
  return s;
}

// A [0,1] grayscale raster (what the reference's load_grayscale returns).
struct GrayImage {
  int rows = 0, cols = 0;
  std::vector<double> px;
  double at(int i, int j) const { return px[size_t(i) * cols + j]; }
};

template <class T>
GridState<T> init_from_image(const GrayImage& img, const Gene& gene) {
  if (img.rows < 3 || img.cols < 3)
    throw ImageTooSmall("image must be at least 3x3, got " + std::to_string(img.rows) + "x" +
                        std::to_string(img.cols));
  GridState<T> s(img.rows, img.cols);
  const T ka = T(gene.ka);
  for (size_t k = 0; k < img.px.size(); ++k) s.u[k] = s.v[k] = ka * T(img.px[k]);
  return s;
}

// ===========================================================================
// Cell model (host scalar utilities; the device kernel is FHN fp32)
// ===========================================================================

template <class M>
concept CellModel = requires(const M m, typename M::value_type x) {
  requires std::is_floating_point_v<typename M::value_type>;
  { m.reaction_u(x, x) } -> std::same_as<typename M::value_type>;
  { m.reaction_v(x, x) } -> std::same_as<typename M::value_type>;
  { m.diffusion_u() } -> std::same_as<typename M::value_type>;
  { m.diffusion_v() } -> std::same_as<typename M::value_type>;
  { m.time_step() } -> std::same_as<typename M::value_type>;
};

template <class T>
struct FhnParams {
  T dt, a, b, eps, c, du, dv;
};

template <class T>
FhnParams<T> make_params(const Gene& g) {
  return {T(g.dt), T(g.a), T(g.b), T(g.eps), T(g.c), T(g.Du), T(g.Dv)};
}

template <class T>
inline T reaction_u(T u, T v, const FhnParams<T>& p) {
  return u * (p.c - u * u / T(3)) - v;
}
template <class T>
inline T reaction_v(T u, T v, const FhnParams<T>& p) {
  return -p.eps * (u - p.b * v + p.a);
}
template <class T>
inline void cell_update(T u, T v, T lu, T lv, const FhnParams<T>& p, T& un, T& vn) {
  un = u + p.dt * (reaction_u(u, v, p) + p.du * lu);
  vn = v + p.dt * (reaction_v(u, v, p) + p.dv * lv);
}
template <class T>
inline T reaction_u(T u, T v, const Gene& g) { return reaction_u(u, v, make_params<T>(g)); }
template <class T>
inline T reaction_v(T u, T v, const Gene& g) { return reaction_v(u, v, make_params<T>(g)); }
template <class T>
inline void cell_update(T u, T v, T lu, T lv, const Gene& g, T& un, T& vn) {
  cell_update(u, v, lu, lv, make_params<T>(g), un, vn);
}

template <class T>
struct FhnModel {
  using value_type = T;
  FhnParams<T> p;
  explicit FhnModel(const Gene& g) : p(make_params<T>(g)) {}
  explicit FhnModel(const FhnParams<T>& q) : p(q) {}
  T reaction_u(T u, T v) const { return rdcnn::reaction_u(u, v, p); }
  T reaction_v(T u, T v) const { return rdcnn::reaction_v(u, v, p); }
  T diffusion_u() const { return p.du; }
  T diffusion_v() const { return p.dv; }
  T time_step() const { return p.dt; }
};

// ===========================================================================
// Backend selection
// ===========================================================================

enum class BackendKind { Reference, Shift, Blocked, Parallel, Cuda };

struct Backend {
  BackendKind kind = BackendKind::Cuda;
  int tile_rows = 64;
  int tile_cols = 64;
  int threads = 0;
  int device = 0;                // CUDA ordinal
  int mode = RDCNN_STRICT;       // RDCNN_STRICT (bit-exact) or RDCNN_FAST
  int levels = 4;                // time levels fused per launch (1, 2, 4, 8)
  // Two or more entries: the lattice is split into row slabs, slab r on
  // CUDA device devices[r] (entries may repeat), halos exchanged by the
  // fused peer ring (rdcnn_ring_*, fp32).  Empty or one entry: one device.
  // The multi-GPU counterpart of the reference's row-band parallelism
  // (kernels.hpp:153-174).
  std::vector<int> devices;
  bool exact_order() const { return kind != BackendKind::Shift && mode == RDCNN_STRICT; }
};

inline const char* backend_name(BackendKind k) {
  switch (k) {
    case BackendKind::Reference: return "reference";
    case BackendKind::Shift: return "shift";
    case BackendKind::Blocked: return "blocked";
    case BackendKind::Parallel: return "parallel";
    case BackendKind::Cuda: return "cuda";
  }
  return "?";
}
inline const char* backend_name(const Backend& b) { return backend_name(b.kind); }

inline BackendKind parse_backend_kind(const std::string& s) {
  for (BackendKind k : {BackendKind::Reference, BackendKind::Shift, BackendKind::Blocked,
                        BackendKind::Parallel, BackendKind::Cuda})
    if (s == backend_name(k)) return k;
  throw std::invalid_argument("unknown backend: " + s +
                              " (expected reference|shift|blocked|parallel|cuda)");
}

inline Backend make_backend(const std::string& name, int tile_rows = 64, int tile_cols = 64,
                            int threads = 0) {
  if (tile_rows < 1 || tile_cols < 1) throw std::invalid_argument("tile dimensions must be >= 1");
  if (threads < 0) throw std::invalid_argument("thread count must be >= 0");
  Backend b;
  b.kind = parse_backend_kind(name);
  b.tile_rows = tile_rows;
  b.tile_cols = tile_cols;
  b.threads = threads;
  return b;
}

// ===========================================================================
// Device handle (RAII over rdcnn_sim_t)
// ===========================================================================

struct CudaError : std::runtime_error {
  int code;
  CudaError(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

namespace detail {

inline void require_cuda(const Backend& b) {
  if (b.kind != BackendKind::Cuda)
    throw std::invalid_argument(std::string("backend '") + backend_name(b) +
                                "' is a reference CPU backend; this library provides 'cuda'");
}

inline void check(int rc, const char* what) {
  if (rc != RDCNN_OK && rc != RDCNN_EBLOWUP)
    throw CudaError(rc, std::string(what) + ": " + rdcnn_last_error());
}

// What a device lattice was created for: a handle is reused only for the
// same device(s), arithmetic mode and fusion depth.
struct SimKey {
  int device = 0, mode = RDCNN_STRICT, levels = 4;
  std::vector<int> devices;
  bool operator==(const SimKey&) const = default;
};

inline SimKey sim_key(const Backend& b) {
  SimKey k{b.device, b.mode, b.levels, {}};
  if (b.devices.size() >= 2) k.devices = b.devices;
  return k;
}

// One lattice of element type T (fp32, or fp64 in strict mode) on one
// device, or -- when the backend names two or more devices -- row slabs of
// it on several (fp32 only; rdcnn_ring_*).
template <class T>
class Sim {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>);

 public:
  Sim(int rows, int cols, const Backend& b) : rows_(rows), cols_(cols), key_(sim_key(b)) {
    if (!key_.devices.empty()) {
      if constexpr (sizeof(T) != 4) {
        throw std::invalid_argument("multi-device row slabs run fp32 lattices only");
      } else {
        rdcnn_ring_t r = nullptr;
        const int ghost = b.levels;
        const int rc = rdcnn_ring_create(rows, cols, key_.devices.data(), int(key_.devices.size()), ghost,
                                         b.mode, &r);
        if (rc == RDCNN_ECUDA && std::strstr(rdcnn_last_error(), "out of memory")) throw std::bad_alloc();
        if (rc == RDCNN_EINVAL) throw std::invalid_argument(rdcnn_last_error());
        check(rc, "rdcnn_ring_create");
        ring_.reset(r);
        return;
      }
    }
    rdcnn_sim_t h = nullptr;
    int rc;
    if constexpr (sizeof(T) == 4) {
      rc = rdcnn_sim_create(rows, cols, 1, b.device, b.mode, &h);
    } else {
      if (b.mode != RDCNN_STRICT) throw std::invalid_argument("fp64 runs in strict mode only");
      rc = rdcnn_sim_create_f64(rows, cols, 1, b.device, &h);
    }
    // Device memory exhaustion surfaces like host exhaustion does in the
    // reference (bench_suite marks such a cell skipped, bench.hpp:130-139).
    if (rc == RDCNN_ECUDA && std::strstr(rdcnn_last_error(), "out of memory")) throw std::bad_alloc();
    check(rc, "rdcnn_sim_create");
    h_.reset(h);
    const int levels = sizeof(T) == 8 ? std::min(b.levels, 4) : b.levels;
    check(rdcnn_sim_set_tuning(h, levels, 0), "rdcnn_sim_set_tuning");
  }
  void set_gene(const Gene& g) {
    const auto v = gene_to_vector(g);
    if (gene_set_ && v == gene_) return;  // unchanged: keep captured launches
    gene_ = v;
    gene_set_ = true;
    if constexpr (sizeof(T) == 4) {
      rdcnn_params_f32 p;
      rdcnn_params_from_gene(v.data(), &p);
      if (ring_) check(rdcnn_ring_set_params(ring_.get(), &p), "rdcnn_ring_set_params");
      else check(rdcnn_sim_set_params(h_.get(), &p, 1), "rdcnn_sim_set_params");
    } else {
      const rdcnn_params_f64 p{v[0], v[1], v[2], v[3], v[4], v[5], v[6]};
      check(rdcnn_sim_set_params_f64(h_.get(), &p, 1), "rdcnn_sim_set_params_f64");
    }
  }
  void upload(const GridState<T>& s) {
    if constexpr (sizeof(T) == 4) {
      if (ring_) check(rdcnn_ring_upload(ring_.get(), s.u.data(), s.v.data()), "rdcnn_ring_upload");
      else check(rdcnn_sim_upload(h_.get(), s.u.data(), s.v.data()), "rdcnn_sim_upload");
    } else {
      check(rdcnn_sim_upload_f64(h_.get(), s.u.data(), s.v.data()), "rdcnn_sim_upload_f64");
    }
  }
  void download(GridState<T>& s) {
    if constexpr (sizeof(T) == 4) {
      if (ring_) check(rdcnn_ring_download(ring_.get(), s.u.data(), s.v.data()), "rdcnn_ring_download");
      else check(rdcnn_sim_download(h_.get(), s.u.data(), s.v.data()), "rdcnn_sim_download");
    } else {
      check(rdcnn_sim_download_f64(h_.get(), s.u.data(), s.v.data()), "rdcnn_sim_download_f64");
    }
  }
  // Returns the 1-based bad iteration within this call, or 0 (exact on a
  // multi-device ring too: rdcnn_ring_advance replays the bad block).
  long advance(long steps) {
    long bad = 0;
    if (ring_) check(rdcnn_ring_advance(ring_.get(), steps, &bad), "rdcnn_ring_advance");
    else check(rdcnn_sim_advance(h_.get(), steps, &bad), "rdcnn_sim_advance");
    return bad;
  }
  // Device time of the last advance (max over devices for a ring).
  double elapsed_ms() const {
    double ms = 0;
    if (ring_) check(rdcnn_ring_elapsed_ms(ring_.get(), &ms), "rdcnn_ring_elapsed_ms");
    else check(rdcnn_sim_elapsed_ms(h_.get(), &ms), "rdcnn_sim_elapsed_ms");
    return ms;
  }
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  bool multi_device() const { return bool(ring_); }
  const SimKey& key() const { return key_; }

 private:
  struct Del {
    void operator()(rdcnn_sim_t h) const { rdcnn_sim_destroy(h); }
  };
  struct RingDel {
    void operator()(rdcnn_ring_t r) const { rdcnn_ring_destroy(r); }
  };
  std::unique_ptr<rdcnn_sim, Del> h_;
  std::unique_ptr<rdcnn_ring, RingDel> ring_;
  int rows_, cols_;
  SimKey key_;
  std::array<double, 7> gene_{};
  bool gene_set_ = false;
};

}  // namespace detail

// ===========================================================================
// StepBuffers / step
// ===========================================================================

/// Double buffer with the reference's public members.  `front` is the host
/// view of the current state; for the cuda backend the state is also held on
/// the device, created on the first step.
template <class T>
struct StepBuffers {
  GridState<T> front;
  GridState<T> back;
  std::vector<T> scratch;
  std::shared_ptr<detail::Sim<T>> device;  // cuda backend state (lazily created)

  explicit StepBuffers(GridState<T> initial) : front(std::move(initial)), back(front.rows, front.cols) {}
  int rows() const { return front.rows; }
  int cols() const { return front.cols; }
  void swap() {
    std::swap(front.u, back.u);
    std::swap(front.v, back.v);
  }
};

namespace detail {

// The buffers' device lattice for backend b: created on first use and
// re-created when b names another device set, mode or fusion depth (the
// host front buffer is uploaded on every call, so nothing is lost).
template <class T>
Sim<T>& device_for(StepBuffers<T>& bufs, const Backend& b) {
  if (!bufs.device || !(bufs.device->key() == sim_key(b))) {
    bufs.device.reset();
    bufs.device = std::make_shared<Sim<T>>(bufs.rows(), bufs.cols(), b);
  }
  return *bufs.device;
}

// Per-call protocol of kernels.hpp:233-259: upload front, advance `n`,
// download into back, swap (always).  Returns the bad iteration or 0.
template <class T>
long advance_host(StepBuffers<T>& bufs, const Gene& g, const Backend& b, long n) {
  require_cuda(b);
  Sim<T>& sim = device_for(bufs, b);
  sim.set_gene(g);
  sim.upload(bufs.front);
  const long bad = sim.advance(n);
  sim.download(bufs.back);
  bufs.swap();
  return bad;
}

}  // namespace detail

/// One iteration on the selected backend; swaps; false on a non-finite value.
template <class T>
bool step(StepBuffers<T>& bufs, const Gene& gene, const Backend& backend) {
  return detail::advance_host(bufs, gene, backend, 1) == 0;
}

/// The CellModel overload (kernels.hpp:233-259, generic over CellModel,
/// model.hpp:13-21).  The FHN model runs on the sm_100a wavefront kernels.
/// Any other model runs on the generic device stencil of
/// rdcnn/cuda_model.cuh when the caller is compiled with nvcc (model methods
/// marked __host__ __device__); a host-compiled caller cannot ship its model
/// to the GPU and gets std::invalid_argument.
template <class M, class T = typename M::value_type>
  requires CellModel<M>
bool step(StepBuffers<T>& bufs, const M& model, const Backend& backend) {
  if constexpr (std::is_same_v<M, FhnModel<T>>) {
    const FhnParams<T>& p = model.p;
    Gene g;
    g.dt = p.dt; g.a = p.a; g.b = p.b; g.eps = p.eps; g.c = p.c; g.Du = p.du; g.Dv = p.dv;
    return step(bufs, g, backend);  // float -> double -> float is exact
  } else {
#if defined(__CUDACC__)
    detail::require_cuda(backend);
    const bool ok = cuda_model::step_device<M, T>(bufs.front.u.data(), bufs.front.v.data(), bufs.back.u.data(),
                                                  bufs.back.v.data(), bufs.rows(), bufs.cols(), model,
                                                  backend.device);
    bufs.swap();
    return ok;
#else
    (void)bufs;
    (void)model;
    (void)backend;
    throw std::invalid_argument(
        "the cuda backend runs non-FHN CellModels only from nvcc-compiled code (rdcnn/cuda_model.cuh)");
#endif
  }
}

// ===========================================================================
// Run configuration and engine
// ===========================================================================

enum class InitMode : int { CenterSquare = 1, FullRandom = 2, Image = 3 };

inline InitMode parse_init_mode(int typ) {
  if (typ < 1 || typ > 3) throw std::invalid_argument("typ must be 1, 2 or 3");
  return InitMode(typ);
}

struct RunConfig {
  InitMode init_mode = InitMode::CenterSquare;
  int nn = 512;
  int nm = 512;
  std::optional<std::string> image_path;
  std::optional<int> image_size;
  long iter_max = 10000;
  int nssp = 5;
  uint64_t seed = 1;
  Backend backend;
  Precision precision = Precision::Single;
};

enum class ConfigErrorKind { InvalidSize, InvalidSchedule, MissingImage, NonFiniteGene };

struct ConfigIssue {
  ConfigErrorKind kind;
  std::string message;
};

inline std::vector<ConfigIssue> validate_config(const RunConfig& cfg, const Gene& gene) {
  std::vector<ConfigIssue> out;
  const std::string shape = std::to_string(cfg.nn) + "x" + std::to_string(cfg.nm);
  if (cfg.nn < 3 || cfg.nm < 3)
    out.push_back({ConfigErrorKind::InvalidSize, "grid must be at least 3x3, got " + shape});
  if (cfg.init_mode == InitMode::CenterSquare && (cfg.nn < 11 || cfg.nm < 11))
    out.push_back({ConfigErrorKind::InvalidSize, "typ=1 needs room for the 11x11 seed square, got " + shape});
  if (cfg.iter_max < 1)
    out.push_back({ConfigErrorKind::InvalidSchedule, "iter_max must be >= 1, got " + std::to_string(cfg.iter_max)});
  if (cfg.nssp < 1 || cfg.nssp > cfg.iter_max)
    out.push_back({ConfigErrorKind::InvalidSchedule, "nssp must satisfy 1 <= nssp <= iter_max, got nssp=" +
                                                         std::to_string(cfg.nssp) +
                                                         " iter_max=" + std::to_string(cfg.iter_max)});
  else if (cfg.iter_max >= 1 && cfg.iter_max % cfg.nssp != 0)
    out.push_back({ConfigErrorKind::InvalidSchedule, "nssp (" + std::to_string(cfg.nssp) +
                                                         ") must divide iter_max (" +
                                                         std::to_string(cfg.iter_max) + ")"});
  if (cfg.init_mode == InitMode::Image && !cfg.image_path)
    out.push_back({ConfigErrorKind::MissingImage, "typ=3 requires an image path"});
  if (!gene_finite(gene))
    out.push_back({ConfigErrorKind::NonFiniteGene, "gene has non-finite fields"});
  else if (!gene_valid(gene))
    out.push_back({ConfigErrorKind::NonFiniteGene, "gene invariant violated (need dt >= 0, Du >= 0, Dv >= 0)"});
  return out;
}

template <class T>
GridState<T> initial_state(const RunConfig& cfg, const Gene& gene,
                           const std::optional<GrayImage>& image = std::nullopt) {
  switch (cfg.init_mode) {
    case InitMode::CenterSquare: return init_center_square<T>(cfg.nn, cfg.nm, cfg.seed);
    case InitMode::FullRandom: return init_full_random<T>(cfg.nn, cfg.nm, cfg.seed);
    case InitMode::Image:
      if (!image) throw std::invalid_argument("typ=3 requires an image");
      return init_from_image<T>(*image, gene);
  }
  throw std::logic_error("unreachable init mode");
}

struct ScheduleError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct BlowUpError : std::runtime_error {
  long iteration;
  explicit BlowUpError(long iter)
      : std::runtime_error("blow-up: non-finite state after iteration " + std::to_string(iter)),
        iteration(iter) {}
};

template <class T>
struct SnapshotBuffer {
  int rows = 0, cols = 0;
  std::vector<std::vector<T>> frames_u;
  std::vector<std::vector<T>> frames_v;
  std::vector<long> labels;
  size_t frame_count() const { return labels.size(); }
};

template <class T>
struct RunOutput {
  GridState<T> final_state;
  SnapshotBuffer<T> snapshots;
  double wall_seconds = 0;
  std::vector<double> snapshot_elapsed;
};

using SnapshotCallback = std::function<void(long, double)>;

/// engine.hpp:54-94 with the state resident on the device between snapshots:
/// one advance per snapshot interval, one download per frame.
template <class T>
RunOutput<T> run(const RunConfig& cfg, const Gene& gene, GridState<T> initial,
                 const SnapshotCallback& on_snapshot = {}) {
  if (initial.rows != cfg.nn || initial.cols != cfg.nm)
    throw std::invalid_argument("initial state shape does not match config");
  if (cfg.nssp < 1 || cfg.nssp > cfg.iter_max || cfg.iter_max % cfg.nssp != 0)
    throw ScheduleError("nssp (" + std::to_string(cfg.nssp) + ") must divide iter_max (" +
                        std::to_string(cfg.iter_max) + ")");
  detail::require_cuda(cfg.backend);
  const long test_mod = cfg.iter_max / cfg.nssp;
  RunOutput<T> out;
  auto& snaps = out.snapshots;
  snaps.rows = cfg.nn;
  snaps.cols = cfg.nm;
  snaps.frames_u.push_back(initial.u);
  snaps.frames_v.push_back(initial.v);
  snaps.labels.push_back(0);

  detail::Sim<T> sim(cfg.nn, cfg.nm, cfg.backend);
  sim.set_gene(gene);
  sim.upload(initial);
  GridState<T> cur(std::move(initial));
  const auto t0 = std::chrono::steady_clock::now();
  for (long done = 0; done < cfg.iter_max; done += test_mod) {
    const long bad = sim.advance(test_mod);
    if (bad) throw BlowUpError(done + bad);
    const double elapsed =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    sim.download(cur);
    snaps.frames_u.push_back(cur.u);
    snaps.frames_v.push_back(cur.v);
    snaps.labels.push_back(done + test_mod);
    out.snapshot_elapsed.push_back(elapsed);
    if (on_snapshot) on_snapshot(done + test_mod, elapsed);
  }
  out.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  out.final_state = std::move(cur);
  return out;
}

/// engine.hpp:98-106: bare timed loop (device-resident), BlowUpError(iter).
/// Leaves bufs.front = the state after the last (or the first bad) iteration.
template <class T>
double run_timed(StepBuffers<T>& bufs, const Gene& gene, const Backend& backend, long iters) {
  detail::require_cuda(backend);
  detail::Sim<T>& sim = detail::device_for(bufs, backend);
  sim.set_gene(gene);
  sim.upload(bufs.front);
  const auto t0 = std::chrono::steady_clock::now();
  const long bad = sim.advance(iters);
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  sim.download(bufs.front);
  if (bad) throw BlowUpError(bad);
  return sec;
}

// ===========================================================================
// Throughput metric (bench.hpp:21-33)
// ===========================================================================

struct ZeroDuration : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct Throughput {
  double mcells_per_s = 0;
  double ns_per_cell_iter = 0;
};

inline Throughput throughput(long nn, long nm, long iter_max, double seconds) {
  if (!(seconds > 0)) throw ZeroDuration("throughput needs seconds > 0");
  const double work = double(nn) * double(nm) * double(iter_max);
  return {work / (seconds * 1e6), seconds * 1e9 / work};
}

// ===========================================================================
// Benchmark protocol (bench.hpp:35-253): the suite the reference's CLI
// `bench` runs, timed through run_timed on the chosen backend.
// ===========================================================================

struct BenchRecord {
  std::string backend;
  std::string hardware;
  int n = 0;
  long iters = 0;
  double seconds = 0;
  double mcells_per_s = 0;
  double ns_per_cell_iter = 0;
  uint64_t checksum = 0;
  bool skipped = false;  // the cell could not allocate (host or device)
};

/// BlowUpError inside a benchmark cell, naming the cell (bench.hpp:48-59).
struct BenchCellError : std::runtime_error {
  std::string backend;
  int n;
  long iteration;
  BenchCellError(std::string be, int size, long iter)
      : std::runtime_error("blow-up in benchmark cell backend=" + be + " N=" + std::to_string(size) +
                           " at iteration " + std::to_string(iter)),
        backend(std::move(be)),
        n(size),
        iteration(iter) {}
};

namespace detail_bench {

/// One cell: `reps` runs of run_timed from the same typ=1 state, the median
/// wall time, the checksum of the last final state (bench.hpp:63-88).
template <class T>
BenchRecord bench_cell(const Backend& backend, int n, long iter_max, const Gene& gene, uint64_t seed, int reps,
                       const std::string& hardware) {
  std::vector<double> seconds;
  uint64_t digest = 0;
  for (int rep = 0; rep < reps; ++rep) {
    StepBuffers<T> bufs(init_center_square<T>(n, n, seed));
    try {
      seconds.push_back(run_timed(bufs, gene, backend, iter_max));
    } catch (const BlowUpError& e) {
      throw BenchCellError(backend_name(backend), n, e.iteration);
    }
    digest = checksum(bufs.front);
  }
  std::sort(seconds.begin(), seconds.end());
  BenchRecord r;
  r.backend = backend_name(backend);
  r.hardware = hardware;
  r.n = n;
  r.iters = iter_max;
  r.seconds = seconds[seconds.size() / 2];
  const Throughput tp = throughput(n, n, iter_max, r.seconds);
  r.mcells_per_s = tp.mcells_per_s;
  r.ns_per_cell_iter = tp.ns_per_cell_iter;
  r.checksum = digest;
  return r;
}

template <class T>
void warm_up(const Backend& backend, int n, long iter_max, const Gene& gene, uint64_t seed) {
  StepBuffers<T> bufs(init_center_square<T>(n, n, seed));
  try {
    run_timed(bufs, gene, backend, std::min<long>(iter_max, 100));
  } catch (const BlowUpError& e) {
    throw BenchCellError(backend_name(backend), n, e.iteration);
  }
}

inline std::string printf_g(const char* fmt, double x) {
  char buf[64];
  std::snprintf(buf, sizeof buf, fmt, x);
  return buf;
}

/// A double as a JSON number in the form the reference's JSON library
/// writes it: round-trip digits, fixed notation with a ".0" on integral
/// values for decimal exponents in (-4, 15], else d.ddde+XX.  Byte-identical
/// to the reference's emit_json except for rare 17-digit values, where its
/// Grisu2 picks a different last digit of the same double (11 of ~8000 random
/// doubles; both strings parse back to the same value).
inline std::string json_number(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
  std::string s(buf, res.ptr);
  std::string sign;
  if (s[0] == '-') {
    sign = "-";
    s.erase(0, 1);
  }
  const size_t e = s.find('e');
  const int point = std::stoi(s.substr(e + 1)) + 1;  // decimal point position after the first digit
  std::string digits = s.substr(0, e);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int k = int(digits.size());
  std::string out;
  if (k <= point && point <= 15) {
    out = digits + std::string(size_t(point - k), '0') + ".0";
  } else if (0 < point && point <= 15) {
    out = digits.substr(0, size_t(point)) + "." + digits.substr(size_t(point));
  } else if (-4 < point && point <= 0) {
    out = "0." + std::string(size_t(-point), '0') + digits;
  } else {
    out = digits.substr(0, 1) + (k > 1 ? "." + digits.substr(1) : std::string());
    const int ex = point - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += eb;
  }
  return sign + out;
}

inline std::string json_string(const std::string& s) {
  std::string out = "\"";
  for (const unsigned char c : s) {
    if (c == '"' || c == '\\') {
      out += '\\';
      out += char(c);
    } else if (c < 0x20) {
      char eb[8];
      std::snprintf(eb, sizeof eb, "\\u%04x", c);
      out += eb;
    } else {
      out += char(c);
    }
  }
  return out + "\"";
}

}  // namespace detail_bench

/// Times every (backend, N) cell on the typ=1 workload (bench.hpp:92-145):
/// one discarded warm-up run per backend before its first cell, the median
/// of `reps` per cell, no snapshots.  A cell that cannot allocate is marked
/// skipped; a blow-up throws BenchCellError.
inline std::vector<BenchRecord> bench_suite(const std::vector<Backend>& backends, const std::vector<int>& sizes,
                                            long iter_max, const Gene& gene, uint64_t seed,
                                            Precision precision = Precision::Single, int reps = 3,
                                            const std::string& hardware = "cpu") {
  if (iter_max < 1) throw std::invalid_argument("bench needs iter_max >= 1");
  if (reps < 1) throw std::invalid_argument("bench needs reps >= 1");
  for (const int n : sizes)
    if (n < 11) throw std::invalid_argument("bench sizes must be >= 11 (typ=1 seed square)");
  const bool single = precision == Precision::Single;
  std::vector<BenchRecord> records;
  for (const Backend& backend : backends) {
    bool warmed = false;
    for (const int n : sizes) {
      try {
        if (!warmed) {
          single ? detail_bench::warm_up<float>(backend, n, iter_max, gene, seed)
                 : detail_bench::warm_up<double>(backend, n, iter_max, gene, seed);
          warmed = true;
        }
        records.push_back(single ? detail_bench::bench_cell<float>(backend, n, iter_max, gene, seed, reps, hardware)
                                 : detail_bench::bench_cell<double>(backend, n, iter_max, gene, seed, reps,
                                                                    hardware));
      } catch (const std::bad_alloc&) {
        BenchRecord r;
        r.backend = backend_name(backend);
        r.hardware = hardware;
        r.n = n;
        r.iters = iter_max;
        r.skipped = true;
        records.push_back(r);
      }
    }
  }
  return records;
}

/// The documented CSV columns; skipped cells are left out (bench.hpp:163-178).
inline std::string emit_csv(const std::vector<BenchRecord>& records) {
  if (records.empty()) throw std::invalid_argument("no benchmark records");
  std::string out = "backend,hardware,n,iters,seconds,mcells_per_s,ns_per_cell_iter,checksum\n";
  for (const BenchRecord& r : records) {
    if (r.skipped) continue;
    out += r.backend + "," + r.hardware + "," + std::to_string(r.n) + "," + std::to_string(r.iters) + "," +
           detail_bench::printf_g("%.5g", r.seconds) + "," + detail_bench::printf_g("%.5g", r.mcells_per_s) + "," +
           detail_bench::printf_g("%.5g", r.ns_per_cell_iter) + "," + checksum_hex(r.checksum) + "\n";
  }
  return out;
}

/// Backend-by-size matrix, each cell "mcells (seconds)", "-" where skipped
/// or absent; a hardware column only when the records carry more than one
/// hardware label (bench.hpp:180-228).
inline std::string emit_table(const std::vector<BenchRecord>& records) {
  if (records.empty()) throw std::invalid_argument("no benchmark records");
  std::vector<int> sizes;
  std::vector<std::pair<std::string, std::string>> keys;  // (backend, hardware), first-seen order
  for (const BenchRecord& r : records) {
    if (std::find(sizes.begin(), sizes.end(), r.n) == sizes.end()) sizes.push_back(r.n);
    const auto key = std::make_pair(r.backend, r.hardware);
    if (std::find(keys.begin(), keys.end(), key) == keys.end()) keys.push_back(key);
  }
  std::sort(sizes.begin(), sizes.end());
  const bool multi_hw = std::any_of(keys.begin(), keys.end(), [&](const auto& k) { return k.second != keys[0].second; });
  auto find = [&](const std::pair<std::string, std::string>& key, int n) -> const BenchRecord* {
    const BenchRecord* hit = nullptr;  // the last record of a repeated cell wins
    for (const BenchRecord& r : records)
      if (r.backend == key.first && r.hardware == key.second && r.n == n) hit = &r;
    return hit;
  };
  std::vector<std::vector<std::string>> cells;
  std::vector<std::string> head{"backend"};
  if (multi_hw) head.push_back("hardware");
  for (const int n : sizes) head.push_back("N=" + std::to_string(n));
  cells.push_back(head);
  for (const auto& key : keys) {
    std::vector<std::string> line{key.first};
    if (multi_hw) line.push_back(key.second);
    for (const int n : sizes) {
      const BenchRecord* r = find(key, n);
      line.push_back(!r || r->skipped ? std::string("-")
                                      : detail_bench::printf_g("%.5g", r->mcells_per_s) + " (" +
                                            detail_bench::printf_g("%.4g", r->seconds) + ")");
    }
    cells.push_back(line);
  }
  std::vector<size_t> width(head.size(), 0);
  for (const auto& line : cells)
    for (size_t c = 0; c < line.size(); ++c) width[c] = std::max(width[c], line[c].size());
  std::string out;
  for (const auto& line : cells) {
    for (size_t c = 0; c < line.size(); ++c) {
      out += line[c];
      if (c + 1 < line.size()) out += std::string(width[c] - line[c].size() + 2, ' ');
    }
    out += "\n";
  }
  return out;
}

/// The CSV fields as a JSON array, two-space indented with keys in sorted
/// order; checksums as hex strings (bench.hpp:230-251).
inline std::string emit_json(const std::vector<BenchRecord>& records) {
  if (records.empty()) throw std::invalid_argument("no benchmark records");
  using detail_bench::json_number;
  using detail_bench::json_string;
  std::string out = "[\n";
  for (size_t i = 0; i < records.size(); ++i) {
    const BenchRecord& r = records[i];
    std::vector<std::pair<std::string, std::string>> kv{{"backend", json_string(r.backend)},
                                                        {"hardware", json_string(r.hardware)},
                                                        {"iters", std::to_string(r.iters)},
                                                        {"n", std::to_string(r.n)}};
    if (r.skipped) {
      kv.emplace_back("skipped", "true");
    } else {
      kv.emplace_back("checksum", json_string(checksum_hex(r.checksum)));
      kv.emplace_back("mcells_per_s", json_number(r.mcells_per_s));
      kv.emplace_back("ns_per_cell_iter", json_number(r.ns_per_cell_iter));
      kv.emplace_back("seconds", json_number(r.seconds));
    }
    std::sort(kv.begin(), kv.end());
    out += "  {\n";
    for (size_t k = 0; k < kv.size(); ++k)
      out += "    \"" + kv[k].first + "\": " + kv[k].second + (k + 1 < kv.size() ? ",\n" : "\n");
    out += i + 1 < records.size() ? "  },\n" : "  }\n";
  }
  return out + "]\n";
}

// ===========================================================================
// Parameter-plane sweeps (sweep.hpp:16-326) on one batched device handle
// ===========================================================================
//
// The reference runs |x|*|y| independent run() calls and classifies every
// snapshot on the host.  Here every cell is one grid of a batched handle
// (per-grid gene, per-grid blow-up iteration); the snapshots stay on the
// device, where the classifier's statistics are computed (min/max, the
// nth_element median, active counts); only per-grid scalars and the final
// states come back.  Labels, digests and labels_csv equal the reference's.
// Not here: the PNG panel and write_sweep_outputs (image rendering and file
// output are out of scope; the Python layer writes the CSV and frames).

enum class Regime { Homogeneous, Patterned, Growing, BlowUp };

inline const char* regime_name(Regime r) {
  switch (r) {
    case Regime::Homogeneous: return "Homogeneous";
    case Regime::Patterned: return "Patterned";
    case Regime::Growing: return "Growing";
    case Regime::BlowUp: return "BlowUp";
  }
  return "?";
}

struct ClassifierConfig {
  double homogeneity_rel = 0.01;
  double homogeneity_floor = 0.01;
  double activity_rel = 0.1;
  double growth_factor = 10.0;
  double dip_tolerance = 0.10;
};

struct RegimeResult {
  Regime label = Regime::Patterned;
  double final_range = 0;
  double final_active_fraction = 0;
  std::vector<long> activity_counts;  // one per snapshot frame
};

/// Shortest decimal form that round-trips the double (config.hpp:102-106).
inline std::string format_double(double x) {
  char buf[32];
  const auto res = std::to_chars(buf, buf + sizeof buf, x);
  return std::string(buf, res.ptr);
}

namespace detail_sweep {

// classify_outcome's decision (sweep.hpp:73-112) from per-frame u statistics:
// mins/maxs per frame, the per-frame active counts at threshold
// activity_rel * final_range, and the cell count.
inline RegimeResult classify(const std::vector<double>& mins, const std::vector<double>& maxs,
                             std::vector<long> counts, size_t cells, const ClassifierConfig& cc) {
  RegimeResult res;
  res.final_range = maxs.back() - mins.back();
  const double gmin = *std::min_element(mins.begin(), mins.end());
  const double gmax = *std::max_element(maxs.begin(), maxs.end());
  const double homog = std::max(cc.homogeneity_floor, cc.homogeneity_rel * (gmax - gmin));
  res.activity_counts = std::move(counts);
  res.final_active_fraction = double(res.activity_counts.back()) / double(cells);
  if (res.final_range < homog) {
    res.label = Regime::Homogeneous;
    return res;
  }
  bool rising = true;
  for (size_t k = 0; k + 1 < res.activity_counts.size(); ++k)
    rising &= double(res.activity_counts[k + 1]) >= (1.0 - cc.dip_tolerance) * double(res.activity_counts[k]);
  const bool grew = res.activity_counts.back() >=
                    std::max<long>(1, long(cc.growth_factor * double(res.activity_counts.front())));
  res.label = rising && grew ? Regime::Growing : Regime::Patterned;
  return res;
}

}  // namespace detail_sweep

/// Per-frame count of cells whose u deviates from the frame's median (the
/// element std::nth_element puts at n/2) by more than `threshold`
/// (sweep.hpp:46-64; host-side, for snapshot buffers the caller holds).
template <class T>
std::vector<long> growth_curve(const SnapshotBuffer<T>& snaps, double threshold) {
  std::vector<long> counts;
  std::vector<T> sorted;
  for (const auto& frame : snaps.frames_u) {
    sorted = frame;
    std::nth_element(sorted.begin(), sorted.begin() + sorted.size() / 2, sorted.end());
    const double median = double(sorted[sorted.size() / 2]);
    counts.push_back(long(std::count_if(frame.begin(), frame.end(),
                                        [&](T x) { return std::abs(double(x) - median) > threshold; })));
  }
  return counts;
}

/// classify_outcome (sweep.hpp:66-112) over a host snapshot buffer.
template <class T>
RegimeResult classify_outcome(const SnapshotBuffer<T>& snaps, const ClassifierConfig& cc = {}) {
  std::vector<double> mins, maxs;
  for (const auto& frame : snaps.frames_u) {
    const auto [mn, mx] = std::minmax_element(frame.begin(), frame.end());
    mins.push_back(double(*mn));
    maxs.push_back(double(*mx));
  }
  const double final_range = maxs.back() - mins.back();
  return detail_sweep::classify(mins, maxs, growth_curve(snaps, cc.activity_rel * final_range),
                                snaps.frames_u.back().size(), cc);
}

struct SweepSpec {
  std::string x_param;
  std::vector<double> x_values;
  std::string y_param;
  std::vector<double> y_values;
  Gene base_gene;
  RunConfig base_config;
  bool keep_buffers = false;   // retain full snapshot buffers per cell
  bool per_cell_seed = false;  // seed + cell index instead of one shared seed
  bool parallel_cells = false; // accepted for source compatibility: cells always run batched
  std::optional<std::pair<double, double>> fixed_range;  // panel option (no panel here)
  ClassifierConfig classifier;
  // typ=3 sweeps: the decoded image (the reference loads base_config.image_path;
  // image decoding is outside this library).
  std::optional<GrayImage> image;
};

inline void validate_sweep_spec(const SweepSpec& spec) {
  if (!is_gene_field(spec.x_param)) throw std::invalid_argument("unknown sweep parameter: " + spec.x_param);
  if (!is_gene_field(spec.y_param)) throw std::invalid_argument("unknown sweep parameter: " + spec.y_param);
  if (spec.x_param == spec.y_param)
    throw std::invalid_argument("sweep axes must differ (both are " + spec.x_param + ")");
  if (spec.x_values.empty() || spec.y_values.empty())
    throw std::invalid_argument("sweep value lists must be non-empty");
}

template <class T>
struct SweepCell {
  double x_value = 0, y_value = 0;
  Gene gene;
  bool blew_up = false;
  long blowup_iteration = 0;
  RegimeResult outcome;
  uint64_t digest = 0;
  std::vector<T> final_u;
  std::optional<SnapshotBuffer<T>> buffer;
};

template <class T>
struct SweepResult {
  std::vector<double> x_values, y_values;
  std::string x_param, y_param;
  int rows = 0, cols = 0;
  std::vector<SweepCell<T>> cells;  // row-major: y outer, x inner
  std::string labels_csv;
  const SweepCell<T>& at(size_t yi, size_t xi) const { return cells[yi * x_values.size() + xi]; }
};

namespace detail_sweep {

template <class T>
std::string labels_csv(const SweepResult<T>& res) {
  std::string out = "x_value,y_value,label,final_range,final_active_fraction,checksum\n";
  for (size_t yi = 0; yi < res.y_values.size(); ++yi)
    for (size_t xi = 0; xi < res.x_values.size(); ++xi) {
      const SweepCell<T>& c = res.at(yi, xi);
      out += format_double(c.x_value) + "," + format_double(c.y_value) + "," + regime_name(c.outcome.label) + ",";
      if (c.blew_up) {
        out += ",,\n";
        continue;
      }
      out += detail_bench::printf_g("%.6g", c.outcome.final_range) + "," +
             detail_bench::printf_g("%.6g", c.outcome.final_active_fraction) + "," + checksum_hex(c.digest) + "\n";
    }
  return out;
}

// The per-thread batched handle sweep_grid<T> keeps for its next call.
struct SimDel {
  void operator()(rdcnn_sim_t h) const { rdcnn_sim_destroy(h); }
};
struct SweepCache {
  std::array<int, 6> key{};
  std::unique_ptr<rdcnn_sim, SimDel> h;
};
template <class T>
SweepCache& sweep_cache() {
  static thread_local SweepCache c;
  return c;
}

}  // namespace detail_sweep

/// Frees the calling thread's cached sweep handles (fp32 and fp64), e.g.
/// before cudaDeviceReset or when a worker thread is done sweeping.
inline void release_sweep_cache() {
  detail_sweep::sweep_cache<float>().h.reset();
  detail_sweep::sweep_cache<double>().h.reset();
}

/// sweep_grid (sweep.hpp:249-326): |x|*|y| cells, one shared seed unless
/// per_cell_seed, blow-ups recorded per cell (never fatal), all cells as the
/// grids of one batched handle on base_config.backend's device.
template <class T>
SweepResult<T> sweep_grid(const SweepSpec& spec) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>);
  validate_sweep_spec(spec);
  RunConfig base = spec.base_config;
  detail::require_cuda(base.backend);
  for (const ConfigIssue& issue : validate_config(base, spec.base_gene))
    if (!(issue.kind == ConfigErrorKind::MissingImage && spec.image)) throw std::invalid_argument(issue.message);
  if (base.iter_max % base.nssp != 0) throw ScheduleError("nssp must divide iter_max for sweep cells");
  if (base.init_mode == InitMode::Image) {
    if (!spec.image) throw std::invalid_argument("typ=3 sweeps need SweepSpec::image (the decoded image)");
    base.nn = spec.image->rows;
    base.nm = spec.image->cols;
  }
  SweepResult<T> res;
  res.x_values = spec.x_values;
  res.y_values = spec.y_values;
  res.x_param = spec.x_param;
  res.y_param = spec.y_param;
  res.rows = base.nn;
  res.cols = base.nm;
  for (const double y : spec.y_values)
    for (const double x : spec.x_values) {
      SweepCell<T> c;
      c.x_value = x;
      c.y_value = y;
      c.gene = spec.base_gene;
      gene_field(c.gene, spec.x_param) = x;
      gene_field(c.gene, spec.y_param) = y;
      if (!gene_valid(c.gene))
        throw std::invalid_argument("sweep cell gene invalid at " + spec.x_param + "=" + format_double(x) + " " +
                                    spec.y_param + "=" + format_double(y));
      res.cells.push_back(std::move(c));
    }

  const int B = int(res.cells.size()), rows = base.nn, cols = base.nm;
  const size_t n = size_t(rows) * cols, nb = size_t(B);
  const Backend& be = base.backend;
  // The batched handle is kept (per thread) for the next sweep of the same
  // shape: creating and destroying one allocates and frees the whole batch
  // and its snapshot frames, which the driver made cost up to seconds.
  // release_sweep_cache() frees it.  The cache is filled only once the
  // handle is fully configured, so a failed configuration is not reused.
  detail_sweep::SweepCache& cached = detail_sweep::sweep_cache<T>();
  const std::array<int, 6> key{rows, cols, B, be.device, be.mode, be.levels};
  if (!cached.h || cached.key != key) {
    cached.h.reset();
    rdcnn_sim_t raw = nullptr;
    int rc;
    if constexpr (sizeof(T) == 4) {
      rc = rdcnn_sim_create(rows, cols, B, be.device, be.mode, &raw);
    } else {
      if (be.mode != RDCNN_STRICT) throw std::invalid_argument("fp64 runs in strict mode only");
      rc = rdcnn_sim_create_f64(rows, cols, B, be.device, &raw);
    }
    if (rc == RDCNN_ECUDA && std::strstr(rdcnn_last_error(), "out of memory")) throw std::bad_alloc();
    detail::check(rc, "rdcnn_sim_create (sweep batch)");
    std::unique_ptr<rdcnn_sim, detail_sweep::SimDel> fresh(raw);
    const int trc = rdcnn_sim_set_tuning(raw, sizeof(T) == 8 ? std::min(be.levels, 4) : be.levels, 0);
    if (trc == RDCNN_EINVAL) throw std::invalid_argument(rdcnn_last_error());
    detail::check(trc, "rdcnn_sim_set_tuning");
    cached.h = std::move(fresh);
    cached.key = key;
  }
  rdcnn_sim* const h_raw = cached.h.get();
  struct View {  // the calls below take h.get()
    rdcnn_sim* p;
    rdcnn_sim* get() const { return p; }
  } const h{h_raw};

  // Per-grid genes, narrowed like make_params<T> (model.hpp:24-32).
  if constexpr (sizeof(T) == 4) {
    std::vector<rdcnn_params_f32> p(nb);
    for (int g = 0; g < B; ++g) rdcnn_params_from_gene(gene_to_vector(res.cells[size_t(g)].gene).data(), &p[size_t(g)]);
    detail::check(rdcnn_sim_set_params(h.get(), p.data(), B), "rdcnn_sim_set_params");
  } else {
    std::vector<rdcnn_params_f64> p(nb);
    for (int g = 0; g < B; ++g) {
      const auto v = gene_to_vector(res.cells[size_t(g)].gene);
      p[size_t(g)] = rdcnn_params_f64{v[0], v[1], v[2], v[3], v[4], v[5], v[6]};
    }
    detail::check(rdcnn_sim_set_params_f64(h.get(), p.data(), B), "rdcnn_sim_set_params_f64");
  }
  // Initial states (init.hpp:67-82): the shared-seed typ 1/2 default is drawn
  // on the device; per-cell seeds and images are built here and uploaded.
  auto upload = [&](const std::vector<T>& u, const std::vector<T>& v) {
    if constexpr (sizeof(T) == 4)
      detail::check(rdcnn_sim_upload(h.get(), u.data(), v.data()), "rdcnn_sim_upload");
    else
      detail::check(rdcnn_sim_upload_f64(h.get(), u.data(), v.data()), "rdcnn_sim_upload_f64");
  };
  auto download = [&](std::vector<T>& u, std::vector<T>& v) {
    if constexpr (sizeof(T) == 4)
      detail::check(rdcnn_sim_download(h.get(), u.data(), v.data()), "rdcnn_sim_download");
    else
      detail::check(rdcnn_sim_download_f64(h.get(), u.data(), v.data()), "rdcnn_sim_download_f64");
  };
  if (base.init_mode != InitMode::Image && !spec.per_cell_seed) {
    detail::check(rdcnn_sim_init(h.get(), int(base.init_mode), base.seed), "rdcnn_sim_init");
  } else {
    std::vector<T> U(n * nb), V(n * nb);
    for (int g = 0; g < B; ++g) {
      RunConfig cfg = base;
      if (spec.per_cell_seed) cfg.seed = base.seed + uint64_t(g);
      const GridState<T> s = initial_state<T>(cfg, res.cells[size_t(g)].gene, spec.image);
      std::copy(s.u.begin(), s.u.end(), U.begin() + std::ptrdiff_t(n * size_t(g)));
      std::copy(s.v.begin(), s.v.end(), V.begin() + std::ptrdiff_t(n * size_t(g)));
    }
    upload(U, V);
  }

  // The run (engine.hpp:54-94): nssp advances of test_mod, a device frame
  // of every grid's u plane before the first and after each.
  const long test_mod = base.iter_max / base.nssp;
  const int F = base.nssp + 1;
  const size_t nf = size_t(F);
  std::vector<std::vector<T>> keep_u, keep_v;  // full states per frame (keep_buffers)
  auto keep = [&]() {
    if (!spec.keep_buffers) return;
    keep_u.emplace_back(n * nb);
    keep_v.emplace_back(n * nb);
    download(keep_u.back(), keep_v.back());
  };
  detail::check(rdcnn_sim_frames_reserve(h.get(), F), "rdcnn_sim_frames_reserve");
  detail::check(rdcnn_sim_frame_capture(h.get(), 0), "rdcnn_sim_frame_capture");
  keep();
  std::vector<long> bad(nb, 0);
  for (int f = 1; f < F; ++f) {
    detail::check(rdcnn_sim_advance(h.get(), test_mod, bad.data()), "rdcnn_sim_advance");
    for (int g = 0; g < B; ++g) {
      SweepCell<T>& c = res.cells[size_t(g)];
      if (bad[size_t(g)] && !c.blew_up) {
        c.blew_up = true;
        c.blowup_iteration = long(f - 1) * test_mod + bad[size_t(g)];
        c.outcome.label = Regime::BlowUp;
      }
    }
    detail::check(rdcnn_sim_frame_capture(h.get(), f), "rdcnn_sim_frame_capture");
    keep();
  }

  // Classifier statistics per frame and grid, on the device.
  const std::vector<double> per_grid(nb, 0.0);
  std::vector<std::vector<double>> mins(nf, per_grid), maxs(nf, per_grid), meds(nf, per_grid);
  for (int f = 0; f < F; ++f)
    detail::check(rdcnn_sim_frame_stats(h.get(), f, mins[size_t(f)].data(), maxs[size_t(f)].data(),
                                        meds[size_t(f)].data()),
                  "rdcnn_sim_frame_stats");
  std::vector<double> thr(nb);
  for (int g = 0; g < B; ++g)
    thr[size_t(g)] = spec.classifier.activity_rel * (maxs[size_t(F - 1)][size_t(g)] - mins[size_t(F - 1)][size_t(g)]);
  std::vector<std::vector<long long>> counts(nf, std::vector<long long>(nb, 0));
  for (int f = 0; f < F; ++f)
    detail::check(rdcnn_sim_frame_active(h.get(), f, meds[size_t(f)].data(), thr.data(), counts[size_t(f)].data()),
                  "rdcnn_sim_frame_active");
  std::vector<uint64_t> digests(nb);
  detail::check(rdcnn_sim_checksums(h.get(), digests.data()), "rdcnn_sim_checksums");
  std::vector<T> fu(n * nb), fv(n * nb);
  download(fu, fv);

  for (int g = 0; g < B; ++g) {
    SweepCell<T>& c = res.cells[size_t(g)];
    if (c.blew_up) continue;
    std::vector<double> mn(nf), mx(nf);
    std::vector<long> cnt(nf);
    for (int f = 0; f < F; ++f) {
      mn[size_t(f)] = mins[size_t(f)][size_t(g)];
      mx[size_t(f)] = maxs[size_t(f)][size_t(g)];
      cnt[size_t(f)] = long(counts[size_t(f)][size_t(g)]);
    }
    c.outcome = detail_sweep::classify(mn, mx, std::move(cnt), n, spec.classifier);
    c.digest = digests[size_t(g)];
    const auto off = std::ptrdiff_t(n * size_t(g));
    c.final_u.assign(fu.begin() + off, fu.begin() + off + std::ptrdiff_t(n));
    if (spec.keep_buffers) {
      SnapshotBuffer<T> sb;
      sb.rows = rows;
      sb.cols = cols;
      for (int f = 0; f < F; ++f) {
        sb.frames_u.emplace_back(keep_u[size_t(f)].begin() + off, keep_u[size_t(f)].begin() + off + std::ptrdiff_t(n));
        sb.frames_v.emplace_back(keep_v[size_t(f)].begin() + off, keep_v[size_t(f)].begin() + off + std::ptrdiff_t(n));
        sb.labels.push_back(long(f) * test_mod);
      }
      c.buffer = std::move(sb);
    }
  }
  res.labels_csv = detail_sweep::labels_csv(res);
  return res;
}

}  // namespace rdcnn
