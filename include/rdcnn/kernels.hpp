// rdcnn/kernels.hpp -- the device handle and the per-call step: StepBuffers, step
// (reference proj/include/rdcnn/kernels.hpp:22-259), for the cuda backend: implemented
// over the C-ABI in include/rdcnn_cuda.h.  Part of the source-compatible
// drop-in API; rdcnn/cuda_api.hpp includes every part.
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
#include "rdcnn/backend.hpp"
#include "rdcnn/gene.hpp"
#include "rdcnn/grid.hpp"
#include "rdcnn/model.hpp"

namespace rdcnn {

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

}  // namespace rdcnn
