// rdcnn/sweep.hpp -- parameter-plane sweeps on one batched device handle: Regime, ClassifierConfig, growth_curve, classify_outcome, SweepSpec, SweepCell, SweepResult, sweep_grid
// (reference proj/include/rdcnn/sweep.hpp:16-326), for the cuda backend: implemented
// over the C-ABI in include/rdcnn_cuda.h.  Part of the source-compatible
// drop-in API; rdcnn/cuda_api.hpp includes every part.
#pragma once

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
#include "rdcnn/bench.hpp"
#include "rdcnn/config.hpp"
#include "rdcnn/engine.hpp"
#include "rdcnn/init.hpp"

namespace rdcnn {

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
