// ref_driver.cpp -- C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/rdcnn, read-only, never copied).  TEST
// INFRASTRUCTURE ONLY: built by oracle/Makefile into oracle/_ref/librdcnn_ref.so
// and loaded only by tests/ and by bench.py's cpu_baseline / --impl reference
// arm.  Each entry point calls the reference's own public API:
//   init_center_square / init_full_random   (init.hpp:20-48)
//   run_timed on a named backend             (engine.hpp:98-106, backend.hpp:44-50)
//   run with snapshots                       (engine.hpp:54-94)
//   checksum                                 (grid.hpp:101-116)
// Kept in its own shared object so the reference's inline definitions never
// meet the product's rdcnn:: types (ODR), see SURVEY.md §7 step 1.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "rdcnn/engine.hpp"
#include "rdcnn/init.hpp"
#include "rdcnn/sweep.hpp"

using namespace rdcnn;

namespace {

Gene gene_from(const double g8[8]) {
  // order: dt, a, b, eps, c, du, dv, ka  (gene_to_vector order + ka, gene.hpp:39-41)
  std::array<double, 7> p{g8[0], g8[1], g8[2], g8[3], g8[4], g8[5], g8[6]};
  return vector_to_gene(p, g8[7]);
}

template <class T>
GridState<T> make_state(int rows, int cols, const T* u, const T* v) {
  GridState<T> s(rows, cols);
  std::memcpy(s.u.data(), u, s.cells() * sizeof(T));
  std::memcpy(s.v.data(), v, s.cells() * sizeof(T));
  return s;
}

template <class T>
int init_dispatch(int typ, int rows, int cols, uint64_t seed, T* u, T* v) {
  try {
    GridState<T> s = typ == 1 ? init_center_square<T>(rows, cols, seed)
                              : init_full_random<T>(rows, cols, seed);
    std::memcpy(u, s.u.data(), s.cells() * sizeof(T));
    std::memcpy(v, s.v.data(), s.cells() * sizeof(T));
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Returns 0 ok, 2 blow-up (bad_iter set), 1 invalid argument.
template <class T>
int run_timed_dispatch(int rows, int cols, T* u, T* v, const double g8[8],
                       const char* backend, int threads, long iters, long* bad_iter,
                       double* seconds) {
  try {
    Backend be = make_backend(backend, 64, 64, threads);
    StepBuffers<T> bufs(make_state<T>(rows, cols, u, v));
    if (bad_iter) *bad_iter = 0;
    int rc = 0;
    try {
      double s = run_timed(bufs, gene_from(g8), be, iters);
      if (seconds) *seconds = s;
    } catch (const BlowUpError& e) {
      if (bad_iter) *bad_iter = e.iteration;
      rc = 2;
    }
    std::memcpy(u, bufs.front.u.data(), bufs.front.cells() * sizeof(T));
    std::memcpy(v, bufs.front.v.data(), bufs.front.cells() * sizeof(T));
    return rc;
  } catch (const std::exception&) {
    return 1;
  }
}

}  // namespace

extern "C" {

int ref_init_f32(int typ, int rows, int cols, uint64_t seed, float* u, float* v) {
  return init_dispatch<float>(typ, rows, cols, seed, u, v);
}
int ref_init_f64(int typ, int rows, int cols, uint64_t seed, double* u, double* v) {
  return init_dispatch<double>(typ, rows, cols, seed, u, v);
}

int ref_run_timed_f32(int rows, int cols, float* u, float* v, const double g8[8],
                      const char* backend, int threads, long iters, long* bad_iter,
                      double* seconds) {
  return run_timed_dispatch<float>(rows, cols, u, v, g8, backend, threads, iters,
                                   bad_iter, seconds);
}
int ref_run_timed_f64(int rows, int cols, double* u, double* v, const double g8[8],
                      const char* backend, int threads, long iters, long* bad_iter,
                      double* seconds) {
  return run_timed_dispatch<double>(rows, cols, u, v, g8, backend, threads, iters,
                                    bad_iter, seconds);
}

// engine.hpp:54-94 with snapshots.  frames_u/frames_v hold (nssp+1) planes
// each; labels holds nssp+1 entries.  Returns 0 ok, 2 blow-up, 3 schedule
// error, 1 other invalid argument.
int ref_run_f32(int rows, int cols, const float* u0, const float* v0,
                const double g8[8], const char* backend, long iter_max, int nssp,
                float* frames_u, float* frames_v, long* labels, long* bad_iter) {
  try {
    RunConfig cfg;
    cfg.nn = rows;
    cfg.nm = cols;
    cfg.iter_max = iter_max;
    cfg.nssp = nssp;
    cfg.backend = make_backend(backend);
    auto out = run(cfg, gene_from(g8), make_state<float>(rows, cols, u0, v0));
    const size_t n = size_t(rows) * cols;
    for (size_t f = 0; f < out.snapshots.frame_count(); ++f) {
      std::memcpy(frames_u + f * n, out.snapshots.frames_u[f].data(), n * sizeof(float));
      std::memcpy(frames_v + f * n, out.snapshots.frames_v[f].data(), n * sizeof(float));
      labels[f] = out.snapshots.labels[f];
    }
    return 0;
  } catch (const BlowUpError& e) {
    if (bad_iter) *bad_iter = e.iteration;
    return 2;
  } catch (const ScheduleError&) {
    return 3;
  } catch (const std::exception&) {
    return 1;
  }
}

uint64_t ref_checksum_f32(int rows, int cols, const float* u, const float* v) {
  return checksum(make_state<float>(rows, cols, u, v));
}
uint64_t ref_checksum_f64(int rows, int cols, const double* u, const double* v) {
  return checksum(make_state<double>(rows, cols, u, v));
}

// sweep_grid (sweep.hpp:255-326) on a typ 1/2 base config; writes the
// labels CSV (sweep.hpp:227-247) into out (NUL-terminated).  Returns 0, or
// 1 on invalid arguments / short buffer.
int ref_sweep_labels_impl(const char* x_param, const double* xs, int nx, const char* y_param,
                          const double* ys, int ny, const double g8[8], int typ, int nn, int nm,
                          long iter_max, int nssp, uint64_t seed, int per_cell_seed, char* out,
                          size_t cap, bool parallel_cells) {
  try {
    SweepSpec spec;
    spec.x_param = x_param;
    spec.y_param = y_param;
    spec.x_values.assign(xs, xs + nx);
    spec.y_values.assign(ys, ys + ny);
    spec.base_gene = gene_from(g8);
    spec.base_config.init_mode = parse_init_mode(typ);
    spec.base_config.nn = nn;
    spec.base_config.nm = nm;
    spec.base_config.iter_max = iter_max;
    spec.base_config.nssp = nssp;
    spec.base_config.seed = seed;
    // parallel_cells: cells run concurrently (sweep.hpp:293-295), each on the
    // single-threaded reference backend; otherwise one cell at a time on the
    // parallel backend.  The labels are the same either way.
    spec.base_config.backend = make_backend(parallel_cells ? "reference" : "parallel");
    spec.parallel_cells = parallel_cells;
    spec.per_cell_seed = per_cell_seed != 0;
    auto res = sweep_grid<float>(spec);
    if (res.labels_csv.size() + 1 > cap) return 1;
    std::memcpy(out, res.labels_csv.c_str(), res.labels_csv.size() + 1);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int ref_sweep_labels_f32(const char* x_param, const double* xs, int nx, const char* y_param,
                         const double* ys, int ny, const double g8[8], int typ, int nn, int nm,
                         long iter_max, int nssp, uint64_t seed, int per_cell_seed, char* out,
                         size_t cap) {
  return ref_sweep_labels_impl(x_param, xs, nx, y_param, ys, ny, g8, typ, nn, nm, iter_max, nssp, seed,
                               per_cell_seed, out, cap, false);
}

int ref_sweep_labels_par_f32(const char* x_param, const double* xs, int nx, const char* y_param,
                             const double* ys, int ny, const double g8[8], int typ, int nn, int nm,
                             long iter_max, int nssp, uint64_t seed, int per_cell_seed, char* out,
                             size_t cap) {
  return ref_sweep_labels_impl(x_param, xs, nx, y_param, ys, ny, g8, typ, nn, nm, iter_max, nssp, seed,
                               per_cell_seed, out, cap, true);
}

// std::to_chars shortest form (config.hpp:103-107), for checking the
// product's labels formatting.
int ref_format_double(double x, char* out, size_t cap) {
  std::string s = format_double(x);
  if (s.size() + 1 > cap) return 1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

// manifest_text (config.hpp:109-134) for a typ 1/2 config on a named backend.
int ref_manifest_text(const double g8[8], int typ, int nn, int nm, long iter_max, int nssp,
                      uint64_t seed, const char* backend, int precision_double, char* out,
                      size_t cap) {
  try {
    RunConfig cfg;
    cfg.init_mode = parse_init_mode(typ);
    cfg.nn = nn;
    cfg.nm = nm;
    cfg.iter_max = iter_max;
    cfg.nssp = nssp;
    cfg.seed = seed;
    cfg.backend = make_backend(backend);
    cfg.precision = precision_double ? Precision::Double : Precision::Single;
    std::string s = manifest_text(gene_from(g8), cfg);
    if (s.size() + 1 > cap) return 1;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// write_png / write_pgm (image.hpp:96-174) of a rows x cols 8-bit raster.
int ref_write_image(const char* path, int rows, int cols, const uint8_t* px, int png) {
  try {
    Image8 img{rows, cols, std::vector<uint8_t>(px, px + size_t(rows) * cols)};
    if (png)
      write_png(path, img);
    else
      write_pgm(path, img);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// normalize_frame<float> (frame.hpp:28-44) into out; lo/hi returned.
int ref_normalize_frame_f32(const float* layer, int rows, int cols, uint8_t* out, double* lo,
                            double* hi) {
  Frame8 f = normalize_frame(std::span<const float>(layer, size_t(rows) * cols), rows, cols);
  std::memcpy(out, f.px.data(), f.px.size());
  *lo = f.lo;
  *hi = f.hi;
  return 0;
}

// typ=3 initial state through the reference's own image path:
// load_grayscale (image.hpp:273-290) + init_from_image (init.hpp:52-62).
int ref_init_image_f32(const char* path, double ka, int* rows, int* cols, float* u, float* v, size_t cap) {
  try {
    GrayImage img = load_grayscale(path);
    Gene g;
    g.ka = ka;
    GridState<float> s = init_from_image<float>(img, g);
    *rows = s.rows;
    *cols = s.cols;
    if (s.cells() > cap) return 1;
    std::memcpy(u, s.u.data(), s.cells() * sizeof(float));
    std::memcpy(v, s.v.data(), s.cells() * sizeof(float));
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

/* OpenMP threads for the reference's own parallel regions that take no
 * explicit count (sweep.hpp:293 parallel_cells); torchrun presets 1. */
void ref_set_threads(int n) {
#if defined(_OPENMP)
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int ref_max_threads(void) {
#if defined(_OPENMP)
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
