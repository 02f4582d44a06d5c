/*
 * fhn_oracle.c -- CPU restatement of the reference FitzHugh-Nagumo RD-CNN
 * time-stepping path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product path
 * (paper_2102_10340_b200/, include/) never links or calls it.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks this file against the
 * reference's recorded known answers (proj/test_output.txt:8, :23,
 * test_engine.cpp:95, test_model.cpp:19-58, test_kernels.cpp:37-50) and
 * against oracle/_ref (the reference headers themselves, compiled by
 * oracle/Makefile) on the fixtures under tests/golden/.
 *
 * Arithmetic contract: every expression below is written in the reference's
 * evaluation order and must be compiled with -ffp-contract=off and without
 * -ffast-math (reference proj/CMakeLists.txt:23-25), so that each operation
 * is one IEEE-754 round-to-nearest step, subnormals preserved.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

/* ---- RNG: splitmix64 (reference proj/include/rdcnn/rng.hpp:11-39) ------- */

static uint64_t orc_mix(uint64_t *state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);          /* rng.hpp:18 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;             /* rng.hpp:19 */
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;             /* rng.hpp:20 */
  return z ^ (z >> 31);                                    /* rng.hpp:21 */
}

/* rng.hpp:28: float(u64 >> 40) * 2^-24 */
static float orc_unit_f32(uint64_t *s) { return (float)(orc_mix(s) >> 40) * 0x1.0p-24f; }
/* rng.hpp:25: double(u64 >> 11) * 2^-53 */
static double orc_unit_f64(uint64_t *s) { return (double)(orc_mix(s) >> 11) * 0x1.0p-53; }

uint64_t orc_rng_u64(uint64_t seed, uint64_t index) {
  uint64_t s = seed;
  uint64_t z = 0;
  for (uint64_t k = 0; k <= index; ++k) z = orc_mix(&s);
  return z;
}

/* ---- gene narrowing (model.hpp:24-32: {dt,a,b,eps,c,du,dv}, T(g.x)) ----- */

void orc_params_f32(const double gene7[7], float out[7]) {
  for (int k = 0; k < 7; ++k) out[k] = (float)gene7[k];
}

/* ---- templated body, instantiated for float and double ----------------- */

#define ORC_DEFINE(T, SFX, UNIT, EXPMASK, UINT)                                 \
                                                                               \
  /* model.hpp:37-40  u*(c - u*u/3) - v */                                     \
  T orc_reaction_u_##SFX(T u, T v, const T p[7]) {                             \
    return u * (p[4] - u * u / (T)3) - v;                                      \
  }                                                                            \
  /* model.hpp:43-46  -eps*(u - b*v + a) */                                    \
  T orc_reaction_v_##SFX(T u, T v, const T p[7]) {                             \
    return -p[3] * (u - p[2] * v + p[1]);                                      \
  }                                                                            \
  /* model.hpp:51-56 */                                                        \
  void orc_cell_update_##SFX(T u, T v, T lu, T lv, const T p[7], T *un,        \
                             T *vn) {                                          \
    *un = u + p[0] * (orc_reaction_u_##SFX(u, v, p) + p[5] * lu);              \
    *vn = v + p[0] * (orc_reaction_v_##SFX(u, v, p) + p[6] * lv);              \
  }                                                                            \
                                                                               \
  /* kernels.hpp:44-56: right + left + down + up - 4*center, down = i+1 */     \
  T orc_laplacian5_##SFX(const T *x, int rows, int cols, int i, int j) {       \
    int iu = (i == 0) ? rows - 1 : i - 1;                                      \
    int id = (i == rows - 1) ? 0 : i + 1;                                      \
    int jl = (j == 0) ? cols - 1 : j - 1;                                      \
    int jr = (j == cols - 1) ? 0 : j + 1;                                      \
    T c = x[(size_t)i * cols + j];                                             \
    T r = x[(size_t)i * cols + jr];                                            \
    T l = x[(size_t)i * cols + jl];                                            \
    T d = x[(size_t)id * cols + j];                                            \
    T up = x[(size_t)iu * cols + j];                                           \
    return r + l + d + up - (T)4 * c;                                          \
  }                                                                            \
                                                                               \
  static int orc_finite_##SFX(T x) { /* grid.hpp:58-67 */                      \
    UINT b;                                                                    \
    memcpy(&b, &x, sizeof b);                                                  \
    return (b & EXPMASK) != EXPMASK;                                           \
  }                                                                            \
                                                                               \
  /* kernels.hpp:86-107 (step_reference).  Returns 1 if every written value   \
   * is finite. */                                                             \
  int orc_step_##SFX(int rows, int cols, const T *u, const T *v, T *un, T *vn, \
                     const T p[7]) {                                           \
    unsigned bad = 0;                                                          \
    for (int i = 0; i < rows; ++i) {                                           \
      for (int j = 0; j < cols; ++j) {                                         \
        size_t c = (size_t)i * cols + j;                                       \
        T uc = u[c], vc = v[c];                                                \
        T lu = orc_laplacian5_##SFX(u, rows, cols, i, j);                      \
        T lv = orc_laplacian5_##SFX(v, rows, cols, i, j);                      \
        T a = uc + p[0] * (orc_reaction_u_##SFX(uc, vc, p) + p[5] * lu);       \
        T b = vc + p[0] * (orc_reaction_v_##SFX(uc, vc, p) + p[6] * lv);       \
        un[c] = a;                                                             \
        vn[c] = b;                                                             \
        bad |= (unsigned)!orc_finite_##SFX(a);                                 \
        bad |= (unsigned)!orc_finite_##SFX(b);                                 \
      }                                                                        \
    }                                                                          \
    return bad == 0;                                                           \
  }                                                                            \
                                                                               \
  /* engine.hpp:98-106 (run_timed): iters steps, double-buffered; the result  \
   * is left in (u,v).  Returns 0, or the 1-based iteration of the first      \
   * non-finite step (the state is then the state after that step).  */       \
  long orc_run_##SFX(int rows, int cols, T *u, T *v, T *su, T *sv,             \
                     const T p[7], long iters) {                               \
    size_t n = (size_t)rows * cols;                                            \
    T *fu = u, *fv = v, *bu = su, *bv = sv;                                    \
    long bad_iter = 0;                                                         \
    for (long it = 0; it < iters; ++it) {                                      \
      int ok = orc_step_##SFX(rows, cols, fu, fv, bu, bv, p);                  \
      T *t = fu; fu = bu; bu = t;                                              \
      t = fv; fv = bv; bv = t;                                                 \
      if (!ok) { bad_iter = it + 1; break; }                                   \
    }                                                                          \
    if (fu != u) {                                                             \
      memcpy(u, fu, n * sizeof(T));                                            \
      memcpy(v, fv, n * sizeof(T));                                            \
    }                                                                          \
    return bad_iter;                                                           \
  }                                                                            \
                                                                               \
  /* init.hpp:20-30 (typ=2) */                                                 \
  void orc_init_full_random_##SFX(int rows, int cols, uint64_t seed, T *u,     \
                                  T *v) {                                      \
    uint64_t s = seed;                                                         \
    size_t n = (size_t)rows * cols;                                            \
    for (size_t k = 0; k < n; ++k) u[k] = UNIT(&s);                            \
    for (size_t k = 0; k < n; ++k) v[k] = UNIT(&s);                            \
  }                                                                            \
                                                                               \
  /* init.hpp:34-48 (typ=1): 11x11 block at ((rows-11)/2, (cols-11)/2) */      \
  int orc_init_center_square_##SFX(int rows, int cols, uint64_t seed, T *u,    \
                                   T *v) {                                     \
    if (rows < 11 || cols < 11) return -1;                                     \
    size_t n = (size_t)rows * cols;                                            \
    memset(u, 0, n * sizeof(T));                                               \
    memset(v, 0, n * sizeof(T));                                               \
    int i0 = (rows - 11) / 2, j0 = (cols - 11) / 2;                            \
    uint64_t s = seed;                                                         \
    for (int i = i0; i < i0 + 11; ++i)                                         \
      for (int j = j0; j < j0 + 11; ++j) u[(size_t)i * cols + j] = UNIT(&s);   \
    for (int i = i0; i < i0 + 11; ++i)                                         \
      for (int j = j0; j < j0 + 11; ++j) v[(size_t)i * cols + j] = UNIT(&s);   \
    return 0;                                                                  \
  }                                                                            \
                                                                               \
  /* init.hpp:51-64 + image.hpp:283: x = px/255.0 (double); u=v=T(ka)*T(x) */  \
  void orc_init_from_image_##SFX(const uint8_t *px, size_t n, double ka, T *u, \
                                 T *v) {                                       \
    T k = (T)ka;                                                               \
    for (size_t i = 0; i < n; ++i) {                                           \
      T x = k * (T)(px[i] / 255.0);                                            \
      u[i] = x;                                                                \
      v[i] = x;                                                                \
    }                                                                          \
  }

ORC_DEFINE(float, f32, orc_unit_f32, 0x7F800000u, uint32_t)
ORC_DEFINE(double, f64, orc_unit_f64, 0x7FF0000000000000ull, uint64_t)

/* ---- digest: FNV-1a 64 over raw bytes of u then v (grid.hpp:101-116) ---- */

uint64_t orc_fnv1a(const void *data, size_t n, uint64_t h) {
  const unsigned char *p = (const unsigned char *)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t orc_checksum(const void *u, const void *v, size_t bytes_per_plane) {
  uint64_t h = orc_fnv1a(u, bytes_per_plane, 0xcbf29ce484222325ull);
  return orc_fnv1a(v, bytes_per_plane, h);
}
