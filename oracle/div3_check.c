/*
 * div3_check.c -- exhaustive proof, over all 2^32 fp32 bit patterns, that the
 * three-instruction quotient used by the product kernel
 *
 *     q0 = RN(x * R)            R = RN(1/3) = 0x3EAAAAAB
 *     e  = RN(fma(-q0, 3, x))   (exact remainder)
 *     q  = RN(fma(e, R, q0))
 *
 * equals the IEEE quotient RN(x / 3) of reference model.hpp:39 (u*u/T(3)) for
 * every finite x, and is non-finite whenever x is non-finite.  TEST
 * INFRASTRUCTURE ONLY (called from tests/test_oracle.py); the GPU repeats the
 * same sweep on its own FMA/FMUL units in tests/test_parity_gpu.py.
 *
 * Build flags must keep every operation separately rounded: -ffp-contract=off,
 * no -ffast-math, and a hardware fmaf (-mfma) so the sweep takes seconds.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static float as_f(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t as_u(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

/* Returns the number of mismatching bit patterns in [lo, hi) (hi <= 2^32);
 * the first mismatch is written to *first_bad (or left untouched). */
uint64_t div3_sweep(uint64_t lo, uint64_t hi, uint32_t *first_bad) {
  const float R = as_f(0x3EAAAAABu);
  uint64_t bad = 0;
  uint32_t first = 0xFFFFFFFFu;
#pragma omp parallel for schedule(static) reduction(+ : bad) reduction(min : first)
  for (int64_t k = (int64_t)lo; k < (int64_t)hi; ++k) {
    uint32_t bits = (uint32_t)k;
    float x = as_f(bits);
    float want = x / 3.0f;
    float q0 = x * R;
    float e = fmaf(-q0, 3.0f, x);
    float q = fmaf(e, R, q0);
    int ok;
    if (isfinite(x))
      ok = as_u(q) == as_u(want);
    else
      ok = !isfinite(q);
    if (!ok) {
      bad += 1;
      if (bits < first) first = bits;
    }
  }
  if (bad && first_bad) *first_bad = first;
  return bad;
}

/*
 * The gated two-op quotient of the strict fp32 kernel (fhn_stencil.cuh
 * div3_rn2):  q2 = RN(fma(x, R, RN(x * C))),  C = RN(1/3 - R) = 0xB22AAAAB.
 *
 * mode 0: count the x >= +0 (sign bit clear, NaN included) where q2 differs
 *         from IEEE RN(x/3) (finite x) or is finite (non-finite x); *lo_bad /
 *         *hi_bad receive the smallest / largest such bit pattern.
 * mode 1: the composite the kernel actually evaluates, RN(c - x/3)
 *         (model.hpp:39), at the gate boundary c = +-2^-90 and at c = 1:
 *         count the x >= +0 where RN(c - q2) != RN(c - RN(x/3)) (or where
 *         exactly one of them is finite).
 */
uint64_t div3_two_op_sweep(int mode, uint32_t *lo_bad, uint32_t *hi_bad) {
  const float R = as_f(0x3EAAAAABu);
  const float C = as_f(0xB22AAAABu);
  const float cs[3] = {as_f(0x12800000u) /* 2^-90 */, as_f(0x92800000u) /* -2^-90 */, 1.0f};
  uint64_t bad = 0;
  uint32_t lo = 0xFFFFFFFFu, hi = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad) reduction(min : lo) reduction(max : hi)
  for (int64_t k = 0; k <= 0x7FFFFFFFLL; ++k) {
    const uint32_t bits = (uint32_t)k;
    const float x = as_f(bits);
    const float want = x / 3.0f;
    const float q2 = fmaf(x, R, x * C);
    int ok = 1;
    if (mode == 0) {
      ok = isfinite(x) ? as_u(q2) == as_u(want) : !isfinite(q2);
    } else {
      for (int j = 0; j < 3; ++j) {
        const float a = cs[j] - q2, b = cs[j] - want;
        if (isfinite(a) != isfinite(b) || (isfinite(a) && as_u(a) != as_u(b))) ok = 0;
      }
    }
    if (!ok) {
      bad += 1;
      if (bits < lo) lo = bits;
      if (bits > hi) hi = bits;
    }
  }
  if (lo_bad) *lo_bad = lo;
  if (hi_bad) *hi_bad = hi;
  return bad;
}
