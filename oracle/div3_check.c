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
