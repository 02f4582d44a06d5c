// rdcnn/rng.hpp -- the seeded splitmix64 stream: SeededRng
// (reference proj/include/rdcnn/rng.hpp:11-39), for the cuda backend: implemented
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

namespace rdcnn {

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

}  // namespace rdcnn
