// rdcnn/backend.hpp -- backend selection: BackendKind (+Cuda), Backend, make_backend
// (reference proj/include/rdcnn/backend.hpp:12-50), for the cuda backend: implemented
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

}  // namespace rdcnn
