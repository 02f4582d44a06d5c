// rdcnn/config.hpp -- run configuration: InitMode, RunConfig, validate_config, format_double
// (reference proj/include/rdcnn/config.hpp:20-106), for the cuda backend: implemented
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
#include "rdcnn/backend.hpp"
#include "rdcnn/gene.hpp"
#include "rdcnn/grid.hpp"

namespace rdcnn {

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


/// Shortest decimal form that round-trips the double (config.hpp:102-106).
inline std::string format_double(double x) {
  char buf[32];
  const auto res = std::to_chars(buf, buf + sizeof buf, x);
  return std::string(buf, res.ptr);
}

}  // namespace rdcnn
