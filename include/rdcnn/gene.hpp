// rdcnn/gene.hpp -- the parameter gene: Gene, gene_valid, gene_to_vector, vector_to_gene, gene_field, stability_advisory
// (reference proj/include/rdcnn/gene.hpp:13-85), for the cuda backend: implemented
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

}  // namespace rdcnn
