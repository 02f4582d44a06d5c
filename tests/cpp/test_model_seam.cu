// test_model_seam.cu -- the CellModel seam (model.hpp:13-21) on the device:
// the reference's "kernels accept any CellModel: pure diffusion conserves
// mass" (test_kernels.cpp:228-256) re-expressed on the cuda backend through
// rdcnn/cuda_model.cuh, plus exactness checks.  Compiled by nvcc
// (-std=c++20 -fmad=false) in __graft_entry__.build(); run on a GPU by
// tests/test_cpp_api_gpu.py.  Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "rdcnn/engine.hpp"
#include "rdcnn/init.hpp"

using namespace rdcnn;

namespace {

int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) {                                                            \
      ++g_pass;                                                            \
    } else {                                                               \
      ++g_fail;                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)

// test_kernels.cpp:228-240: a minimal non-FHN model (methods marked for the device).
struct PureDiffusion {
  using value_type = float;
  RDCNN_HD float reaction_u(float, float) const { return 0.0f; }
  RDCNN_HD float reaction_v(float, float) const { return 0.0f; }
  RDCNN_HD float diffusion_u() const { return 0.1f; }
  RDCNN_HD float diffusion_v() const { return 0.1f; }
  RDCNN_HD float time_step() const { return 0.5f; }
};
static_assert(CellModel<PureDiffusion>);

// FitzHugh-Nagumo written as a user model (model.hpp:37-56 formulas, IEEE
// division): through the generic seam it must equal the built-in kernels.
struct UserFhn {
  using value_type = float;
  float dt, a, b, eps, c, du, dv;
  RDCNN_HD float reaction_u(float u, float v) const { return u * (c - u * u / 3.0f) - v; }
  RDCNN_HD float reaction_v(float u, float v) const { return -eps * (u - b * v + a); }
  RDCNN_HD float diffusion_u() const { return du; }
  RDCNN_HD float diffusion_v() const { return dv; }
  RDCNN_HD float time_step() const { return dt; }
};

// The same arithmetic on the host (-ffp-contract=off), the exact-order check.
template <class M>
void host_step(const M& m, const GridState<float>& s, GridState<float>& o) {
  const int R = s.rows, C = s.cols;
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < C; ++j) {
      const int iu = i == 0 ? R - 1 : i - 1, id = i == R - 1 ? 0 : i + 1;
      const int jl = j == 0 ? C - 1 : j - 1, jr = j == C - 1 ? 0 : j + 1;
      const size_t c = (size_t)i * C + j;
      const float uc = s.u[c], vc = s.v[c];
      const float lu = s.u[(size_t)i * C + jr] + s.u[(size_t)i * C + jl] + s.u[(size_t)id * C + j] +
                       s.u[(size_t)iu * C + j] - 4.0f * uc;
      const float lv = s.v[(size_t)i * C + jr] + s.v[(size_t)i * C + jl] + s.v[(size_t)id * C + j] +
                       s.v[(size_t)iu * C + j] - 4.0f * vc;
      o.u[c] = uc + m.time_step() * (m.reaction_u(uc, vc) + m.diffusion_u() * lu);
      o.v[c] = vc + m.time_step() * (m.reaction_v(uc, vc) + m.diffusion_v() * lv);
    }
}

// A model whose output overflows (non-finite detection).
struct Explode {
  using value_type = float;
  RDCNN_HD float reaction_u(float u, float) const { return u * 1e38f; }
  RDCNN_HD float reaction_v(float, float) const { return 0.0f; }
  RDCNN_HD float diffusion_u() const { return 0.0f; }
  RDCNN_HD float diffusion_v() const { return 0.0f; }
  RDCNN_HD float time_step() const { return 10.0f; }
};

bool same_bits(const std::vector<float>& a, const std::vector<float>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0;
}

}  // namespace

int main() {
  // test_kernels.cpp:242-256: 50 steps of pure diffusion conserve the u mass.
  {
    GridState<float> s = init_full_random<float>(16, 16, 17);
    double before = 0;
    for (float x : s.u) before += x;
    GridState<float> ref = s, tmp(16, 16);
    StepBuffers<float> bufs(std::move(s));
    bool ok = true;
    for (int k = 0; k < 50; ++k) {
      ok = ok && step(bufs, PureDiffusion{}, Backend{});
      host_step(PureDiffusion{}, ref, tmp);
      std::swap(ref, tmp);
    }
    CHECK(ok);
    double after = 0;
    for (float x : bufs.front.u) after += x;
    CHECK(std::fabs(after - before) <= 1e-4 * std::fabs(before));
    CHECK(same_bits(bufs.front.u, ref.u) && same_bits(bufs.front.v, ref.v));  // exact order
  }
  // A user-written FHN model through the seam == the built-in FHN kernels.
  {
    const Gene g;  // reference default gene
    const FhnParams<float> p = make_params<float>(g);
    const UserFhn um{p.dt, p.a, p.b, p.eps, p.c, p.du, p.dv};
    GridState<float> s = init_full_random<float>(40, 52, 9);
    StepBuffers<float> seam(s), builtin(s);
    for (int k = 0; k < 30; ++k) {
      CHECK(step(seam, um, Backend{}));
      CHECK(step(builtin, g, Backend{}));
    }
    CHECK(same_bits(seam.front.u, builtin.front.u) && same_bits(seam.front.v, builtin.front.v));
  }
  // Non-finite results are reported (and the buffers still swap).
  {
    StepBuffers<float> bufs(init_full_random<float>(8, 8, 3));
    const std::vector<float> before = bufs.front.u;
    CHECK(!step(bufs, Explode{}, Backend{}));
    CHECK(same_bits(bufs.back.u, before));  // swapped: the old front is now back
  }
  std::printf("model seam: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
