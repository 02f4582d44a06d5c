// ref_cuda_driver.cpp -- the reference's OWN headers (proj/include, patched
// at build time by integration/reference_cuda_backend.patch into a temporary
// copy) with the new `cuda` backend beside its CPU backends.  Runs the
// reference's acceptance criterion 1 (acceptance_main.cpp:76-100, backend
// equivalence) with cuda added, criterion 10's 64^2 known answer through the
// per-step path (kernels.hpp:233-259), the blow-up iteration of
// test_engine.cpp:82-108 through run_timed (engine.hpp:98-106), and the
// double instantiation.  Exit code = failed checks.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "rdcnn/backend.hpp"
#include "rdcnn/engine.hpp"
#include "rdcnn/init.hpp"

using namespace rdcnn;

static int g_pass = 0, g_fail = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    if (c) {                                                             \
      ++g_pass;                                                          \
    } else {                                                             \
      ++g_fail;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);           \
    }                                                                    \
  } while (0)

template <class T>
static uint64_t criterion1(const Backend& b) {
  RunConfig cfg;
  cfg.nn = cfg.nm = 256;
  cfg.iter_max = 1000;
  cfg.nssp = 1;
  cfg.seed = 42;
  cfg.backend = b;
  auto out = run(cfg, Gene{}, init_center_square<T>(256, 256, 42));
  return checksum(out.final_state);
}

int main() {
  // Criterion 1 with the cuda backend beside the reference's own backends
  // (the CPU backends stay; "cuda" is one more kind).
  const std::vector<Backend> backends = {Backend{BackendKind::Reference}, Backend{BackendKind::Blocked, 64, 64},
                                         Backend{BackendKind::Parallel, 64, 64, 4}, make_backend("cuda")};
  std::vector<uint64_t> d;
  for (const Backend& b : backends) {
    d.push_back(criterion1<float>(b));
    std::printf("criterion 1 %-9s %s\n", backend_name(b), checksum_hex(d.back()).c_str());
  }
  for (uint64_t x : d) CHECK(x == d[0]);
  CHECK(checksum_hex(d[0]) == "1026befcb693b1e5");  // test_output.txt:8
  CHECK(make_backend("cuda").exact_order() && backend_name(make_backend("cuda")) == std::string("cuda"));

  // Criterion 10 (64^2 x 200, test_output.txt:23) through step() per call.
  for (const Backend& b : {Backend{BackendKind::Reference}, make_backend("cuda")}) {
    StepBuffers<float> bufs(init_center_square<float>(64, 64, 42));
    const FhnModel<float> m(Gene{});
    bool ok = true;
    for (int k = 0; k < 200; ++k) ok &= step(bufs, m, b);
    std::printf("criterion 10 %-9s %s (per-step)\n", backend_name(b), checksum_hex(checksum(bufs.front)).c_str());
    CHECK(ok && checksum_hex(checksum(bufs.front)) == "ced829150965fba9");
  }

  // Blow-up iteration (test_engine.cpp:95) through run_timed, and the state
  // it leaves behind: the same cells non-finite, the finite ones equal.
  Gene g;
  g.dt = 100;
  std::vector<long> its;
  std::vector<GridState<float>> fronts;
  for (const Backend& b : {Backend{BackendKind::Reference}, make_backend("cuda")}) {
    StepBuffers<float> bufs(init_center_square<float>(16, 16, 42));
    long it = 0;
    try {
      run_timed(bufs, g, b, 1000);
    } catch (const BlowUpError& e) {
      it = e.iteration;
    }
    std::printf("blow-up %-9s iteration %ld\n", backend_name(b), it);
    its.push_back(it);
    fronts.push_back(bufs.front);
  }
  CHECK(its[0] == 4 && its[1] == its[0]);
  bool same = true;
  for (size_t k = 0; k < fronts[0].u.size(); ++k) {
    const float a = fronts[0].u[k], b = fronts[1].u[k];
    same &= std::isfinite(a) == std::isfinite(b) && (!std::isfinite(a) || a == b);
  }
  CHECK(same);

  // The double instantiation (grid.hpp:13-28).
  const uint64_t r64 = criterion1<double>(Backend{BackendKind::Parallel, 64, 64, 4});
  const uint64_t c64 = criterion1<double>(make_backend("cuda"));
  std::printf("criterion 1 (double) parallel %s cuda %s\n", checksum_hex(r64).c_str(), checksum_hex(c64).c_str());
  CHECK(r64 == c64);

  std::printf("ref-binding: %d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
