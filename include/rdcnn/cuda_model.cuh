// rdcnn/cuda_model.cuh -- the CellModel seam on the device (nvcc only).
//
// The reference's kernels are generic over any CellModel (model.hpp:13-21):
// reaction_u/v, diffusion_u/v, time_step.  The sm_100a wavefront kernel is
// specialised to FitzHugh-Nagumo; this header keeps the seam for other models.
// Include it from a .cu file compiled with nvcc, with the model's methods
// marked __host__ __device__ (RDCNN_HD), and
//
//     rdcnn::step(bufs, MyModel{}, rdcnn::Backend{})
//
// runs the model on the GPU: one plain one-level stencil kernel, the
// canonical kern::stencil_cell arithmetic (kernels.hpp:63-72) with one IEEE
// round-to-nearest operation per source operation, in the reference order.
// The call follows step()'s per-call protocol: compute into `back`, swap,
// and return false on any non-finite value (kernels.hpp:233-259).  Build the
// model with -fmad=false (as the reference builds with -ffp-contract=off)
// for results bit-identical to the reference CPU backends.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#ifndef RDCNN_HD
#define RDCNN_HD __host__ __device__
#endif

namespace rdcnn {
namespace cuda_model {

__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// kern::stencil_cell over the torus, one thread per cell (grid-stride).
template <class M, class T>
__global__ void model_step_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ un,
                                  T* __restrict__ vn, int rows, int cols, const M m, unsigned* bad) {
  const long long n = (long long)rows * cols;
  unsigned local = 0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = int(c / cols), j = int(c - (long long)i * cols);
    const long long iu = i == 0 ? rows - 1 : i - 1, id = i == rows - 1 ? 0 : i + 1;  // kernels.hpp:46-49
    const int jl = j == 0 ? cols - 1 : j - 1, jr = j == cols - 1 ? 0 : j + 1;
    const long long r = (long long)i * cols + jr, l = (long long)i * cols + jl;
    const long long dn = id * cols + j, up = iu * cols + j;
    const T uc = u[c], vc = v[c];
    // right + left + down + up - 4*center, down = row i+1
    const T lap_u = sub_rn(add_rn(add_rn(add_rn(u[r], u[l]), u[dn]), u[up]), mul_rn(T(4), uc));
    const T lap_v = sub_rn(add_rn(add_rn(add_rn(v[r], v[l]), v[dn]), v[up]), mul_rn(T(4), vc));
    const T dt = m.time_step();
    const T nu = add_rn(uc, mul_rn(dt, add_rn(m.reaction_u(uc, vc), mul_rn(m.diffusion_u(), lap_u))));
    const T nv = add_rn(vc, mul_rn(dt, add_rn(m.reaction_v(uc, vc), mul_rn(m.diffusion_v(), lap_v))));
    un[c] = nu;
    vn[c] = nv;
    local |= unsigned(!isfinite(nu)) | unsigned(!isfinite(nv));
  }
  if (local) atomicOr(bad, 1u);
}

// Device scratch of the calling thread (one per element type), grown on
// demand and re-allocated when the calling thread moves to another device.
template <class T>
struct Scratch {
  T* d = nullptr;
  unsigned* bad = nullptr;
  size_t cells = 0;
  int device = -1;
  void release() {
    if (device >= 0) cudaSetDevice(device);
    if (d) cudaFree(d);
    if (bad) cudaFree(bad);
    d = nullptr;
    bad = nullptr;
    cells = 0;
  }
  ~Scratch() { release(); }
  void ensure(size_t n, int dev) {
    if (dev != device) {
      release();
      device = dev;
    }
    if (cudaSetDevice(dev) != cudaSuccess) throw std::runtime_error("cuda_model: cudaSetDevice");
    if (n <= cells) return;
    if (d) cudaFree(d);
    d = nullptr;
    if (cudaMalloc(&d, 4 * n * sizeof(T)) != cudaSuccess) throw std::runtime_error("cuda_model: out of device memory");
    if (!bad && cudaMalloc(&bad, sizeof(unsigned)) != cudaSuccess) throw std::runtime_error("cuda_model: cudaMalloc");
    cells = n;
  }
};

// One step of model m on CUDA device `device` (Backend::device).
template <class M, class T>
bool step_device(T* front_u, T* front_v, T* back_u, T* back_v, int rows, int cols, const M& m, int device = 0) {
  static thread_local Scratch<T> s;
  const size_t n = (size_t)rows * cols;
  s.ensure(n, device);
  T *du = s.d, *dv = s.d + n, *dun = s.d + 2 * n, *dvn = s.d + 3 * n;
  auto ok = [](cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("cuda_model: ") + what + ": " + cudaGetErrorString(e));
  };
  ok(cudaMemcpy(du, front_u, n * sizeof(T), cudaMemcpyHostToDevice), "upload u");
  ok(cudaMemcpy(dv, front_v, n * sizeof(T), cudaMemcpyHostToDevice), "upload v");
  ok(cudaMemset(s.bad, 0, sizeof(unsigned)), "memset");
  const long long blocks = ((long long)n + 255) / 256;
  model_step_kernel<M, T><<<(unsigned)(blocks < 65536 ? blocks : 65536), 256>>>(du, dv, dun, dvn, rows, cols, m,
                                                                               s.bad);
  ok(cudaGetLastError(), "launch");
  unsigned bad = 0;
  ok(cudaMemcpy(back_u, dun, n * sizeof(T), cudaMemcpyDeviceToHost), "download u");
  ok(cudaMemcpy(back_v, dvn, n * sizeof(T), cudaMemcpyDeviceToHost), "download v");
  ok(cudaMemcpy(&bad, s.bad, sizeof bad, cudaMemcpyDeviceToHost), "download flag");
  return bad == 0;
}

}  // namespace cuda_model
}  // namespace rdcnn
