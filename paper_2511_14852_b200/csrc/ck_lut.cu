// Device-side LUT construction: T_k on a uniform grid, float64 build
// precision, bit-identical to the reference's lut_build (lut.py:76-94).
#include <cfloat>
#include <cstring>
#include <vector>

#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

// grid node i: -1 + step*i (numpy evaluates step*arange first), last = 1.0
__device__ __forceinline__ double grid_node(int i, int n, double step) {
  return i == n - 1 ? 1.0 : __dadd_rn(-1.0, __dmul_rn(step, static_cast<double>(i)));
}

// One thread per node: walk the recurrence T_{k+1} = (2t) T_k - T_{k-1}
// (basis.py:112-119; no FMA contraction so rounding matches numpy) for the
// node and its right neighbour, emitting values and the cell slope.
__global__ void lut_build_kernel(int degree, int n, double step, double* __restrict__ v64,
                                 float* __restrict__ v_pm, float* __restrict__ s_pm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int K = degree + 1;
  const double t0 = grid_node(i, n, step);
  const bool has_right = i + 1 < n;
  const double t1 = has_right ? grid_node(i + 1, n, step) : 0.0;
  const double two_t0 = __dmul_rn(2.0, t0), two_t1 = __dmul_rn(2.0, t1);
  double p0 = 1.0, c0 = t0, p1 = 1.0, c1 = t1;  // T_{k-1}, T_k at both nodes
  for (int k = 0; k < K; ++k) {
    double a, b;
    if (k == 0) {
      a = 1.0;
      b = 1.0;
    } else if (k == 1) {
      a = t0;
      b = t1;
    } else {
      a = __dsub_rn(__dmul_rn(two_t0, c0), p0);
      b = __dsub_rn(__dmul_rn(two_t1, c1), p1);
      p0 = c0;
      c0 = a;
      p1 = c1;
      c1 = b;
    }
    v64[static_cast<int64_t>(k) * n + i] = a;
    v_pm[static_cast<int64_t>(i) * K + k] = __double2float_rn(a);
    if (has_right) s_pm[static_cast<int64_t>(i) * K + k] = __double2float_rn(__ddiv_rn(__dsub_rn(b, a), step));
  }
}

// Reference cell of float32 input x (lut.py:97-106 after kernels.py:288).
__device__ __forceinline__ int ref_cell(float x, int n) {
  int idx;
  double fr, t;
  cell_f64(x, n, idx, fr, t);
  return idx;
}

// dxrows[i] = {boundary_i, slope_1..slope_d of cell i}; boundary_i is the
// smallest float32 x with ref_cell(x) >= i, found from atanh(node_i) by
// stepping one float32 ulp at a time (ref_cell is monotone in x).
__global__ void lut_dxrows_kernel(int K, int n, double step, const float* __restrict__ s_pm,
                                  float* __restrict__ rows) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float b;
  if (i == 0) {
    b = -INFINITY;
  } else if (i >= n - 1) {
    b = INFINITY;  // cell n-1 is never selected (idx = min(., n-2))
  } else {
    const double node = __dadd_rn(-1.0, __dmul_rn(step, static_cast<double>(i)));
    float x = __double2float_rn(atanh(node));
    if (isinf(x)) x = copysignf(FLT_MAX, x);
    int guard = 0;
    while (ref_cell(x, n) >= i && guard++ < 4096) x = nextafterf(x, -INFINITY);
    guard = 0;
    while (ref_cell(x, n) < i && guard++ < 4096) x = nextafterf(x, INFINITY);
    b = x;
  }
  rows[static_cast<int64_t>(i) * K] = b;
  for (int k = 1; k < K; ++k)
    rows[static_cast<int64_t>(i) * K + k] = i < n - 1 ? s_pm[static_cast<int64_t>(i) * K + k] : 0.0f;
}

__global__ void lut_pack_kernel(int K, int n, const double* __restrict__ v64, const float* __restrict__ s_fm,
                                float* __restrict__ v_pm, float* __restrict__ s_pm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < K; ++k) {
    v_pm[static_cast<int64_t>(i) * K + k] = __double2float_rn(v64[static_cast<int64_t>(k) * n + i]);
    if (i + 1 < n) s_pm[static_cast<int64_t>(i) * K + k] = s_fm[static_cast<int64_t>(k) * (n - 1) + i];
  }
}

int lut_alloc(int degree, int lut_size, int device, ck_lut** out) {
  CK_CHECK(out != nullptr, "ck_lut: out handle pointer is NULL");
  CK_CHECK(lut_size >= 2, "lut_size must be >= 2");
  CK_CHECK(degree >= 0, "degree must be >= 0, got " + std::to_string(degree));
  CK_CHECK(degree <= 255, "degree must be <= 255");
  CK_CHECK(static_cast<int64_t>(lut_size) * (degree + 1) < (int64_t(1) << 31), "lut too large");
  CK_CUDA(cudaSetDevice(device));
  ck_lut* l = new ck_lut();
  l->degree = degree;
  l->n_feat = degree + 1;
  l->lut_size = lut_size;
  l->step = 2.0 / static_cast<double>(lut_size - 1);
  l->device = device;
  const size_t kn = static_cast<size_t>(l->n_feat) * lut_size;
  cudaError_t e = cudaMalloc(&l->values64, kn * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&l->values_pm, kn * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&l->slopes_pm, kn * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&l->dxrows, kn * sizeof(float));
  if (e != cudaSuccess) {
    ck_lut_destroy(l);
    set_error(std::string("ck_lut: cudaMalloc failed: ") + cudaGetErrorString(e));
    return kCudaError;
  }
  // last (unused) slope row stays zero
  e = cudaMemset(l->slopes_pm, 0, kn * sizeof(float));
  if (e != cudaSuccess) {
    ck_lut_destroy(l);
    set_error(std::string("ck_lut: cudaMemset failed: ") + cudaGetErrorString(e));
    return kCudaError;
  }
  *out = l;
  return kOk;
}

}  // namespace
}  // namespace ck

extern "C" int ck_lut_build(int degree, int lut_size, int device, ck_lut** out) {
  ck_lut* l = nullptr;
  CK_TRY(ck::lut_alloc(degree, lut_size, device, &l));
  const int threads = 256;
  const int blocks = static_cast<int>(ck::ceil_div(lut_size, threads));
  ck::LaunchScope scope(ck::kKLut, nullptr);
  ck::lut_build_kernel<<<blocks, threads>>>(degree, lut_size, l->step, l->values64, l->values_pm,
                                            l->slopes_pm);
  ck::lut_dxrows_kernel<<<blocks, threads>>>(l->n_feat, lut_size, l->step, l->slopes_pm, l->dxrows);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    ck_lut_destroy(l);
    ck::set_error(std::string("ck_lut_build: ") + cudaGetErrorString(e));
    return ck::kCudaError;
  }
  *out = l;
  return ck::kOk;
}

extern "C" int ck_lut_create(int degree, int lut_size, const double* values_host, const float* slopes_host,
                             int device, ck_lut** out) {
  CK_CHECK(values_host != nullptr && slopes_host != nullptr, "ck_lut_create: NULL table");
  ck_lut* l = nullptr;
  CK_TRY(ck::lut_alloc(degree, lut_size, device, &l));
  const size_t kn = static_cast<size_t>(l->n_feat) * lut_size;
  const size_t ks = static_cast<size_t>(l->n_feat) * (lut_size - 1);
  float* s_fm = nullptr;
  cudaError_t e = cudaMemcpy(l->values64, values_host, kn * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&s_fm, ks * sizeof(float) + 16);
  if (e == cudaSuccess) e = cudaMemcpy(s_fm, slopes_host, ks * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const int threads = 256;
    ck::lut_pack_kernel<<<static_cast<int>(ck::ceil_div(lut_size, threads)), threads>>>(
        l->n_feat, lut_size, l->values64, s_fm, l->values_pm, l->slopes_pm);
    ck::lut_dxrows_kernel<<<static_cast<int>(ck::ceil_div(lut_size, threads)), threads>>>(
        l->n_feat, lut_size, l->step, l->slopes_pm, l->dxrows);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (s_fm) cudaFree(s_fm);
  if (e != cudaSuccess) {
    ck_lut_destroy(l);
    ck::set_error(std::string("ck_lut_create: ") + cudaGetErrorString(e));
    return ck::kCudaError;
  }
  *out = l;
  return ck::kOk;
}

extern "C" void ck_lut_destroy(ck_lut* l) {
  if (!l) return;
  if (l->values64) cudaFree(l->values64);
  if (l->values_pm) cudaFree(l->values_pm);
  if (l->slopes_pm) cudaFree(l->slopes_pm);
  if (l->dxrows) cudaFree(l->dxrows);
  delete l;
}

extern "C" int ck_lut_info(const ck_lut* l, int* degree, int* lut_size, double* step) {
  CK_CHECK(l != nullptr, "ck_lut_info: NULL handle");
  if (degree) *degree = l->degree;
  if (lut_size) *lut_size = l->lut_size;
  if (step) *step = l->step;
  return ck::kOk;
}

extern "C" int ck_lut_read(const ck_lut* l, double* values_host, float* slopes_host) {
  CK_CHECK(l != nullptr, "ck_lut_read: NULL handle");
  const int K = l->n_feat, N = l->lut_size;
  if (values_host) {
    CK_CUDA(cudaMemcpy(values_host, l->values64, sizeof(double) * K * static_cast<size_t>(N),
                       cudaMemcpyDeviceToHost));
  }
  if (slopes_host) {
    std::vector<float> pm(static_cast<size_t>(K) * N);
    CK_CUDA(cudaMemcpy(pm.data(), l->slopes_pm, sizeof(float) * pm.size(), cudaMemcpyDeviceToHost));
    for (int k = 0; k < K; ++k)
      for (int i = 0; i + 1 < N; ++i) slopes_host[static_cast<size_t>(k) * (N - 1) + i] = pm[static_cast<size_t>(i) * K + k];
  }
  return ck::kOk;
}
