// LUT construction: basis values on a uniform grid in float64 (bit-identical
// to the reference's lut_build, lut.py:76-94), packed on the device into the
// float32 position-major tables and exact-cell rows the kernels read.
#include <cfloat>
#include <cstring>
#include <vector>

#include <cmath>

#include "ck_basis.cuh"
#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

// grid node i: -1 + step*i (numpy evaluates step*arange first), last = 1.0
// (lut.py:82-84)
double grid_node_host(int i, int n, double step) { return i == n - 1 ? 1.0 : -1.0 + step * static_cast<double>(i); }

// values[K][N] of basis_rows(kind, degree, grid) (basis.py:87-119) in float64
// with numpy's operation order: each recurrence step is
// (beta_k(x) * B_k - gamma_k * B_{k-1}) / alpha_k, beta_k(x) evaluated first
// (basis.py:116-119 with the coefficients of basis.py:52-77); Fourier seeds
// cos/sin(pi x) from libm (numpy's float64 cos/sin are libm's) and walks the
// angle-addition identities (basis.py:100-110).  The host compiler is run
// with -ffp-contract=off, so no FMA changes the rounding.
void basis_rows_host(int kind, int degree, int n, double step, double* v) {
  const int K = ck::basis_features(kind, degree);
  for (int i = 0; i < n; ++i) {
    const double x = grid_node_host(i, n, step);
    auto at = [&](int k) -> double& { return v[static_cast<int64_t>(k) * n + i]; };
    at(0) = 1.0;
    if (degree < 1) continue;
    if (kind == ck::kFourier) {
      const double theta = M_PI * x;
      const double c1 = cos(theta), s1 = sin(theta);
      at(1) = c1;
      at(2) = s1;
      for (int k = 1; k < degree; ++k) {
        const double a = at(2 * k - 1), b = at(2 * k);
        at(2 * k + 1) = c1 * a - s1 * b;
        at(2 * k + 2) = s1 * a + c1 * b;
      }
      continue;
    }
    at(1) = kind == ck::kHermite ? 2.0 * x : x;
    for (int k = 1; k < K - 1; ++k) {
      double alpha, beta, gamma;
      if (kind == ck::kLegendre) {
        alpha = static_cast<double>(k + 1);
        beta = (2.0 * k + 1.0) * x;
        gamma = static_cast<double>(k);
      } else if (kind == ck::kHermite) {
        alpha = 1.0;
        beta = 2.0 * x;
        gamma = 2.0 * k;
      } else {
        alpha = 1.0;
        beta = 2.0 * x;
        gamma = 1.0;
      }
      at(k + 1) = (beta * at(k) - gamma * at(k - 1)) / alpha;
    }
  }
}

// Position-major float32 copies and float32 cell slopes
// (values[:,1:] - values[:,:-1]) / step (lut.py:86, 93) from the float64
// table; one thread per node.  slopes_fm (nullable) supplies the slopes
// instead (ck_lut_create of a loaded PKLT table).
__global__ void lut_pack_kernel(int K, int n, double step, const double* __restrict__ v64,
                                const float* __restrict__ slopes_fm, float* __restrict__ v_pm,
                                float* __restrict__ s_pm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < K; ++k) {
    const double a = v64[static_cast<int64_t>(k) * n + i];
    v_pm[static_cast<int64_t>(i) * K + k] = __double2float_rn(a);
    if (i + 1 < n) {
      float sl;
      if (slopes_fm) {
        sl = slopes_fm[static_cast<int64_t>(k) * (n - 1) + i];
      } else {
        const double b = v64[static_cast<int64_t>(k) * n + i + 1];
        sl = __double2float_rn(__ddiv_rn(__dsub_rn(b, a), step));
      }
      s_pm[static_cast<int64_t>(i) * K + k] = sl;
    }
  }
}

// Reference cell of float32 input x (lut.py:97-106 after kernels.py:288).
__device__ __forceinline__ int ref_cell(float x, int n) {
  int idx;
  double fr, t;
  cell_f64(x, n, idx, fr, t);
  return idx;
}

// dxrows row i = {slopes_1..slopes_d of cell i, b_i, b_{i+1}, 0 pad} (d =
// K-1): the slopes first, so the common case (a float32 position safely
// inside its cell) gathers only ceil(d/4) 16-byte words.  b_i is the
// smallest float32 x with ref_cell(x) >= i, found from atanh(node_i) by
// stepping one float32 ulp at a time (ref_cell is monotone in x).  Thread i
// writes b_i into its own row and into row i-1's upper-boundary slot.
__global__ void lut_dxrows_kernel(int K, int n, double step, const float* __restrict__ s_pm,
                                  float* __restrict__ rows) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int S = dxrow_stride(K), d = K - 1;
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
  float* row = rows + static_cast<int64_t>(i) * S;
  for (int k = 1; k < K; ++k) row[k - 1] = i < n - 1 ? s_pm[static_cast<int64_t>(i) * K + k] : 0.0f;
  row[d] = b;
  if (i == n - 1) row[d + 1] = INFINITY;
  for (int j = d + 2; j < S; ++j) row[j] = 0.0f;
  if (i > 0) rows[static_cast<int64_t>(i - 1) * S + d + 1] = b;
}

int check_kind(int kind, int degree, bool exact) {
  CK_CHECK(kind >= ck::kCheb && kind <= ck::kChebTrig, "unsupported basis kind: " + std::to_string(kind));
  CK_CHECK(exact || kind != ck::kChebTrig, "the trig path applies to exact evaluation only");
  CK_CHECK(degree >= 0, "degree must be >= 0, got " + std::to_string(degree));
  CK_CHECK(degree <= 255, "degree must be <= 255");
  return kOk;
}

int lut_alloc(int kind, int degree, int lut_size, int device, ck_lut** out) {
  CK_CHECK(out != nullptr, "ck_lut: out handle pointer is NULL");
  CK_CHECK(lut_size >= 2, "lut_size must be >= 2");
  CK_TRY(check_kind(kind, degree, false));
  const int K = basis_features(kind, degree);
  CK_CHECK(static_cast<int64_t>(lut_size) * K < (int64_t(1) << 31), "lut too large");
  CK_CUDA(cudaSetDevice(device));
  ck_lut* l = new ck_lut();
  l->kind = kind;
  l->degree = degree;
  l->n_feat = K;
  l->lut_size = lut_size;
  l->step = 2.0 / static_cast<double>(lut_size - 1);
  l->device = device;
  const size_t kn = static_cast<size_t>(l->n_feat) * lut_size;
  cudaError_t e = cudaMalloc(&l->values64, kn * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&l->values_pm, kn * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&l->slopes_pm, kn * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&l->dxrows, static_cast<size_t>(dxrow_stride(K)) * lut_size * sizeof(float));
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

// Upload float64 values (and optional float32 slopes, [K][N-1]) and derive
// the kernels' tables.  Destroys the handle on failure.
int lut_finish(ck_lut* l, const double* values_host, const float* slopes_host) {
  const int K = l->n_feat, n = l->lut_size;
  const size_t kn = static_cast<size_t>(K) * n;
  float* s_fm = nullptr;
  cudaError_t e = cudaMemcpy(l->values64, values_host, kn * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && slopes_host) {
    const size_t ks = static_cast<size_t>(K) * (n - 1);
    e = cudaMalloc(&s_fm, ks * sizeof(float) + 16);
    if (e == cudaSuccess) e = cudaMemcpy(s_fm, slopes_host, ks * sizeof(float), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) {
    const int threads = 256;
    const int blocks = static_cast<int>(ceil_div(n, threads));
    LaunchScope scope(kKLut, nullptr);
    lut_pack_kernel<<<blocks, threads>>>(K, n, l->step, l->values64, s_fm, l->values_pm, l->slopes_pm);
    lut_dxrows_kernel<<<blocks, threads>>>(K, n, l->step, l->slopes_pm, l->dxrows);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (s_fm) cudaFree(s_fm);
  if (e != cudaSuccess) {
    ck_lut_destroy(l);
    set_error(std::string("ck_lut: ") + cudaGetErrorString(e));
    return kCudaError;
  }
  return kOk;
}

}  // namespace
}  // namespace ck

extern "C" int ck_lut_build(int kind, int degree, int lut_size, int device, ck_lut** out) {
  ck_lut* l = nullptr;
  CK_TRY(ck::lut_alloc(kind, degree, lut_size, device, &l));
  std::vector<double> v(static_cast<size_t>(l->n_feat) * lut_size);
  ck::basis_rows_host(kind, degree, lut_size, l->step, v.data());
  CK_TRY(ck::lut_finish(l, v.data(), nullptr));
  *out = l;
  return ck::kOk;
}

extern "C" int ck_lut_create(int kind, int degree, int lut_size, const double* values_host, const float* slopes_host,
                             int device, ck_lut** out) {
  CK_CHECK(values_host != nullptr && slopes_host != nullptr, "ck_lut_create: NULL table");
  ck_lut* l = nullptr;
  CK_TRY(ck::lut_alloc(kind, degree, lut_size, device, &l));
  CK_TRY(ck::lut_finish(l, values_host, slopes_host));
  *out = l;
  return ck::kOk;
}

extern "C" int ck_basis_exact(int kind, int degree, int device, ck_lut** out) {
  CK_CHECK(out != nullptr, "ck_basis_exact: out handle pointer is NULL");
  CK_TRY(ck::check_kind(kind, degree, true));
  CK_CUDA(cudaSetDevice(device));
  ck_lut* l = new ck_lut();
  l->kind = kind;
  l->exact = 1;
  l->degree = degree;
  l->n_feat = ck::basis_features(kind, degree);
  l->device = device;
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

extern "C" int ck_lut_kind(const ck_lut* l, int* kind, int* n_feat, int* exact) {
  CK_CHECK(l != nullptr, "ck_lut_kind: NULL handle");
  if (kind) *kind = l->kind;
  if (n_feat) *n_feat = l->n_feat;
  if (exact) *exact = l->exact;
  return ck::kOk;
}

extern "C" int ck_lut_read(const ck_lut* l, double* values_host, float* slopes_host) {
  CK_CHECK(l != nullptr, "ck_lut_read: NULL handle");
  CK_CHECK(!l->exact, "ck_lut_read: exact-evaluation handles have no table");
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
