// Basis expansion kernels: T_k(tanh x) by linear interpolation in a
// shared-memory lookup table (lut.py:97-123 semantics), plus the fused
// input-gradient combine that uses the derivative (slope) table.
//
// All kernels are HBM-bound streaming kernels: grid = a few CTAs per SM,
// grid-stride loops, the LUT staged once per CTA in shared memory when it
// fits (else read through L1/L2 from the position-major global copy).
#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

constexpr int kThreads = 256;
constexpr int kSmemLutMax = 96 * 1024;  // stage tables up to this size in smem

// Exact cell choice (float64), lut.py:97-106: clip, pos = (t+1)*0.5*(N-1),
// idx = min(trunc(pos), N-2), frac snapped to {0,1} within 1e-9.
__device__ __forceinline__ void cell_f64(float xv, int n, int& idx, double& frac, double& t) {
  t = tanh(static_cast<double>(xv));
  const double tc = fmin(fmax(t, -1.0), 1.0);
  const double pos = __dmul_rn(__dmul_rn(__dadd_rn(tc, 1.0), 0.5), static_cast<double>(n - 1));
  long long i = static_cast<long long>(pos);
  if (i > n - 2) i = n - 2;
  idx = static_cast<int>(i);
  frac = __dsub_rn(pos, static_cast<double>(idx));
  if (frac < 1e-9) frac = 0.0;
  if (frac > 1.0 - 1e-9) frac = 1.0;
}

// Fast cell choice for value interpolation (float32).  frac is formed with
// one rounding (fma of t*h against the exact h - idx), so the interpolated
// value is accurate to ~k^2 * ulp(t); a cell flip at an edge is harmless for
// values because the interpolant is continuous.
__device__ __forceinline__ void cell_f32(float xv, int n, int& idx, float& frac) {
  float t = tanhf(xv);
  t = fminf(fmaxf(t, -1.0f), 1.0f);
  const float h = 0.5f * static_cast<float>(n - 1);
  const float pos = fmaf(t, h, h);
  int i = static_cast<int>(pos);
  i = min(i, n - 2);
  idx = i;
  frac = fmaf(t, h, h - static_cast<float>(i));
}

__device__ __forceinline__ float lerp_ref(float v0, float v1, float f) {
  // v_left (1-f) + v_right f  (lut.py:115), exact at f = 0 and f = 1
  return fmaf(v1, f, v0 * (1.0f - f));
}

template <bool kSmem>
__device__ __forceinline__ const float* stage_table(const float* g, int count, float* s) {
  if (!kSmem) return g;
  for (int j = threadIdx.x; j < count; j += blockDim.x) s[j] = g[j];
  __syncthreads();
  return s;
}

// phi[e][k], slopes[e][k] for element e = r*cols + c.
template <bool kSmem>
__global__ void __launch_bounds__(kThreads) expand_f32_kernel(const float* __restrict__ x, int64_t n_elem,
                                                              LutView lut, float* __restrict__ phi,
                                                              float* __restrict__ slopes) {
  extern __shared__ float sm_tab[];
  const int K = lut.K, N = lut.N;
  const float* vt = stage_table<kSmem>(lut.values_pm, N * K, sm_tab);
  const float* st = slopes ? stage_table<kSmem>(lut.slopes_pm, N * K, sm_tab + N * K) : nullptr;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_elem;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int idx;
    double frac, t;
    cell_f64(x[e], N, idx, frac, t);
    const float f = static_cast<float>(frac);
    const float* v0 = vt + static_cast<int64_t>(idx) * K;
    for (int k = 0; k < K; ++k) phi[e * K + k] = lerp_ref(v0[k], v0[k + K], f);
    if (st) {
      const float* s0 = st + static_cast<int64_t>(idx) * K;
      for (int k = 0; k < K; ++k) slopes[e * K + k] = s0[k];
    }
  }
}

// hi/lo planes [k-k0][r][ld], two columns per thread (packed bf16x2 stores).
template <bool kSmem>
__global__ void __launch_bounds__(kThreads) expand_planes_kernel(const float* __restrict__ x, int64_t rows,
                                                                 int cols, LutView lut, int k0,
                                                                 uint32_t* __restrict__ hi,
                                                                 uint32_t* __restrict__ lo, int64_t ld,
                                                                 int64_t plane) {
  extern __shared__ float sm_tab[];
  const int K = lut.K, N = lut.N;
  const float* vt = stage_table<kSmem>(lut.values_pm, N * K, sm_tab);
  const int pairs = (cols + 1) >> 1;
  const int64_t n_items = rows * pairs;
  for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < n_items;
       it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = it / pairs;
    const int c = static_cast<int>(it - r * pairs) * 2;
    const bool second = c + 1 < cols;
    int ia, ib;
    float fa, fb;
    cell_f32(x[r * cols + c], N, ia, fa);
    cell_f32(second ? x[r * cols + c + 1] : 0.0f, N, ib, fb);
    const float* va = vt + static_cast<int64_t>(ia) * K;
    const float* vb = vt + static_cast<int64_t>(ib) * K;
    const int64_t o = (r * ld + c) >> 1;
    for (int k = k0; k < K; ++k) {
      const float a = lerp_ref(va[k], va[k + K], fa);
      const float b = second ? lerp_ref(vb[k], vb[k + K], fb) : 0.0f;
      uint32_t h2, l2;
      split_pack2(a, b, h2, l2);
      const int64_t off = ((k - k0) * plane >> 1) + o;
      hi[off] = h2;
      lo[off] = l2;
    }
  }
}

// Transposed hi/lo planes [k-k0][c][ldr] via a 64(r) x 32(c) smem tile.
constexpr int kTR = 64, kTC = 32, kTP = kTR + 2;  // padded row (bf16) -> 33 words
template <bool kSmem>
__global__ void __launch_bounds__(kThreads) expand_planes_t_kernel(const float* __restrict__ x, int64_t rows,
                                                                   int cols, LutView lut, int k0,
                                                                   __nv_bfloat16* __restrict__ hi,
                                                                   __nv_bfloat16* __restrict__ lo,
                                                                   int64_t ldr, int64_t plane) {
  extern __shared__ float sm_tab[];
  __shared__ __align__(16) __nv_bfloat16 t_hi[kTC * kTP];
  __shared__ __align__(16) __nv_bfloat16 t_lo[kTC * kTP];
  const int K = lut.K, N = lut.N;
  const float* vt = stage_table<kSmem>(lut.values_pm, N * K, sm_tab);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r_tiles = ceil_div(rows, kTR);
  const int64_t c_tiles = ceil_div(cols, kTC);
  for (int64_t tile = blockIdx.x; tile < r_tiles * c_tiles; tile += gridDim.x) {
    const int64_t r0 = (tile % r_tiles) * kTR;
    const int c0 = static_cast<int>(tile / r_tiles) * kTC;
    const int c = c0 + tx;
    int idx[kTR / 8];
    float fr[kTR / 8];
    bool ok[kTR / 8];
#pragma unroll
    for (int j = 0; j < kTR / 8; ++j) {
      const int64_t r = r0 + ty + 8 * j;
      ok[j] = (r < rows) && (c < cols);
      cell_f32(ok[j] ? x[r * cols + c] : 0.0f, N, idx[j], fr[j]);
    }
    for (int k = k0; k < K; ++k) {
#pragma unroll
      for (int j = 0; j < kTR / 8; ++j) {
        const float* v = vt + static_cast<int64_t>(idx[j]) * K + k;
        const float val = ok[j] ? lerp_ref(v[0], v[K], fr[j]) : 0.0f;
        __nv_bfloat16 h, l;
        split_bf16(val, h, l);
        t_hi[tx * kTP + ty + 8 * j] = h;
        t_lo[tx * kTP + ty + 8 * j] = l;
      }
      __syncthreads();
      // each warp writes whole rows (fixed c) of 64 r-values = 32 words
      for (int cc = ty; cc < kTC; cc += kThreads / 32) {
        const int col = c0 + cc;
        const int64_t r = r0 + 2 * tx;
        if (col < cols && r < ldr) {
          const int64_t off = (k - k0) * plane + static_cast<int64_t>(col) * ldr + r;
          *reinterpret_cast<uint32_t*>(hi + off) =
              *reinterpret_cast<const uint32_t*>(&t_hi[cc * kTP + 2 * tx]);
          *reinterpret_cast<uint32_t*>(lo + off) =
              *reinterpret_cast<const uint32_t*>(&t_lo[cc * kTP + 2 * tx]);
        }
      }
      __syncthreads();
    }
  }
}

// dx = J * sum_{k>=1} slope_k * g_{k-1}  (kernels.py:430-444); the cell is
// chosen in float64 so the piecewise-constant slope matches the reference.
template <bool kSmem>
__global__ void __launch_bounds__(kThreads) dx_combine_kernel(const float* __restrict__ g, int64_t g_plane,
                                                              const float* __restrict__ x, int64_t n_elem,
                                                              LutView lut, int jacobian,
                                                              float* __restrict__ dx) {
  extern __shared__ float sm_tab[];
  const int K = lut.K, N = lut.N;
  const float* st = stage_table<kSmem>(lut.slopes_pm, N * K, sm_tab);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_elem;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int idx;
    double frac, t;
    cell_f64(x[e], N, idx, frac, t);
    const float* s0 = st + static_cast<int64_t>(idx) * K;
    float acc = 0.0f;
    for (int k = 1; k < K; ++k) acc = fmaf(s0[k], g[(k - 1) * g_plane + e], acc);
    double v = static_cast<double>(acc);
    if (jacobian) v *= 1.0 - t * t;
    dx[e] = static_cast<float>(v);
  }
}

int grid_for(int64_t items, int per_sm) {
  const int64_t want = ceil_div(items, kThreads);
  const int64_t cap = static_cast<int64_t>(num_sms()) * per_sm;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

int launch_expand_f32(const float* x, int64_t rows, int cols, const ck_lut* lut, float* phi, float* slopes,
                      cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return kOk;
  const LutView v = view(lut);
  const size_t tab = sizeof(float) * v.N * v.K * (slopes ? 2 : 1);
  const int blocks = grid_for(n, 8);
  LaunchScope scope(kKExpand, s);
  if (tab <= static_cast<size_t>(kSmemLutMax)) {
    CK_CUDA(cudaFuncSetAttribute(expand_f32_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(tab)));
    expand_f32_kernel<true><<<blocks, kThreads, tab, s>>>(x, n, v, phi, slopes);
  } else {
    expand_f32_kernel<false><<<blocks, kThreads, 0, s>>>(x, n, v, phi, slopes);
  }
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_expand_planes(const float* x, int64_t rows, int cols, const ck_lut* lut, int k0,
                         __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ld, int64_t plane, cudaStream_t s) {
  if (rows == 0 || cols == 0 || k0 >= lut->n_feat) return kOk;
  CK_CHECK(ld % 2 == 0 && plane % 2 == 0, "expand_planes: pitch must be even");
  const LutView v = view(lut);
  const size_t tab = sizeof(float) * v.N * v.K;
  const int blocks = grid_for(rows * ((cols + 1) / 2), 8);
  auto* h = reinterpret_cast<uint32_t*>(hi);
  auto* l = reinterpret_cast<uint32_t*>(lo);
  LaunchScope scope(kKExpand, s);
  if (tab <= static_cast<size_t>(kSmemLutMax)) {
    CK_CUDA(cudaFuncSetAttribute(expand_planes_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(tab)));
    expand_planes_kernel<true><<<blocks, kThreads, tab, s>>>(x, rows, cols, v, k0, h, l, ld, plane);
  } else {
    expand_planes_kernel<false><<<blocks, kThreads, 0, s>>>(x, rows, cols, v, k0, h, l, ld, plane);
  }
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_expand_planes_t(const float* x, int64_t rows, int cols, const ck_lut* lut, int k0,
                           __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ldr, int64_t plane, cudaStream_t s) {
  if (rows == 0 || cols == 0 || k0 >= lut->n_feat) return kOk;
  CK_CHECK(ldr % 2 == 0 && plane % 2 == 0, "expand_planes_t: pitch must be even");
  const LutView v = view(lut);
  const size_t tab = sizeof(float) * v.N * v.K;
  const int64_t tiles = ceil_div(rows, kTR) * ceil_div(cols, kTC);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 4;
  const int blocks = static_cast<int>(tiles < cap ? tiles : cap);
  LaunchScope scope(kKExpandT, s);
  if (tab <= static_cast<size_t>(kSmemLutMax)) {
    CK_CUDA(cudaFuncSetAttribute(expand_planes_t_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(tab)));
    expand_planes_t_kernel<true><<<blocks, kThreads, tab, s>>>(x, rows, cols, v, k0, hi, lo, ldr, plane);
  } else {
    expand_planes_t_kernel<false><<<blocks, kThreads, 0, s>>>(x, rows, cols, v, k0, hi, lo, ldr, plane);
  }
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_dx_combine(const float* g, int64_t g_plane, const float* x, int64_t rows, int cols,
                      const ck_lut* lut, int jacobian, float* dx, cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return kOk;
  const LutView v = view(lut);
  const size_t tab = sizeof(float) * v.N * v.K;
  const int blocks = grid_for(n, 8);
  LaunchScope scope(kKDxCombine, s);
  if (tab <= static_cast<size_t>(kSmemLutMax)) {
    CK_CUDA(cudaFuncSetAttribute(dx_combine_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(tab)));
    dx_combine_kernel<true><<<blocks, kThreads, tab, s>>>(g, g_plane, x, n, v, jacobian, dx);
  } else {
    dx_combine_kernel<false><<<blocks, kThreads, 0, s>>>(g, g_plane, x, n, v, jacobian, dx);
  }
  CK_CUDA(cudaGetLastError());
  return kOk;
}

}  // namespace ck
