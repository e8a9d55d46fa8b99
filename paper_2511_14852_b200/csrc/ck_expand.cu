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
constexpr int kMaxK = 64;                // planes kernels: degree <= 63

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

// --- table columns ---------------------------------------------------------
// Column source for the two table entries bracketing a cell.  kLutSmem reads
// the float32 position-major table staged in shared memory; kLutNodes
// recomputes T_k at the two grid nodes (exact float64 nodes, lut.py:83-84,
// rounded to float32) by the recurrence T_{k+1} = 2x T_k - T_{k-1}
// (basis.py:112-119) in float32 -- the same table entries to ~k^2 ulp, with
// no memory traffic.  Both then interpolate v0 (1-f) + v1 f.
// Grid node -1 + i*step (lut.py:82-84) rounded to float32: (2i - (N-1)) / (N-1)
// with an exact integer numerator and one correctly rounded fp32 division
// (the FP64 pipe is too narrow on B200 to spend it here).
__device__ __forceinline__ float grid_node_f(int i, int n, double /*step*/) {
  return i >= n - 1 ? 1.0f : __fdiv_rn(static_cast<float>(2 * i - (n - 1)), static_cast<float>(n - 1));
}

template <int kSrc>
struct Columns {
  // Calls emit(k, value) for k = k0..K-1 in ascending order.
  template <typename F>
  __device__ __forceinline__ static void run(const float* tab, int K, int n, double step, int idx, float frac, int k0,
                                             F&& emit) {
    if constexpr (kSrc == kLutSmem) {
      const float* v = tab + static_cast<int64_t>(idx) * K;
      for (int k = k0; k < K; ++k) emit(k, lerp_ref(v[k], v[k + K], frac));
    } else {
      const float x0 = grid_node_f(idx, n, step), x1 = grid_node_f(idx + 1, n, step);
      const float tx0 = 2.0f * x0, tx1 = 2.0f * x1;
      float a_prev = 1.0f, a = x0, b_prev = 1.0f, b = x1;
      if (k0 == 0) emit(0, 1.0f);
      if (K > 1 && k0 <= 1) emit(1, lerp_ref(x0, x1, frac));
      for (int k = 2; k < K; ++k) {
        const float an = fmaf(tx0, a, -a_prev), bn = fmaf(tx1, b, -b_prev);
        a_prev = a;
        a = an;
        b_prev = b;
        b = bn;
        if (k >= k0) emit(k, lerp_ref(a, b, frac));
      }
    }
  }
};

// Planes for features k = 1..D of two elements (a, b), fully unrolled:
// out[k-1] packs (value_a, value_b) as bf16x2 hi / lo words.
template <int kSrc, int D>
__device__ __forceinline__ void pair_planes(const float* vt, int K, int n, double step, int ia, float fa, int ib,
                                            float fb, uint32_t (&hw)[D], uint32_t (&lw)[D]) {
  if constexpr (kSrc == kLutSmem) {
    const float* pa = vt + static_cast<int64_t>(ia) * K;
    const float* pb = vt + static_cast<int64_t>(ib) * K;
#pragma unroll
    for (int k = 1; k <= D; ++k)
      split_pack2(lerp_ref(pa[k], pa[k + K], fa), lerp_ref(pb[k], pb[k + K], fb), hw[k - 1], lw[k - 1]);
  } else {
    const float a0 = grid_node_f(ia, n, step), a1 = grid_node_f(ia + 1, n, step);
    const float b0 = grid_node_f(ib, n, step), b1 = grid_node_f(ib + 1, n, step);
    const float ta0 = 2.0f * a0, ta1 = 2.0f * a1, tb0 = 2.0f * b0, tb1 = 2.0f * b1;
    float pa0 = 1.0f, ca0 = a0, pa1 = 1.0f, ca1 = a1, pb0 = 1.0f, cb0 = b0, pb1 = 1.0f, cb1 = b1;
    split_pack2(lerp_ref(a0, a1, fa), lerp_ref(b0, b1, fb), hw[0], lw[0]);
#pragma unroll
    for (int k = 2; k <= D; ++k) {
      float t;
      t = fmaf(ta0, ca0, -pa0); pa0 = ca0; ca0 = t;
      t = fmaf(ta1, ca1, -pa1); pa1 = ca1; ca1 = t;
      t = fmaf(tb0, cb0, -pb0); pb0 = cb0; cb0 = t;
      t = fmaf(tb1, cb1, -pb1); pb1 = cb1; cb1 = t;
      split_pack2(lerp_ref(ca0, ca1, fa), lerp_ref(cb0, cb1, fb), hw[k - 1], lw[k - 1]);
    }
  }
}

// Split planes k = 1..D, hi/lo [k-1][r][ld]: each thread expands 4 adjacent
// columns of one row (two bf16x2 pairs) and writes one 8-byte word per plane
// for hi and lo (a warp stores 256 contiguous bytes per plane).
template <int kSrc, int D>
__global__ void __launch_bounds__(kThreads) expand_quads_kernel(const float* __restrict__ x, int64_t rows, int cols,
                                                                LutView lut, uint2* __restrict__ hi,
                                                                uint2* __restrict__ lo, int64_t ld, int64_t plane) {
  extern __shared__ float sm_tab[];
  const int K = lut.K, N = lut.N;
  const float* vt = kSrc == kLutSmem ? stage_table<true>(lut.values_pm, N * K, sm_tab) : nullptr;
  const int64_t pq = plane >> 2;  // plane stride in 8-byte words
  const int quads = (cols + 3) >> 2;
  const int64_t n_items = rows * quads;
  const bool vec = (cols & 3) == 0;
  for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < n_items;
       it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = it / quads;
    const int c = static_cast<int>(it - r * quads) * 4;
    const float* xr = x + r * cols + c;
    float xv[4];
    if (vec) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(xr));
      xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) xv[e] = c + e < cols ? __ldg(xr + e) : 0.0f;
    }
    int id[4];
    float fr[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) cell_f32(xv[e], N, id[e], fr[e]);
    uint32_t h0[D], l0[D], h1[D], l1[D];
    pair_planes<kSrc, D>(vt, K, N, lut.step, id[0], fr[0], id[1], fr[1], h0, l0);
    pair_planes<kSrc, D>(vt, K, N, lut.step, id[2], fr[2], id[3], fr[3], h1, l1);
    // padded columns (c+e >= cols) are written as zeros inside [cols, ld)
    const uint32_t m0 = c + 1 < cols ? 0xffffffffu : (c < cols ? 0xffffu : 0u);
    const uint32_t m1 = c + 3 < cols ? 0xffffffffu : (c + 2 < cols ? 0xffffu : 0u);
    uint2* hp = hi + ((r * ld + c) >> 2);
    uint2* lp = lo + ((r * ld + c) >> 2);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      *hp = make_uint2(h0[k] & m0, h1[k] & m1);
      *lp = make_uint2(l0[k] & m0, l1[k] & m1);
      hp += pq;
      lp += pq;
    }
  }
}

// Generic (any degree) fallbacks: hi/lo planes [k-k0][r][ld], two columns
// per thread.
template <int kSrc>
__global__ void __launch_bounds__(kThreads) expand_planes_kernel(const float* __restrict__ x, int64_t rows,
                                                                 int cols, LutView lut, int k0,
                                                                 uint32_t* __restrict__ hi,
                                                                 uint32_t* __restrict__ lo, int64_t ld,
                                                                 int64_t plane) {
  extern __shared__ float sm_tab[];
  const int K = lut.K, N = lut.N;
  const float* vt = kSrc == kLutSmem ? stage_table<true>(lut.values_pm, N * K, sm_tab) : nullptr;
  const int pairs = (cols + 1) >> 1;
  const int64_t n_items = rows * pairs;
  const int64_t pl = plane >> 1;
  for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < n_items;
       it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = it / pairs;
    const int c = static_cast<int>(it - r * pairs) * 2;
    const bool second = c + 1 < cols;
    const float xa = x[r * cols + c];
    const float xb = second ? x[r * cols + c + 1] : 0.0f;
    int ia, ib;
    float fa, fb;
    cell_f32(xa, N, ia, fa);
    cell_f32(xb, N, ib, fb);
    uint32_t* h = hi + ((r * ld + c) >> 1);
    uint32_t* l = lo + ((r * ld + c) >> 1);
    Columns<kSrc>::run(vt, K, N, lut.step, ia, fa, k0, [&](int k, float v) {
      float vb2 = 0.0f;
      if (second) {
        // second element: recompute through the same source (rare generic path)
        Columns<kSrc>::run(vt, K, N, lut.step, ib, fb, k, [&](int kk, float w) {
          if (kk == k) vb2 = w;
        });
      }
      uint32_t h2, l2;
      split_pack2(v, vb2, h2, l2);
      h[(k - k0) * pl] = h2;
      l[(k - k0) * pl] = l2;
    });
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


template <int kSrc>
int launch_quads(int d, const float* x, int64_t rows, int cols, const LutView& v, uint2* h, uint2* l, int64_t ld,
                 int64_t plane, size_t tab, int blocks, cudaStream_t s) {
  const size_t smem = kSrc == kLutSmem ? tab : 0;
#define CK_QUADS_CASE(D)                                                                                     \
  case D:                                                                                                    \
    if (smem) {                                                                                              \
      CK_CUDA(cudaFuncSetAttribute(expand_quads_kernel<kSrc, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                   static_cast<int>(smem)));                                                 \
    }                                                                                                        \
    expand_quads_kernel<kSrc, D><<<blocks, kThreads, smem, s>>>(x, rows, cols, v, h, l, ld, plane);          \
    break;
  switch (d) {
    CK_QUADS_CASE(1) CK_QUADS_CASE(2) CK_QUADS_CASE(3) CK_QUADS_CASE(4) CK_QUADS_CASE(5) CK_QUADS_CASE(6)
    CK_QUADS_CASE(7) CK_QUADS_CASE(8) CK_QUADS_CASE(9) CK_QUADS_CASE(10) CK_QUADS_CASE(11) CK_QUADS_CASE(12)
    CK_QUADS_CASE(13) CK_QUADS_CASE(14) CK_QUADS_CASE(15) CK_QUADS_CASE(16)
    default:
      return kUnsupported;
  }
#undef CK_QUADS_CASE
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int pick_source(size_t table_bytes) {
  const int o = lut_source_override();
  if (o == kLutSmem && table_bytes <= static_cast<size_t>(kSmemLutMax)) return kLutSmem;
  // default: recompute columns (no gathers, no bank conflicts)
  return kLutNodes;
}

int launch_expand_planes(const float* x, int64_t rows, int cols, const ck_lut* lut, int k0,
                         __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ld, int64_t plane, cudaStream_t s) {
  if (rows == 0 || cols == 0 || k0 >= lut->n_feat) return kOk;
  CK_CHECK(ld % 2 == 0 && plane % 2 == 0, "expand_planes: pitch must be even");
  const LutView v = view(lut);
  const size_t tab = sizeof(float) * v.N * v.K;
  const int src = pick_source(tab);
  auto* h = reinterpret_cast<uint32_t*>(hi);
  auto* l = reinterpret_cast<uint32_t*>(lo);
  LaunchScope scope(kKExpand, s);
  if (k0 == 1 && ld % 4 == 0 && plane % 4 == 0) {
    const int d = v.K - 1;
    const int qb = grid_for(rows * ((cols + 3) / 4), 8);
    auto* h8 = reinterpret_cast<uint2*>(hi);
    auto* l8 = reinterpret_cast<uint2*>(lo);
    const int rc = src == kLutSmem ? launch_quads<kLutSmem>(d, x, rows, cols, v, h8, l8, ld, plane, tab, qb, s)
                                   : launch_quads<kLutNodes>(d, x, rows, cols, v, h8, l8, ld, plane, tab, qb, s);
    if (rc != kUnsupported) return rc;
  }
  const int blocks = grid_for(rows * ((cols + 1) / 2), 8);
  if (src == kLutSmem) {
    CK_CUDA(cudaFuncSetAttribute(expand_planes_kernel<kLutSmem>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(tab)));
    expand_planes_kernel<kLutSmem><<<blocks, kThreads, tab, s>>>(x, rows, cols, v, k0, h, l, ld, plane);
  } else {
    expand_planes_kernel<kLutNodes><<<blocks, kThreads, 0, s>>>(x, rows, cols, v, k0, h, l, ld, plane);
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
