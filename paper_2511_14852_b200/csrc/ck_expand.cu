// Basis expansion kernels: B_k(tanh x) by linear interpolation in the
// lookup table (lut.py:97-123 semantics) or, for exact-evaluation handles,
// by the family's recurrence at t itself (basis_rows, kernels.py:219-224);
// plus the unfused input-gradient combine that uses the slope table or the
// analytic derivatives (only for degrees beyond the fused GEMM epilogue).
//
// All kernels are HBM-bound streaming kernels: grid = a few CTAs per SM,
// grid-stride loops.  The GEMM operand planes are written as bf16 hi/lo
// pairs [k-1][row][ld] with 8-byte (4-column) stores per plane.
#include "ck_basis.cuh"
#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

constexpr int kThreads = 256;
constexpr int kSmemLutMax = 96 * 1024;  // fp32 API: stage tables up to this size in smem
constexpr int kMaxK = 64;                // runtime-degree paths: features <= 64
constexpr int kMaxPlanesFused = 16;      // specialized (unrolled) kernels: 1..16 planes

template <bool kSmem>
__device__ __forceinline__ const float* stage_table(const float* g, int count, float* s) {
  if constexpr (!kSmem) {
    return g;
  } else {
    for (int j = threadIdx.x; j < count; j += blockDim.x) s[j] = g[j];
    __syncthreads();
    return s;
  }
}

// fp32 API (ck_expand): phi[e][k], slopes[e][k] for element e = r*cols + c.
// LUT handles: float64 reference cell, table values and slopes.  Exact
// handles: basis and derivative at float32 tanh(x).
template <bool kSmem>
__global__ void __launch_bounds__(kThreads) expand_f32_kernel(const float* __restrict__ x, int64_t n_elem,
                                                              LutView lut, float* __restrict__ phi,
                                                              float* __restrict__ slopes) {
  pdl_wait();
  extern __shared__ float sm_tab[];
  const int K = lut.K, N = lut.N;
  const float* vt = lut.exact ? nullptr : stage_table<kSmem>(lut.values_pm, N * K, sm_tab);
  const float* st = (slopes && !lut.exact) ? stage_table<kSmem>(lut.slopes_pm, N * K, sm_tab + N * K) : nullptr;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_elem;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (lut.exact) {
      float v[kMaxK], dv[kMaxK];
      basis_deriv_rt(lut.kind, K - 1, tanhf(x[e]), v, slopes ? dv : nullptr);
      for (int k = 0; k < K; ++k) phi[e * K + k] = v[k];
      if (slopes)
        for (int k = 0; k < K; ++k) slopes[e * K + k] = dv[k];
      continue;
    }
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

// Basis at normalized points t (no tanh): table interpolation with the
// reference's float64 cell and slopes (lut_interp / interp_rows_with_slope,
// lut.py:109-140), or basis_rows / derivative_rows (basis.py:87-204).
__global__ void __launch_bounds__(kThreads) basis_eval_kernel(const float* __restrict__ t, int64_t n_elem,
                                                              LutView lut, float* __restrict__ vals,
                                                              float* __restrict__ slopes) {
  pdl_wait();
  const int K = lut.K, N = lut.N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_elem;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (lut.exact) {
      float v[kMaxFeaturesRt], dv[kMaxFeaturesRt];
      basis_deriv_rt(lut.kind, K - 1, t[e], v, slopes ? dv : nullptr);
      for (int k = 0; k < K; ++k) vals[e * K + k] = v[k];
      if (slopes)
        for (int k = 0; k < K; ++k) slopes[e * K + k] = dv[k];
      continue;
    }
    int idx;
    double frac;
    cell_f64_at(static_cast<double>(t[e]), N, idx, frac);
    const float f = static_cast<float>(frac);
    const float* v0 = lut.values_pm + static_cast<int64_t>(idx) * K;
    for (int k = 0; k < K; ++k) vals[e * K + k] = lerp_ref(v0[k], v0[k + K], f);
    if (slopes) {
      const float* s0 = lut.slopes_pm + static_cast<int64_t>(idx) * K;
      for (int k = 0; k < K; ++k) slopes[e * K + k] = s0[k];
    }
  }
}

// --- specialized planes kernels ----------------------------------------------
// Expand the 4 x values of one quad (row r, columns c..c+3) into planes
// k = 1..D and store one 8-byte hi and lo word per plane; padded columns
// (c+e >= cols) are written as zeros inside [cols, ld).
template <int kSrc, int KIND, int D>
__device__ __forceinline__ void quad_emit(const float (&xv)[4], int64_t r, int c, int cols, int lut_n,
                                          uint2* __restrict__ hi, uint2* __restrict__ lo, int64_t ld, int64_t pq) {
  uint32_t h0[D], l0[D], h1[D], l1[D];
  {
    float a[D], b[D];
    elem_planes<kSrc, KIND, D>(xv[0], lut_n, a);
    elem_planes<kSrc, KIND, D>(xv[1], lut_n, b);
#pragma unroll
    for (int k = 0; k < D; ++k) split_pack2(a[k], b[k], h0[k], l0[k]);
  }
  {
    float a[D], b[D];
    elem_planes<kSrc, KIND, D>(xv[2], lut_n, a);
    elem_planes<kSrc, KIND, D>(xv[3], lut_n, b);
#pragma unroll
    for (int k = 0; k < D; ++k) split_pack2(a[k], b[k], h1[k], l1[k]);
  }
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
  // the row's last quad also zero-fills the pitch padding [c + 4, ld): a
  // partly written 32-byte sector at every row end made the L2 fetch it from
  // DRAM first (ncu, 32000 x 257 d15: +31 MB of reads, half the write rate)
  if (c + 4 >= cols && c + 4 < ld) {
    for (int64_t w = c + 4; w < ld; w += 4) {
      uint2* hz = hi + ((r * ld + w) >> 2);
      uint2* lz = lo + ((r * ld + w) >> 2);
      for (int k = 0; k < D; ++k) {
        *hz = make_uint2(0u, 0u);
        *lz = make_uint2(0u, 0u);
        hz += pq;
        lz += pq;
      }
    }
  }
}

// B_{k+1} from B_k (cur) and B_{k-1} (prev): basis_f32's recurrence step k,
// the same operations (bitwise the same values).
template <int KIND>
__device__ __forceinline__ float rec_next(int k, float x, float cur, float prev) {
  if constexpr (KIND == kCheb) {
    return fmaf(2.0f * x, cur, -prev);
  } else if constexpr (KIND == kLegendre) {
    const float num = fmaf(static_cast<float>(2 * k + 1) * x, cur, -static_cast<float>(k) * prev);
    return num * (1.0f / static_cast<float>(k + 1));
  } else {
    return fmaf(2.0f * x, cur, -static_cast<float>(2 * k) * prev);
  }
}

// quad_emit for the LUT path of the three-term families, streamed plane by
// plane: the 8 node recurrences (4 elements x 2 grid nodes) advance one
// feature at a time and each plane's hi/lo words are stored as soon as they
// exist, so the state is 16 floats instead of 4 D-element arrays (d15: 114
// registers, 23 % occupancy, issue-bound at ~13 instructions per value).
// Bitwise the values of quad_emit.
template <int KIND, int D>
__device__ __forceinline__ void quad_emit_stream(const float (&xv)[4], int64_t r, int c, int cols, int lut_n,
                                                 uint2* __restrict__ hi, uint2* __restrict__ lo, int64_t ld,
                                                 int64_t pq) {
  float f[4], xn[8], pv[8], cv[8];
  const float step = 2.0f / static_cast<float>(lut_n - 1);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int idx;
    cell_f32(xv[e], lut_n, idx, f[e]);
    xn[2 * e] = grid_node_f(idx, lut_n, step);
    xn[2 * e + 1] = grid_node_f(idx + 1, lut_n, step);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    pv[j] = 1.0f;
    cv[j] = KIND == kHermite ? 2.0f * xn[j] : xn[j];  // B_1
  }
  const uint32_t m0 = c + 1 < cols ? 0xffffffffu : (c < cols ? 0xffffu : 0u);
  const uint32_t m1 = c + 3 < cols ? 0xffffffffu : (c + 2 < cols ? 0xffffu : 0u);
  uint2* hp = hi + ((r * ld + c) >> 2);
  uint2* lp = lo + ((r * ld + c) >> 2);
#pragma unroll
  for (int k = 1; k <= D; ++k) {
    if (k > 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float nv = rec_next<KIND>(k - 1, xn[j], cv[j], pv[j]);
        pv[j] = cv[j];
        cv[j] = nv;
      }
    }
    uint32_t h0, l0, h1, l1;
    split_pack2(lerp_ref(cv[0], cv[1], f[0]), lerp_ref(cv[2], cv[3], f[1]), h0, l0);
    split_pack2(lerp_ref(cv[4], cv[5], f[2]), lerp_ref(cv[6], cv[7], f[3]), h1, l1);
    *hp = make_uint2(h0 & m0, h1 & m1);
    *lp = make_uint2(l0 & m0, l1 & m1);
    hp += pq;
    lp += pq;
  }
  if (c + 4 >= cols && c + 4 < ld) {  // pitch padding (see quad_emit)
    for (int64_t w = c + 4; w < ld; w += 4) {
      uint2* hz = hi + ((r * ld + w) >> 2);
      uint2* lz = lo + ((r * ld + w) >> 2);
      for (int k = 0; k < D; ++k) {
        *hz = make_uint2(0u, 0u);
        *lz = make_uint2(0u, 0u);
        hz += pq;
        lz += pq;
      }
    }
  }
}

template <int kSrc, int KIND, int D>
__device__ __forceinline__ void quad_out(const float (&xv)[4], int64_t r, int c, int cols, int lut_n,
                                         uint2* __restrict__ hi, uint2* __restrict__ lo, int64_t ld, int64_t pq) {
  if constexpr (kSrc == kSrcNodes && (KIND == kCheb || KIND == kLegendre || KIND == kHermite)) {
    quad_emit_stream<KIND, D>(xv, r, c, cols, lut_n, hi, lo, ld, pq);
  } else {
    quad_emit<kSrc, KIND, D>(xv, r, c, cols, lut_n, hi, lo, ld, pq);
  }
}

// Ragged rows (cols % 4 != 0: x rows are not 16-byte aligned, e.g. the 257
// spectrogram bins of the C3 input layer): a block's 256 consecutive quads
// cover one contiguous stretch of x, loaded cooperatively with aligned
// 16-byte loads into shared memory; each thread then reads its quad there.
// (Per-thread scalar loads left this case at half the aligned layers' write
// rate: ncu 12 long-scoreboard stalls per issue, LSU throttle.)
template <int kSrc, int KIND, int D>
__device__ __forceinline__ void quads_ragged(const float* __restrict__ x, int64_t rows, int cols, int lut_n,
                                             uint2* __restrict__ hi, uint2* __restrict__ lo, int64_t ld,
                                             int64_t pq) {
  __shared__ float sx[4 * (kThreads + 2)];
  const int quads = (cols + 3) >> 2;
  const int64_t n_items = rows * quads;
  const int64_t total = rows * cols;
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int64_t bstride = static_cast<int64_t>(gridDim.x) * kThreads;
  // stretch of x covered by the block's quads [base, base + 256): first
  // aligned float index and the number of 16-byte slots
  auto stretch = [&](int64_t base, int64_t& rb, int& qb, int64_t& a0) -> int {
    const int64_t last = (base + kThreads < n_items ? base + kThreads : n_items) - 1;
    rb = base / quads;
    qb = static_cast<int>(base - rb * quads);
    const int64_t rl = last / quads;
    const int ql = static_cast<int>(last - rl * quads);
    const int64_t f1 = rl * cols + (4 * ql + 4 < cols ? 4 * ql + 4 : cols);  // exclusive
    a0 = (rb * cols + 4 * qb) & ~static_cast<int64_t>(3);
    return static_cast<int>((f1 - a0 + 3) >> 2);  // <= kThreads + 2
  };
  auto load_slot = [&](int64_t a) -> float4 {
    float4 v;
    if (aligned && a + 4 <= total) {
      v = __ldg(reinterpret_cast<const float4*>(x + a));
    } else {
      v.x = a < total ? __ldg(x + a) : 0.0f;
      v.y = a + 1 < total ? __ldg(x + a + 1) : 0.0f;
      v.z = a + 2 < total ? __ldg(x + a + 2) : 0.0f;
      v.w = a + 3 < total ? __ldg(x + a + 3) : 0.0f;
    }
    return v;
  };
  // the next stretch is loaded into registers while the current one is
  // expanded (slots tid and, for tid < 2, 256 + tid)
  float4 nx0 = make_float4(0.f, 0.f, 0.f, 0.f), nx1 = nx0;
  auto prefetch = [&](int64_t base) {
    if (base >= n_items) return;
    int64_t rb, a0;
    int qb;
    const int nv = stretch(base, rb, qb, a0);
    if (static_cast<int>(threadIdx.x) < nv) nx0 = load_slot(a0 + 4 * threadIdx.x);
    if (static_cast<int>(threadIdx.x) + kThreads < nv) nx1 = load_slot(a0 + 4 * (threadIdx.x + kThreads));
  };
  int64_t base = blockIdx.x * static_cast<int64_t>(kThreads);
  prefetch(base);
  for (; base < n_items; base += bstride) {
    int64_t rb, a0;
    int qb;
    const int nv = stretch(base, rb, qb, a0);
    __syncthreads();  // the previous stretch's readers are done
    if (static_cast<int>(threadIdx.x) < nv) *reinterpret_cast<float4*>(sx + 4 * threadIdx.x) = nx0;
    if (static_cast<int>(threadIdx.x) + kThreads < nv) *reinterpret_cast<float4*>(sx + 4 * (threadIdx.x + kThreads)) = nx1;
    __syncthreads();
    prefetch(base + bstride);
    const int64_t it = base + threadIdx.x;
    if (it < n_items) {
      const int qq = qb + static_cast<int>(threadIdx.x);
      const int64_t r = rb + qq / quads;
      const int c = (qq % quads) * 4;
      const int64_t off = r * cols + c - a0;
      float xv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) xv[e] = c + e < cols ? sx[off + e] : 0.0f;
      quad_out<kSrc, KIND, D>(xv, r, c, cols, lut_n, hi, lo, ld, pq);
    }
  }
}

// Planes k = 1..D, hi/lo [k-1][r][ld]: each thread expands 4 adjacent
// columns of one row (two bf16x2 pairs) and writes one 8-byte word per plane
// for hi and lo (a warp stores 256 contiguous bytes per plane).
template <int kSrc, int KIND, int D>
__global__ void __launch_bounds__(kThreads) expand_quads_kernel(const float* __restrict__ x, int64_t rows, int cols,
                                                                int lut_n, uint2* __restrict__ hi,
                                                                uint2* __restrict__ lo, int64_t ld, int64_t plane) {
  pdl_wait();
  const int64_t pq = plane >> 2;  // plane stride in 8-byte words
  const int quads = (cols + 3) >> 2;
  const bool vec = (cols & 3) == 0;
  if (!vec) {
    quads_ragged<kSrc, KIND, D>(x, rows, cols, lut_n, hi, lo, ld, pq);
    return;
  }
  // grid-stride over (row, quad) items, advanced incrementally (one division
  // per thread instead of a 64-bit division per item)
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t it0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t sr = stride / quads;
  const int sq = static_cast<int>(stride - sr * quads);
  int64_t r = it0 / quads;
  int q = static_cast<int>(it0 - r * quads);
  // x of the next item is loaded before this item is expanded: the loop was
  // bound by the load latency at the occupancy the high-degree planes leave
  // (ncu, 32000 x 257 d15: 71 % long-scoreboard stalls, 29 % issue)
  auto load_x = [&](int64_t rr, int qq, float (&v4)[4]) {
    if (rr >= rows) return;
    const int cc = qq * 4;
    const float* xr = x + rr * cols + cc;
    if (vec) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(xr));
      v4[0] = v.x; v4[1] = v.y; v4[2] = v.z; v4[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) v4[e] = cc + e < cols ? __ldg(xr + e) : 0.0f;
    }
  };
  float xn[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  load_x(r, q, xn);
  for (; r < rows; r += sr, q += sq) {
    if (q >= quads) {
      q -= quads;
      ++r;
      if (r >= rows) break;
    }
    const int c = q * 4;
    float xv[4] = {xn[0], xn[1], xn[2], xn[3]};
    {
      int64_t rn = r + sr;
      int qn = q + sq;
      if (qn >= quads) {
        qn -= quads;
        ++rn;
      }
      load_x(rn, qn, xn);
    }
    quad_out<kSrc, KIND, D>(xv, r, c, cols, lut_n, hi, lo, ld, pq);
  }
}

// Generic (any degree / first feature k0 >= 1, runtime kind) planes
// [k-k0][r][ld]: two columns per thread, features streamed by Rec at the two
// grid nodes of each element (LUT) or at t (exact).
__global__ void __launch_bounds__(kThreads) expand_planes_kernel(const float* __restrict__ x, int64_t rows,
                                                                 int cols, LutView lut, int k0,
                                                                 uint32_t* __restrict__ hi,
                                                                 uint32_t* __restrict__ lo, int64_t ld,
                                                                 int64_t plane) {
  pdl_wait();
  const int K = lut.K, N = lut.N;
  const int pairs = (cols + 1) >> 1;
  const int64_t n_items = rows * pairs;
  const int64_t pl = plane >> 1;
  for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < n_items;
       it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = it / pairs;
    const int c = static_cast<int>(it - r * pairs) * 2;
    const bool second = c + 1 < cols;
    const float xs[2] = {x[r * cols + c], second ? x[r * cols + c + 1] : 0.0f};
    Rec ra[2], rb[2];
    float fr[2];
    for (int e = 0; e < 2; ++e) {
      if (lut.exact) {
        ra[e].init(lut.kind, tanhf(xs[e]));
      } else {
        int idx;
        cell_f32(xs[e], N, idx, fr[e]);
        ra[e].init(lut.kind, grid_node_f(idx, N, 2.0f / static_cast<float>(N - 1)));
        rb[e].init(lut.kind, grid_node_f(idx + 1, N, 2.0f / static_cast<float>(N - 1)));
      }
    }
    uint32_t* h = hi + ((r * ld + c) >> 1);
    uint32_t* l = lo + ((r * ld + c) >> 1);
    for (int k = 1; k < K; ++k) {
      float v[2];
      for (int e = 0; e < 2; ++e) {
        const float a = ra[e].next();
        v[e] = lut.exact ? a : lerp_ref(a, rb[e].next(), fr[e]);
      }
      if (k < k0) continue;
      uint32_t h2, l2;
      split_pack2(v[0], second ? v[1] : 0.0f, h2, l2);
      h[(k - k0) * pl] = h2;
      l[(k - k0) * pl] = l2;
    }
  }
}

// dx = J * sum_{k>=1} slope_k * g[k-1]  (kernels.py:430-444).  LUT: the
// cell is chosen in float64 so the piecewise-constant slope matches the
// reference.  Exact: derivative_rows at t (kernels.py:224).
template <bool kSmem>
__global__ void __launch_bounds__(kThreads) dx_combine_kernel(const float* __restrict__ g, int64_t g_plane,
                                                              const float* __restrict__ x, int64_t n_elem,
                                                              LutView lut, int jacobian,
                                                              float* __restrict__ dx) {
  pdl_wait();
  extern __shared__ float sm_tab[];
  const int K = lut.K, N = lut.N;
  const float* st = lut.exact ? nullptr : stage_table<kSmem>(lut.slopes_pm, N * K, sm_tab);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_elem;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = 0.0f;
    if (lut.exact) {
      float v[kMaxK], dv[kMaxK];
      const float t = tanhf(x[e]);
      basis_deriv_rt(lut.kind, K - 1, t, v, dv);
      for (int k = 1; k < K; ++k) acc = fmaf(dv[k], g[(k - 1) * g_plane + e], acc);
      dx[e] = jacobian ? acc * (1.0f - t * t) : acc;
      continue;
    }
    int idx;
    double frac, t;
    cell_f64(x[e], N, idx, frac, t);
    const float* s0 = st + static_cast<int64_t>(idx) * K;
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

template <int kSrc, int KIND>
int launch_quads_kind(int d, const float* x, int64_t rows, int cols, int lut_n, uint2* h, uint2* l, int64_t ld,
                      int64_t plane, int blocks, cudaStream_t s) {
#define CK_QUADS_CASE(D)                                                                            \
  case D:                                                                                           \
    if constexpr (KIND != kFourier || D % 2 == 0) {                                                 \
      CK_CUDA(launch_k((expand_quads_kernel<kSrc, KIND, D>), blocks, kThreads, 0, s, x, rows, cols, lut_n, h, l, ld, plane)); \
      break;                                                                                        \
    } else {                                                                                        \
      return kUnsupported;                                                                          \
    }
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

template <int kSrc>
int launch_quads(const LutView& v, const float* x, int64_t rows, int cols, uint2* h, uint2* l, int64_t ld,
                 int64_t plane, int blocks, cudaStream_t s) {
  const int d = v.K - 1;
  switch (v.kind) {
    case kCheb:
      return launch_quads_kind<kSrc, kCheb>(d, x, rows, cols, v.N, h, l, ld, plane, blocks, s);
    case kLegendre:
      return launch_quads_kind<kSrc, kLegendre>(d, x, rows, cols, v.N, h, l, ld, plane, blocks, s);
    case kHermite:
      return launch_quads_kind<kSrc, kHermite>(d, x, rows, cols, v.N, h, l, ld, plane, blocks, s);
    case kFourier:
      return launch_quads_kind<kSrc, kFourier>(d, x, rows, cols, v.N, h, l, ld, plane, blocks, s);
    case kChebTrig:
      if constexpr (kSrc == kSrcExact) {
        return launch_quads_kind<kSrc, kChebTrig>(d, x, rows, cols, v.N, h, l, ld, plane, blocks, s);
      }
      return kUnsupported;
    default:
      return kUnsupported;
  }
}

}  // namespace

int launch_expand_f32(const float* x, int64_t rows, int cols, const ck_lut* lut, float* phi, float* slopes,
                      cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return kOk;
  const LutView v = view(lut);
  CK_CHECK(v.K <= kMaxK, "ck_expand: at most 64 features");
  const size_t tab = v.exact ? 0 : sizeof(float) * v.N * v.K * (slopes ? 2 : 1);
  const int blocks = grid_for(n, 8);
  LaunchScope scope(kKExpand, s);
  if (tab > 0 && tab <= static_cast<size_t>(kSmemLutMax)) {
    CK_CUDA(cudaFuncSetAttribute(expand_f32_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(tab)));
    CK_CUDA(launch_k((expand_f32_kernel<true>), blocks, kThreads, tab, s, x, n, v, phi, slopes));
  } else {
    CK_CUDA(launch_k((expand_f32_kernel<false>), blocks, kThreads, 0, s, x, n, v, phi, slopes));
  }
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_basis_eval(const float* t, int64_t n, const ck_lut* lut, float* vals, float* slopes, cudaStream_t s) {
  if (n == 0) return kOk;
  const LutView v = view(lut);
  CK_CHECK(v.K <= kMaxFeaturesRt, "ck_basis_eval: at most 64 features");
  LaunchScope scope(kKExpand, s);
  CK_CUDA(launch_k((basis_eval_kernel), grid_for(n, 8), kThreads, 0, s, t, n, v, vals, slopes));
  return kOk;
}

int launch_expand_planes(const float* x, int64_t rows, int cols, const ck_lut* lut, int k0,
                         __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ld, int64_t plane, cudaStream_t s) {
  if (rows == 0 || cols == 0 || k0 >= lut->n_feat) return kOk;
  CK_CHECK(ld % 2 == 0 && plane % 2 == 0, "expand_planes: pitch must be even");
  const LutView v = view(lut);
  LaunchScope scope(kKExpand, s);
  if (k0 == 1 && ld % 4 == 0 && plane % 4 == 0 && v.K - 1 <= kMaxPlanesFused) {
    const int qb = grid_for(rows * ((cols + 3) / 4), 8);
    auto* h8 = reinterpret_cast<uint2*>(hi);
    auto* l8 = reinterpret_cast<uint2*>(lo);
    const int rc = v.exact ? launch_quads<kSrcExact>(v, x, rows, cols, h8, l8, ld, plane, qb, s)
                           : launch_quads<kSrcNodes>(v, x, rows, cols, h8, l8, ld, plane, qb, s);
    if (rc != kUnsupported) return rc;
  }
  const int blocks = grid_for(rows * ((cols + 1) / 2), 8);
  CK_CUDA(launch_k((expand_planes_kernel), blocks, kThreads, 0, s, x, rows, cols, v, k0, reinterpret_cast<uint32_t*>(hi),
                                                   reinterpret_cast<uint32_t*>(lo), ld, plane));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_dx_combine(const float* g, int64_t g_plane, const float* x, int64_t rows, int cols,
                      const ck_lut* lut, int jacobian, float* dx, cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return kOk;
  const LutView v = view(lut);
  CK_CHECK(!v.exact || v.K <= kMaxK, "exact input gradient: at most 64 features");
  const size_t tab = v.exact ? 0 : sizeof(float) * v.N * v.K;
  const int blocks = grid_for(n, 8);
  LaunchScope scope(kKDxCombine, s);
  if (tab > 0 && tab <= static_cast<size_t>(kSmemLutMax)) {
    CK_CUDA(cudaFuncSetAttribute(dx_combine_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(tab)));
    CK_CUDA(launch_k((dx_combine_kernel<true>), blocks, kThreads, tab, s, g, g_plane, x, n, v, jacobian, dx));
  } else {
    CK_CUDA(launch_k((dx_combine_kernel<false>), blocks, kThreads, 0, s, g, g_plane, x, n, v, jacobian, dx));
  }
  CK_CUDA(cudaGetLastError());
  return kOk;
}

}  // namespace ck
