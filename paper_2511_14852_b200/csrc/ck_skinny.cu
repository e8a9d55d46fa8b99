// Skinny-output layers (d_out <= 8, e.g. the tabular regression head
// [512 -> 1]): CUDA-core kernels that evaluate the basis in registers and
// never materialise basis planes.  A tensor-core tile would be >= 128 wide
// in the output dimension, so for a handful of outputs the contraction is a
// per-row dot product (arithmetic intensity ~ 2*O*K flops per 4-byte input):
// HBM-bound on x (and dy), not tensor-bound.
//
// forward : y[b][o] = sum_i sum_k B_k(tanh x[b][i]) C[k][o][i] + bias[o]
//           one warp per 4 rows, lanes stride the inputs, fixed shuffle-tree
//           row reduction (deterministic)
// backward: one pass over (x, dy): dX in place; dC[k][o][i] and db as
//           per-row-block partials (fixed warp order), then the ordered
//           slot merge -- the reference's two-stage reduction
//           (kernels.py:428-442) without atomics.
#include "ck_basis.cuh"
#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

// Basis values v[0..P] of one element (P = compile-time bound >= K-1; the
// entries past K-1 are finite and meet zero coefficients): the LUT
// interpolation between the two (float32-rounded) grid nodes of the element's
// float32 cell, or the basis at t (exact handles).  The kind switch is
// uniform across the launch; each case is a fully unrolled recurrence.
template <int P>
__device__ __forceinline__ void elem_basis(const LutView& L, float xv, float (&v)[P + 1]) {
  float a[P + 1], b[P + 1];
  float x0, x1 = 0.0f, f = 0.0f;
  if (L.exact) {
    x0 = tanhf(xv);
  } else {
    int idx;
    cell_f32(xv, L.N, idx, f);
    x0 = grid_node_f(idx, L.N, 2.0f / static_cast<float>(L.N - 1));
    x1 = grid_node_f(idx + 1, L.N, 2.0f / static_cast<float>(L.N - 1));
  }
  switch (L.kind) {
    case kLegendre:
      basis_f32<kLegendre, P>(x0, a);
      if (!L.exact) basis_f32<kLegendre, P>(x1, b);
      break;
    case kHermite:
      basis_f32<kHermite, P>(x0, a);
      if (!L.exact) basis_f32<kHermite, P>(x1, b);
      break;
    case kFourier:
      if constexpr (P % 2 == 0) {  // Fourier K = 2d + 1: P = K - 1 is even
        basis_f32<kFourier, P>(x0, a);
        if (!L.exact) basis_f32<kFourier, P>(x1, b);
      }
      break;
    case kChebTrig:
      basis_f32<kChebTrig, P>(x0, a);
      break;
    default:
      basis_f32<kCheb, P>(x0, a);
      if (!L.exact) basis_f32<kCheb, P>(x1, b);
      break;
  }
#pragma unroll
  for (int k = 0; k <= P; ++k) v[k] = L.exact ? a[k] : lerp_ref(a[k], b[k], f);
}

// Analytic derivatives at t (exact handles).
template <int P>
__device__ __forceinline__ void elem_deriv(int kind, float t, float (&dv)[P + 1]) {
  switch (kind) {
    case kLegendre:
      deriv_f32<kLegendre, P>(t, dv);
      break;
    case kHermite:
      deriv_f32<kHermite, P>(t, dv);
      break;
    case kFourier:
      if constexpr (P % 2 == 0) deriv_f32<kFourier, P>(t, dv);
      break;
    default:
      deriv_f32<kCheb, P>(t, dv);  // also the trig form (same derivative)
      break;
  }
}

// LUT cell slopes sv[1..P] of one element (sv[0] = 0, entries >= K zero):
// the exact reference cell as in the fused dX epilogue (float32 position; the
// cell boundaries loaded only inside the guard band), then the chord slopes
// recomputed at the cell's float32 grid nodes (three-term families) or the
// table's slopes (Fourier).
template <int P>
__device__ __forceinline__ void elem_slopes_lut(const LutView& L, float xv, float t, float (&sv)[P + 1]) {
  const float hN = 0.5f * static_cast<float>(L.N - 1);
  const float pos = fmaf(t, hN, hN);
  int cell = min(static_cast<int>(pos), L.N - 2);
  const float fr = pos - static_cast<float>(cell);
  const float guard = fminf(0.5f, fmaxf(1e-3f, 4e-7f * static_cast<float>(L.N)));
  const int S = dxrow_stride(L.K);
  if (fr < guard || fr > 1.0f - guard) {
    const float* row = L.dxrows + static_cast<int64_t>(cell) * S;
    const float bl = __ldg(row + L.K - 1), bh = __ldg(row + L.K);
    cell = min(cell + (xv < bl ? -1 : (xv < bh ? 0 : 1)), L.N - 2);  // x = +inf: N-2 as the reference
  }
  float sl[P];
  if (L.kind == kFourier) {
    const float* row = L.dxrows + static_cast<int64_t>(cell) * S;
#pragma unroll
    for (int k = 1; k <= P; ++k) sl[k - 1] = k < L.K ? __ldg(row + k - 1) : 0.0f;
  } else {
    const float stepf = 2.0f / static_cast<float>(L.N - 1);
    const float b = grid_node_f(cell, L.N, stepf), a = grid_node_f(cell + 1, L.N, stepf);
    if (L.kind == kLegendre) {
      chord_slopes<kLegendre, P>(b, a, sl);
    } else if (L.kind == kHermite) {
      chord_slopes<kHermite, P>(b, a, sl);
    } else {
      chord_slopes<kCheb, P>(b, a, sl);
    }
  }
  sv[0] = 0.0f;
#pragma unroll
  for (int k = 1; k <= P; ++k) sv[k] = k < L.K ? sl[k - 1] : 0.0f;
}

// One warp per row (grid-stride), lanes stride the inputs four at a time
// (independent basis evaluations in flight); fixed shuffle tree for the row
// reduction (deterministic).  KMAX = P + 1 >= K.
template <int O, int P>
__global__ void __launch_bounds__(256) skinny_fwd_kernel(const float* __restrict__ x, int64_t rows, int I, int K,
                                                         const float* __restrict__ c, const float* __restrict__ bias,
                                                         LutView L, float* __restrict__ y) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t plane = static_cast<int64_t>(O) * I;  // C[k] stride
  for (int64_t b = warp; b < rows; b += nwarps) {
    float acc[O];
#pragma unroll
    for (int o = 0; o < O; ++o) acc[o] = 0.0f;
    const float* xr = x + b * I;
    for (int i0 = lane; i0 < I; i0 += 128) {
      float xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = i0 + 32 * u < I ? __ldg(xr + i0 + 32 * u) : 0.0f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u;
        float v[P + 1];
        elem_basis<P>(L, xv[u], v);
        if (i < I) {
#pragma unroll
          for (int k = 0; k <= P; ++k) {
            if (k < K) {
#pragma unroll
              for (int o = 0; o < O; ++o)
                acc[o] = fmaf(v[k], __ldg(c + k * plane + static_cast<int64_t>(o) * I + i), acc[o]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < O; ++o) {
      float a = acc[o];
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) a += __shfl_xor_sync(0xffffffffu, a, s);
      acc[o] = a;
    }
    if (lane < O) {
      float out = acc[0];
#pragma unroll
      for (int o = 1; o < O; ++o)
        if (lane == o) out = acc[o];
      y[b * O + lane] = out + (bias ? bias[lane] : 0.0f);
    }
  }
}

// grid (slots, ceil(I/32)); block 256 = 8 warps; thread = (warp w, column
// i = 32*blockIdx.y + lane); rows of slot s: [s*rb, min((s+1)*rb, rows)),
// warp w takes rows w, w+8, ...  P + 1 = compile-time bound on K (loops are
// unrolled with k < K guards so the per-thread state stays in registers).
template <int O, int P>
__global__ void __launch_bounds__(256) skinny_bwd_kernel(const float* __restrict__ x, const float* __restrict__ dy,
                                                         int64_t rows, int I, int K, const float* __restrict__ c,
                                                         LutView L, int jacobian, int64_t rb,
                                                         float* __restrict__ dx, float* __restrict__ part_c,
                                                         double* __restrict__ part_b) {
  pdl_wait();
  constexpr int KMAX = P + 1;
  __shared__ float red[8][KMAX * O][32];
  __shared__ double redb[8][O];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.y * 32 + lane;
  const bool col_ok = i < I;
  const int ic = col_ok ? i : I - 1;
  const int64_t plane = static_cast<int64_t>(O) * I;
  float cr[KMAX][O], acc[KMAX][O];
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
#pragma unroll
    for (int o = 0; o < O; ++o) {
      cr[k][o] = k < K ? __ldg(c + k * plane + static_cast<int64_t>(o) * I + ic) : 0.0f;
      acc[k][o] = 0.0f;
    }
  double db[O];
#pragma unroll
  for (int o = 0; o < O; ++o) db[o] = 0.0;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rb;
  const int64_t r1 = r0 + rb < rows ? r0 + rb : rows;
  // Rows in groups of R (independent basis evaluations in flight); x and dy
  // of the next group are loaded while the current one is evaluated -- the
  // row loop was bound by the HBM latency of x (ncu: long-scoreboard stalls
  // on tanh's input).
  constexpr int R = KMAX * O <= 8 ? 4 : (KMAX * O <= 16 ? 2 : 1);  // register budget
  float xn[R], gn[R][O];
  auto load_group = [&](int64_t bg) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int64_t b = bg + 8 * u;
      const bool ok = b < r1;
      xn[u] = ok ? __ldg(x + b * I + ic) : 0.0f;
#pragma unroll
      for (int o = 0; o < O; ++o) gn[u][o] = ok ? __ldg(dy + b * O + o) : 0.0f;
    }
  };
  load_group(r0 + w);
  for (int64_t bg = r0 + w; bg < r1; bg += 8 * R) {
    float xg[R], g[R][O];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      xg[u] = xn[u];
#pragma unroll
      for (int o = 0; o < O; ++o) g[u][o] = gn[u][o];
    }
    load_group(bg + 8 * R);
    if (blockIdx.y == 0 && lane == 0) {
#pragma unroll
      for (int u = 0; u < R; ++u)
#pragma unroll
        for (int o = 0; o < O; ++o) db[o] += static_cast<double>(g[u][o]);  // zero past r1
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int64_t b = bg + 8 * u;
      if (b >= r1) break;
      const float xv = xg[u];
      float t = tanhf(xv);
      float vv[KMAX], sv[KMAX];
      if (L.exact) {
        elem_basis<P>(L, xv, vv);
        elem_deriv<P>(L.kind, t, sv);
      } else {
        t = fminf(fmaxf(t, -1.0f), 1.0f);
        elem_basis<P>(L, xv, vv);  // values are continuous: the float32 cell is fine
        elem_slopes_lut<P>(L, xv, t, sv);
      }
      float gx = 0.0f;
#pragma unroll
      for (int k = 1; k < KMAX; ++k) {
        float gk = 0.0f;
#pragma unroll
        for (int o = 0; o < O; ++o) gk = fmaf(g[u][o], cr[k][o], gk);
        gx = fmaf(sv[k], gk, gx);
      }
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int o = 0; o < O; ++o) acc[k][o] = fmaf(g[u][o], vv[k], acc[k][o]);
      if (dx && col_ok) dx[b * I + i] = jacobian ? gx * (1.0f - t * t) : gx;
    }
  }
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
#pragma unroll
    for (int o = 0; o < O; ++o) red[w][k * O + o][lane] = acc[k][o];
  if (lane == 0) {
#pragma unroll
    for (int o = 0; o < O; ++o) redb[w][o] = db[o];
  }
  __syncthreads();
  // fold the 8 warps in order
  for (int e = w; e < K * O; e += 8) {
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += red[j][e][lane];
    const int k = e / O, o = e - k * O;
    if (col_ok) part_c[(static_cast<int64_t>(blockIdx.x) * K + k) * plane + static_cast<int64_t>(o) * I + i] = s;
  }
  if (blockIdx.y == 0 && threadIdx.x < O) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += redb[j][threadIdx.x];
    part_b[static_cast<int64_t>(blockIdx.x) * O + threadIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// LUT-mode kernels of the three-term families (Chebyshev / Legendre /
// Hermite): the hot skinny path (the tabular head [512 -> 1]).  The kernels
// above spend ~115 (forward) / ~200 (backward) instructions per element
// (runtime kind switch per element, C reloaded per element and feature, tanh
// and both nodes' recurrences evaluated twice in the backward); these are
// issue-bound, so the per-element work is cut to the minimum:
//   forward : lanes own 4 consecutive inputs per 128-wide chunk (float4 x and
//             C loads, one C load per 4 elements and feature), one recurrence
//             per grid node, interpolate, dot;
//   backward: one tanh; the exact reference cell as in the fused dX
//             epilogue; ONE divided-difference recurrence over the cell
//             gives the chord slopes S_k (dX) and the left node's values
//             B_k(b), and the interpolated values follow as
//             B_k(b) + f (a - b) S_k  (= lerp(B_k(b), B_k(a), f)).

// S[k-1] = chord slope of feature k (k = 1..P) over [b, a] and vb[k] = B_k(b)
// (k = 0..P): chord_slopes (ck_basis.cuh) extended by the last value.
template <int KIND, int P>
__device__ __forceinline__ void chord_and_values(float b, float a, float (&S)[P], float (&vb)[P + 1]) {
  float pv = 1.0f, cv = KIND == kHermite ? 2.0f * b : b;  // B_0(b), B_1(b)
  float sp = 0.0f, sc = KIND == kHermite ? 2.0f : 1.0f;   // S_0, S_1
  vb[0] = 1.0f;
  vb[1] = cv;
  S[0] = sc;
#pragma unroll
  for (int k = 1; k < P; ++k) {
    float sn, vn;
    if constexpr (KIND == kCheb) {
      sn = fmaf(2.0f * a, sc, fmaf(2.0f, cv, -sp));
      vn = fmaf(2.0f * b, cv, -pv);
    } else if constexpr (KIND == kLegendre) {
      const float c2 = static_cast<float>(2 * k + 1), ck = static_cast<float>(k);
      const float inv = 1.0f / static_cast<float>(k + 1);
      sn = fmaf(c2, fmaf(a, sc, cv), -ck * sp) * inv;
      vn = fmaf(c2 * b, cv, -ck * pv) * inv;
    } else {
      const float c2k = static_cast<float>(2 * k);
      sn = fmaf(2.0f, fmaf(a, sc, cv), -c2k * sp);
      vn = fmaf(2.0f * b, cv, -c2k * pv);
    }
    S[k] = sn;
    vb[k + 1] = vn;
    sp = sc;
    sc = sn;
    pv = cv;
    cv = vn;
  }
}

// x, 4 consecutive inputs i0..i0+3 of a row (zero past I); vec: 16-byte path
__device__ __forceinline__ void load4(const float* p, int i0, int I, bool vec, float (&v)[4]) {
  if (vec && i0 + 4 <= I) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p + i0));
    v[0] = q.x;
    v[1] = q.y;
    v[2] = q.z;
    v[3] = q.w;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = i0 + e < I ? __ldg(p + i0 + e) : 0.0f;
  }
}

// Interpolated LUT values v[1..P] of one element (the forward's float32
// cell; the interpolant is continuous, so no boundary check): one recurrence
// per grid node, then lerp.  ~4P + 16 instructions.
template <int KIND, int P>
__device__ __forceinline__ void lut_values(float xv, float hN, float stepf, int N, float (&v)[P + 1]) {
  const float t = tanh_fast(xv);  // in [-1, 1]
  const int idx = min(static_cast<int>(fmaf(t, hN, hN)), N - 2);
  const float fi = static_cast<float>(idx);
  const float f = fmaf(t, hN, hN - fi);
  const float x0 = fmaf(fi, stepf, -1.0f);
  const float x1 = idx + 1 >= N - 1 ? 1.0f : fmaf(fi + 1.0f, stepf, -1.0f);  // grid_node_f(idx + 1)
  float v0[P + 1], v1[P + 1];
  basis_f32<KIND, P>(x0, v0);
  basis_f32<KIND, P>(x1, v1);
#pragma unroll
  for (int k = 1; k <= P; ++k) v[k] = lerp_ref(v0[k], v1[k], f);
}

// One pass of a lane: QJ quads of inputs p0 + 4 (lane + 32 j).  FULL: all
// in range and 16-byte aligned (no checks); otherwise C loads past I read as
// zero, so padded inputs (x = 0, finite values) contribute nothing.
template <int KIND, int O, int P, int QJ, bool FULL, bool KX>
__device__ __forceinline__ void skinny_fwd_pass(const float (&xq)[QJ][4], int p0, int lane, int I, int K,
                                                const float* __restrict__ c, int64_t plane, float hN, float stepf,
                                                int N, float (&acc)[O]) {
#pragma unroll
  for (int j = 0; j < QJ; ++j) {
    const int i0 = p0 + 4 * (lane + 32 * j);
    if (!FULL && i0 >= I) break;
    float v[4][P + 1];
#pragma unroll
    for (int e = 0; e < 4; ++e) lut_values<KIND, P>(xq[j][e], hN, stepf, N, v[e]);
#pragma unroll
    for (int k = 0; k <= P; ++k) {
      if (KX || k < K) {  // KX: K == P + 1 (compile-time)
#pragma unroll
        for (int o = 0; o < O; ++o) {
          const float* cp = c + k * plane + static_cast<int64_t>(o) * I + i0;
          float cv[4];
          if (FULL) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(cp));
            cv[0] = q.x; cv[1] = q.y; cv[2] = q.z; cv[3] = q.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) cv[e] = i0 + e < I ? __ldg(cp + e) : 0.0f;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[o] = k == 0 ? acc[o] + cv[e] : fmaf(v[e][k], cv[e], acc[o]);  // B_0 == 1
        }
      }
    }
  }
}

// One warp per row (grid-stride over rows); a pass covers 512 inputs of the
// row: lane l owns the 4-input quads l, l + 32, l + 64, l + 96 (float4 x and C
// loads).  The x of the next pass (this row's next 512 inputs or the next
// row's first) is loaded before the current pass is evaluated, so the HBM
// latency of x overlaps the basis work (ncu: the row loop stalled on x,
// 33 % long-scoreboard).  Full passes (16-byte aligned, 512 inputs in range)
// skip every bounds check.
template <int KIND, int O, int P>
__device__ __forceinline__ void skinny_fwd_lut_rows(const float* __restrict__ x, int64_t rows, int I, int K,
                                                    const float* __restrict__ c, const float* __restrict__ bias,
                                                    int N, bool vec, float* __restrict__ y) {
  constexpr int QJ = 4, PASS = 128 * QJ;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t plane = static_cast<int64_t>(O) * I;
  const float hN = 0.5f * static_cast<float>(N - 1);
  const float stepf = 2.0f / static_cast<float>(N - 1);
  const int passes = (I + PASS - 1) / PASS;
  auto load_pass = [&](int64_t b, int p0, float (&xq)[QJ][4]) {
    if (b >= rows) return;
    const float* xr = x + b * I;
#pragma unroll
    for (int j = 0; j < QJ; ++j) load4(xr, p0 + 4 * (lane + 32 * j), I, vec, xq[j]);
  };
  float xn[QJ][4];
  load_pass(warp, 0, xn);
  for (int64_t b = warp; b < rows; b += nwarps) {
    float acc[O];
#pragma unroll
    for (int o = 0; o < O; ++o) acc[o] = 0.0f;
    for (int p = 0; p < passes; ++p) {
      const int p0 = p * PASS;
      float xq[QJ][4];
#pragma unroll
      for (int j = 0; j < QJ; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) xq[j][e] = xn[j][e];
      if (p + 1 < passes) {
        load_pass(b, p0 + PASS, xn);
      } else {
        load_pass(b + nwarps, 0, xn);
      }
      if (vec && p0 + PASS <= I) {
        if (K == P + 1) {
          skinny_fwd_pass<KIND, O, P, QJ, true, true>(xq, p0, lane, I, K, c, plane, hN, stepf, N, acc);
        } else {
          skinny_fwd_pass<KIND, O, P, QJ, true, false>(xq, p0, lane, I, K, c, plane, hN, stepf, N, acc);
        }
      } else {
        skinny_fwd_pass<KIND, O, P, QJ, false, false>(xq, p0, lane, I, K, c, plane, hN, stepf, N, acc);
      }
    }
#pragma unroll
    for (int o = 0; o < O; ++o) {
      float a = acc[o];
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) a += __shfl_xor_sync(0xffffffffu, a, s);
      acc[o] = a;
    }
    if (lane < O) {
      float out = acc[0];
#pragma unroll
      for (int o = 1; o < O; ++o)
        if (lane == o) out = acc[o];
      y[b * O + lane] = out + (bias ? bias[lane] : 0.0f);
    }
  }
}

template <int O, int P>
__global__ void __launch_bounds__(256) skinny_fwd_lut_kernel(const float* __restrict__ x, int64_t rows, int I, int K,
                                                             const float* __restrict__ c,
                                                             const float* __restrict__ bias, LutView L, int vec,
                                                             float* __restrict__ y) {
  pdl_wait();
  switch (L.kind) {  // uniform: one body runs
    case kLegendre:
      skinny_fwd_lut_rows<kLegendre, O, P>(x, rows, I, K, c, bias, L.N, vec != 0, y);
      break;
    case kHermite:
      skinny_fwd_lut_rows<kHermite, O, P>(x, rows, I, K, c, bias, L.N, vec != 0, y);
      break;
    default:
      skinny_fwd_lut_rows<kCheb, O, P>(x, rows, I, K, c, bias, L.N, vec != 0, y);
      break;
  }
}

template <int KIND, int O, int P>
__device__ __forceinline__ void skinny_bwd_lut_body(const float* __restrict__ x, const float* __restrict__ dy,
                                                    int64_t rows, int I, int K, const float* __restrict__ c,
                                                    const LutView& L, int jacobian, int64_t rb,
                                                    float* __restrict__ dx, float* __restrict__ part_c,
                                                    double* __restrict__ part_b, float (*red)[(P + 1) * O][32],
                                                    double (*redb)[O]) {
  constexpr int KMAX = P + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.y * 32 + lane;
  const bool col_ok = i < I;
  const int ic = col_ok ? i : I - 1;
  const int64_t plane = static_cast<int64_t>(O) * I;
  const int N = L.N, S = dxrow_stride(K);
  const float hN = 0.5f * static_cast<float>(N - 1);
  const float stepf = 2.0f / static_cast<float>(N - 1);
  const float guard = fminf(0.5f, fmaxf(1e-3f, 4e-7f * static_cast<float>(N)));
  float cr[KMAX][O], acc[KMAX][O];
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
#pragma unroll
    for (int o = 0; o < O; ++o) {
      cr[k][o] = k < K ? __ldg(c + k * plane + static_cast<int64_t>(o) * I + ic) : 0.0f;
      acc[k][o] = 0.0f;
    }
  double db[O];
#pragma unroll
  for (int o = 0; o < O; ++o) db[o] = 0.0;
  // this warp's rows: first, first + 8, ... < r1 (n of them); running
  // pointers, one 64-bit add per row instead of an index product
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rb;
  const int64_t r1 = r0 + rb < rows ? r0 + rb : rows;
  const int64_t first = r0 + w;
  const int n = first < r1 ? static_cast<int>((r1 - first + 7) / 8) : 0;
  const int64_t xs = 8 * static_cast<int64_t>(I);
  const float* xp = x + first * I + ic;
  const float* gp = dy + first * O;
  float* dxp = (dx != nullptr && col_ok) ? dx + first * I + i : nullptr;
  const bool db_block = blockIdx.y == 0;  // uniform
  constexpr int R = KMAX * O <= 8 ? 4 : (KMAX * O <= 16 ? 2 : 1);  // rows in flight (register budget)
  float xn[R], gn[R][O];
  auto load_group = [&](int j0) {
    const float* xq = xp;
    const float* gq = gp;
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const bool ok = j0 + u < n;
      xn[u] = ok ? __ldg(xq) : 0.0f;
#pragma unroll
      for (int o = 0; o < O; ++o) gn[u][o] = ok ? __ldg(gq + o) : 0.0f;
      xq += xs;
      gq += 8 * O;
    }
  };
  load_group(0);
  for (int j = 0; j < n; j += R) {
    float xg[R], g[R][O];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      xg[u] = xn[u];
#pragma unroll
      for (int o = 0; o < O; ++o) g[u][o] = gn[u][o];
    }
    xp += R * xs;
    gp += R * 8 * O;
    load_group(j + R);
    if (db_block) {
#pragma unroll
      for (int u = 0; u < R; ++u)
#pragma unroll
        for (int o = 0; o < O; ++o) db[o] += static_cast<double>(g[u][o]);  // zero past n
    }
    // phase 1, all rows of the group: tanh, float32 cell and, inside the
    // guard band, the loads of the cell's reference boundaries -- issued for
    // the whole group before any is consumed (a band element in ~half the
    // warps made every row wait one L2 round trip: 31 % long-scoreboard
    // stalls on the boundary compare)
    float tg[R], jg[R], bl[R], bh[R];
    int cg[R];
    bool band[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      tanh_jac(xg[u], tg[u], jg[u]);
      const float pos = fmaf(tg[u], hN, hN);
      cg[u] = min(static_cast<int>(pos), N - 2);
      const float fr = pos - static_cast<float>(cg[u]);
      band[u] = fr < guard || fr > 1.0f - guard;
      bl[u] = bh[u] = 0.0f;
      if (band[u]) {
        const float* row = L.dxrows + static_cast<int64_t>(cg[u]) * S;
        bl[u] = __ldg(row + K - 1);
        bh[u] = __ldg(row + K);
      }
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      if (j + u >= n) break;
      const float xv = xg[u];
      const float t = tg[u], jac = jg[u];
      int cell = cg[u];
      if (band[u]) {
        // exact reference cell b_c <= x < b_{c+1} (at most one step off)
        cell = min(cell + (xv < bl[u] ? -1 : (xv < bh[u] ? 0 : 1)), N - 2);  // x = +inf: N-2 as the reference
      }
      const float fc = static_cast<float>(cell);
      const float f = fmaf(t, hN, hN - fc);
      const float nb = fmaf(fc, stepf, -1.0f);
      const float na = cell + 1 >= N - 1 ? 1.0f : fmaf(fc + 1.0f, stepf, -1.0f);  // grid_node_f(cell + 1)
      float sl[P], vb[P + 1];
      chord_and_values<KIND, P>(nb, na, sl, vb);
      const float fs = f * (na - nb);
      float gx = 0.0f;
#pragma unroll
      for (int o = 0; o < O; ++o) {
        float so = 0.0f;
#pragma unroll
        for (int k = 1; k < KMAX; ++k) so = fmaf(sl[k - 1], cr[k][o], so);
        gx = fmaf(g[u][o], so, gx);
        acc[0][o] += g[u][o];
      }
#pragma unroll
      for (int k = 1; k < KMAX; ++k) {
        const float v = fmaf(fs, sl[k - 1], vb[k]);  // lerp(B_k(b), B_k(a), f)
#pragma unroll
        for (int o = 0; o < O; ++o) acc[k][o] = fmaf(g[u][o], v, acc[k][o]);
      }
      if (dxp != nullptr) dxp[static_cast<int64_t>(j + u) * xs] = jacobian ? gx * jac : gx;
    }
  }
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
#pragma unroll
    for (int o = 0; o < O; ++o) red[w][k * O + o][lane] = acc[k][o];
  if (lane == 0) {
#pragma unroll
    for (int o = 0; o < O; ++o) redb[w][o] = db[o];
  }
  __syncthreads();
  for (int e = w; e < K * O; e += 8) {  // fold the 8 warps in order
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += red[j][e][lane];
    const int k = e / O, o = e - k * O;
    if (col_ok) part_c[(static_cast<int64_t>(blockIdx.x) * K + k) * plane + static_cast<int64_t>(o) * I + i] = s;
  }
  if (blockIdx.y == 0 && threadIdx.x < O) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += redb[j][threadIdx.x];
    part_b[static_cast<int64_t>(blockIdx.x) * O + threadIdx.x] = s;
  }
}

template <int O, int P>
__global__ void __launch_bounds__(256) skinny_bwd_lut_kernel(const float* __restrict__ x, const float* __restrict__ dy,
                                                             int64_t rows, int I, int K, const float* __restrict__ c,
                                                             LutView L, int jacobian, int64_t rb,
                                                             float* __restrict__ dx, float* __restrict__ part_c,
                                                             double* __restrict__ part_b) {
  __shared__ float red[8][(P + 1) * O][32];
  __shared__ double redb[8][O];
  pdl_wait();
  switch (L.kind) {
    case kLegendre:
      skinny_bwd_lut_body<kLegendre, O, P>(x, dy, rows, I, K, c, L, jacobian, rb, dx, part_c, part_b, red, redb);
      break;
    case kHermite:
      skinny_bwd_lut_body<kHermite, O, P>(x, dy, rows, I, K, c, L, jacobian, rb, dx, part_c, part_b, red, redb);
      break;
    default:
      skinny_bwd_lut_body<kCheb, O, P>(x, dy, rows, I, K, c, L, jacobian, rb, dx, part_c, part_b, red, redb);
      break;
  }
}

// the LUT kernels above serve the three-term families; exact handles and
// Fourier tables take the generic kernels
bool skinny_lut_fast(const LutView& L) {
  return !L.exact && (L.kind == kCheb || L.kind == kLegendre || L.kind == kHermite);
}

int round_o(int O) { return O <= 1 ? 1 : O <= 2 ? 2 : O <= 4 ? 4 : 8; }

int skinny_p(int O, int K) {
  if (O == 1 && K <= 9) return K > 2 ? K - 1 : (K == 2 ? 1 : 1);
  return K <= 5 ? 4 : K <= 9 ? 8 : K <= 17 ? 16 : 32;
}

}  // namespace

bool skinny_layer(int d_in, int d_out, int n_feat) {
  (void)d_in;
  return d_out <= kSkinnyMaxO && n_feat * round_o(d_out) <= kSkinnyMaxKO;
}

// Resident blocks per SM of the backward instantiation for (O, K): the grid
// is sized to one full wave (a partial second wave cost up to a third of the
// kernel: 592 blocks of the C2 head on 444 slots).
int skinny_bwd_blocks_per_sm(int O, int K) {
  const int pm = skinny_p(O, K);
  int n = 0;
#define CK_OCC(OO, PP)                                                                           \
  if (O == OO && pm == PP) {                                                                     \
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, skinny_bwd_lut_kernel<OO, PP>, 256, 0) != \
        cudaSuccess)                                                                                 \
      n = 0;                                                                                         \
  } else
  CK_OCC(1, 1) CK_OCC(1, 2) CK_OCC(1, 3) CK_OCC(1, 5) CK_OCC(1, 6) CK_OCC(1, 7)
  CK_OCC(1, 4) CK_OCC(1, 8) CK_OCC(1, 16) CK_OCC(1, 32) CK_OCC(2, 4) CK_OCC(2, 8) CK_OCC(2, 16)
  CK_OCC(3, 4) CK_OCC(3, 8) CK_OCC(4, 4) CK_OCC(4, 8)
  CK_OCC(5, 4) CK_OCC(6, 4) CK_OCC(7, 4) CK_OCC(8, 4) {}
#undef CK_OCC
  return n > 0 ? n : 1;
}

int skinny_slots(int64_t rows, int d_in, int d_out, int n_feat) {
  const int64_t colblocks = ceil_div(d_in, 32);
  const int64_t wave = static_cast<int64_t>(skinny_bwd_blocks_per_sm(d_out, n_feat)) * num_sms();
  int64_t slots = wave / colblocks;
  const int64_t max_slots = ceil_div(rows > 0 ? rows : 1, 64);  // >= 64 rows per slot
  if (slots > max_slots) slots = max_slots;
  if (slots > kSkinnyMaxSlots) slots = kSkinnyMaxSlots;
  return static_cast<int>(slots < 1 ? 1 : slots);
}

int launch_skinny_forward(const float* x, int64_t rows, int I, int O, const float* c, const float* bias,
                          const ck_lut* lut, float* y, cudaStream_t s) {
  if (rows == 0) return kOk;
  const LutView L = view(lut);
  const int64_t want = ceil_div(rows * 32, 256);  // one warp per row
  const int K = L.K;
  LaunchScope scope(kKSkinny, s);
  // P: smallest of 4 / 8 / 16 / 32 with P + 1 >= K (even, as Fourier needs);
  // single-output heads get P = K - 1 exactly up to K = 9
  const int pm = skinny_p(O, K);
  const bool fast = skinny_lut_fast(L);
  // 16-byte x / C loads when every row and coefficient row starts aligned
  const int vec = (I % 4 == 0) && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(c) & 15) == 0;
  // grid: one wave of resident blocks (grid-stride over rows)
  auto blocks_for = [&](auto kernel) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
    const int64_t cap = static_cast<int64_t>(num_sms()) * per_sm;
    return static_cast<int>(want < cap ? want : cap);
  };
#define CK_SK(OO, PP)                                                                                            \
  if (O == OO && pm == PP) {                                                                                     \
    if (fast) {                                                                                                  \
      CK_CUDA(launch_k((skinny_fwd_lut_kernel<OO, PP>), blocks_for(skinny_fwd_lut_kernel<OO, PP>), 256, 0, s, x, \
                       rows, I, K, c, bias, L, vec, y));                                                         \
    } else {                                                                                                     \
      CK_CUDA(launch_k((skinny_fwd_kernel<OO, PP>), blocks_for(skinny_fwd_kernel<OO, PP>), 256, 0, s, x, rows, I, \
                       K, c, bias, L, y));                                                                       \
    }                                                                                                            \
  } else
  CK_SK(1, 1) CK_SK(1, 2) CK_SK(1, 3) CK_SK(1, 5) CK_SK(1, 6) CK_SK(1, 7)
  CK_SK(1, 4) CK_SK(1, 8) CK_SK(1, 16) CK_SK(1, 32) CK_SK(2, 4) CK_SK(2, 8) CK_SK(2, 16)
  CK_SK(3, 4) CK_SK(3, 8) CK_SK(4, 4) CK_SK(4, 8)
  CK_SK(5, 4) CK_SK(6, 4) CK_SK(7, 4) CK_SK(8, 4) {
    set_error("skinny forward: unsupported (d_out, features)");
    return kUnsupported;
  }
#undef CK_SK
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_skinny_backward(const float* x, const float* dy, int64_t rows, int I, int O, const float* c,
                           const ck_lut* lut, int jacobian, float* dx, float* part_c, double* part_b, int slots,
                           cudaStream_t s) {
  const LutView L = view(lut);
  const int K = L.K;
  const int64_t rb = ceil_div(rows > 0 ? rows : 1, slots);
  const dim3 grid(static_cast<unsigned>(slots), static_cast<unsigned>(ceil_div(I, 32)));
  LaunchScope scope(kKSkinny, s);
  const int ro = round_o(O);
  CK_CHECK(K * ro <= kSkinnyMaxKO, "skinny backward: too many features x outputs");
  // P + 1 >= K as in the forward (register budget: K * round_o(O) <= 32)
  const int pm = skinny_p(O, K);
#define CK_SKB(OO, PP)                                                                                        \
  if (O == OO && pm == PP) {                                                                                  \
    if (skinny_lut_fast(L)) {                                                                                 \
      CK_CUDA(launch_k((skinny_bwd_lut_kernel<OO, PP>), grid, 256, 0, s, x, dy, rows, I, K, c, L, jacobian, rb, dx, \
                       part_c, part_b));                                                                      \
    } else {                                                                                                  \
      CK_CUDA(launch_k((skinny_bwd_kernel<OO, PP>), grid, 256, 0, s, x, dy, rows, I, K, c, L, jacobian, rb, dx, \
                       part_c, part_b));                                                                      \
    }                                                                                                         \
  } else
  CK_SKB(1, 1) CK_SKB(1, 2) CK_SKB(1, 3) CK_SKB(1, 5) CK_SKB(1, 6) CK_SKB(1, 7)
  CK_SKB(1, 4) CK_SKB(1, 8) CK_SKB(1, 16) CK_SKB(1, 32) CK_SKB(2, 4) CK_SKB(2, 8) CK_SKB(2, 16)
  CK_SKB(3, 4) CK_SKB(3, 8) CK_SKB(4, 4) CK_SKB(4, 8)
  CK_SKB(5, 4) CK_SKB(6, 4) CK_SKB(7, 4) CK_SKB(8, 4) {
    set_error("skinny backward: unsupported (d_out, features)");
    return kUnsupported;
  }
#undef CK_SKB
  CK_CUDA(cudaGetLastError());
  return kOk;
}

}  // namespace ck

// ---------------------------------------------------------------------------
// The reference's two-stage forward, stage by stage (forward_partial /
// combine, kernels.py:263-348), for callers that use the partial buffer
// itself.  One warp per (row b, output tile to): lanes own the tile's
// outputs; the features of 32 inputs at a time are evaluated one per lane
// (table interpolation or exact, streamed by Rec) and broadcast by shuffles;
// every (b, to, ti) slot is written exactly once, in fp32 FMA order
// j ascending, k ascending.  CUDA cores: the fast path is ck_forward.
namespace ck {
namespace {

__global__ void __launch_bounds__(256) forward_partial_kernel(const float* __restrict__ x, int64_t rows, int I, int O,
                                                              int K, const float* __restrict__ c, LutView L,
                                                              int tile_in, int tile_out, int g_x, int g_y,
                                                              float* __restrict__ part,
                                                              unsigned long long* __restrict__ counts) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t items = rows * g_y;
  for (int64_t w = warp; w < items; w += nwarps) {
    const int64_t b = w / g_y;
    const int to = static_cast<int>(w - b * g_y);
    const float* xr = x + b * I;
    for (int ty0 = 0; ty0 < tile_out; ty0 += 32) {
      const int ty = ty0 + lane;
      const int o = to * tile_out + ty;
      const bool o_ok = ty < tile_out && o < O;
      for (int ti = 0; ti < g_x; ++ti) {
        const int j_begin = ti * tile_in;
        const int j_end = min(I, j_begin + tile_in);
        float acc = 0.0f;
        for (int j0 = j_begin; j0 < j_end; j0 += 32) {
          const int jl = j0 + lane;
          const bool j_ok = jl < j_end;
          const float xv = j_ok ? __ldg(xr + jl) : 0.0f;
          Rec ra, rb;
          float f = 0.0f;
          if (L.exact) {
            ra.init(L.kind, tanhf(xv));
          } else {
            int idx;
            cell_f32(xv, L.N, idx, f);
            const float step = 2.0f / static_cast<float>(L.N - 1);
            ra.init(L.kind, grid_node_f(idx, L.N, step));
            rb.init(L.kind, grid_node_f(idx + 1, L.N, step));
          }
          const int nj = min(32, j_end - j0);
          for (int k = 0; k < K; ++k) {
            float v = 1.0f;
            if (k > 0) {
              const float a = ra.next();
              v = L.exact ? a : lerp_ref(a, rb.next(), f);
            }
            const float* crow = c + (static_cast<int64_t>(k) * O + (o_ok ? o : 0)) * I + j0;
            for (int jj = 0; jj < nj; ++jj) {
              const float vj = __shfl_sync(0xffffffffu, v, jj);
              if (o_ok) acc = fmaf(vj, __ldg(crow + jj), acc);
            }
          }
        }
        if (o_ok) {
          const int64_t slot = ((static_cast<int64_t>(to) * g_x + ti) * rows + b) * tile_out + ty;
          part[slot] = acc;
          // instrumented buffers: every store counts itself (atomically, so
          // a second writer of a slot would show up as 2)
          if (counts) atomicAdd(counts + slot, 1ull);
        }
      }
    }
  }
}

// y[b][o] = sum_{ti ascending} part[to][ti][b][ty] (+ bias[o])
__global__ void __launch_bounds__(256) combine_kernel(const float* __restrict__ part, int64_t rows, int O, int tile_out,
                                                      int g_x, const float* __restrict__ bias, float* __restrict__ y) {
  pdl_wait();
  const int64_t n = rows * O;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = e / O;
    const int o = static_cast<int>(e - b * O);
    const int to = o / tile_out, ty = o - to * tile_out;
    float acc = part[((static_cast<int64_t>(to) * g_x) * rows + b) * tile_out + ty];
    for (int ti = 1; ti < g_x; ++ti) acc += part[((static_cast<int64_t>(to) * g_x + ti) * rows + b) * tile_out + ty];
    y[e] = bias ? acc + bias[o] : acc;
  }
}

}  // namespace
}  // namespace ck

extern "C" int ck_forward_partial(const float* x, int64_t batch, int d_in, int d_out, const ck_lut* lut,
                                  const float* coeff_doj, int tile_in, int tile_out, float* partial,
                                  long long* write_counts, void* stream) {
  CK_CHECK(lut != nullptr, "LUT mode requires a LutTable");
  CK_CHECK(batch >= 0 && d_in >= 1 && d_out >= 1, "d_in and d_out must be >= 1");
  CK_CHECK(tile_in >= 1 && tile_out >= 1, "tile and lane sizes must be >= 1");
  if (batch == 0) return ck::kOk;
  CK_CHECK(x && coeff_doj && partial, "ck_forward_partial: NULL tensor");
  const int g_x = static_cast<int>(ck::ceil_div(d_in, tile_in)), g_y = static_cast<int>(ck::ceil_div(d_out, tile_out));
  const ck::LutView L = ck::view(lut);
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t warps = batch * g_y;
  const int64_t want = ck::ceil_div(warps * 32, 256);
  const int64_t cap = static_cast<int64_t>(ck::num_sms()) * 16;
  ck::LaunchScope scope(ck::kKSkinny, s);
  CK_CUDA(ck::launch_k((ck::forward_partial_kernel), static_cast<int>(want < cap ? want : cap), 256, 0, s, x, batch,
                       d_in, d_out, L.K, coeff_doj, L, tile_in, tile_out, g_x, g_y, partial,
                       reinterpret_cast<unsigned long long*>(write_counts)));
  return ck::kOk;
}

extern "C" int ck_combine(const float* partial, int64_t batch, int d_out, int tile_in_groups, int tile_out,
                          const float* bias, float* y, void* stream) {
  CK_CHECK(batch >= 0 && d_out >= 1 && tile_in_groups >= 1 && tile_out >= 1, "ck_combine: bad extents");
  if (batch == 0) return ck::kOk;
  CK_CHECK(partial && y, "ck_combine: NULL tensor");
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t want = ck::ceil_div(batch * d_out, 256);
  const int64_t cap = static_cast<int64_t>(ck::num_sms()) * 8;
  ck::LaunchScope scope(ck::kKReduce, s);
  CK_CUDA(ck::launch_k((ck::combine_kernel), static_cast<int>(want < cap ? want : cap), 256, 0, s, partial, batch,
                       d_out, tile_out, tile_in_groups, bias, y));
  return ck::kOk;
}
