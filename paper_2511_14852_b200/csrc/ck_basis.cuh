// Basis families evaluated in float32 on the device: values (basis_rows,
// basis.py:87-119) and analytic derivatives (derivative_rows,
// basis.py:155-204) of the Chebyshev / Legendre / Hermite / Fourier
// families, plus the cos(k acos t) Chebyshev form (trig_rows,
// basis.py:144-152).  P = number of non-constant features (K - 1), a
// compile-time constant so every recurrence fully unrolls into registers.
//
// Used by the expansion kernels (values at the two grid nodes of a LUT cell,
// or at t itself in exact mode) and by the exact-mode input-gradient
// epilogue (derivatives at t).
#pragma once

#include <cuda_runtime.h>

namespace ck {

enum BasisKindId : int { kCheb = 0, kLegendre = 1, kHermite = 2, kFourier = 3, kChebTrig = 4 };

// runtime-degree paths (local arrays): features <= 64
constexpr int kMaxFeaturesRt = 64;

// feature_count (basis.py:24-34)
__host__ __device__ inline int basis_features(int kind, int degree) {
  return kind == kFourier ? 2 * degree + 1 : degree + 1;
}

// tanh(x) in 5 instructions (ex2 / rcp approximations; tanhf is ~14 plus a
// branch): with r = 1 / (1 + e^{2|x|}) in (0, 1/2], t = sign(x) (1 - 2r),
// |t| <= 1 by construction, +-inf -> +-1.  Absolute error ~1e-7 over the
// whole range -- what the LUT paths consume: the cell position has ~1e-7 * N
// cells of error (the same order as a 2-ulp tanhf near |t| = 1), and the
// interpolated values are continuous in t.  (Exact-mode bases keep tanhf:
// there t itself is the argument of the polynomial.)
__device__ __forceinline__ float tanh_r(float x, float& r) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(x) * 2.8853900817779268f));  // e^{2|x|}
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
  return copysignf(fmaf(-2.0f, r, 1.0f), x);
}

__device__ __forceinline__ float tanh_fast(float x) {
  float r;
  return tanh_r(x, r);
}

// Fast cell choice for value interpolation (float32).  frac is formed with
// one rounding (fma of t*h against the exact h - idx), so the interpolated
// value is accurate to ~k^2 * ulp(t); a cell flip at an edge is harmless for
// values because the interpolant is continuous.
__device__ __forceinline__ void cell_f32(float xv, int n, int& idx, float& frac) {
  const float t = tanh_fast(xv);  // in [-1, 1]
  const float h = 0.5f * static_cast<float>(n - 1);
  const float pos = fmaf(t, h, h);
  int i = static_cast<int>(pos);
  i = min(i, n - 2);
  idx = i;
  frac = fmaf(t, h, h - static_cast<float>(i));
}

// t = tanh(x) and the Jacobian J = 1 - t^2 of the input-gradient paths in
// ~9 instructions (tanhf alone is 14 plus 2 for J): with r = 1 / (1 + e^{2|x|})
// in (0, 1/2], t = sign(x) (1 - 2r) and J = 4 r (1 - r) -- no cancellation,
// so J keeps ~1e-6 relative accuracy out to |x| ~ 44 where 1 - t*t in float32
// has none.  t has ~1e-7 absolute error (ex2 / rcp approximations): the
// position it gives is within 1.2e-7 * N cells of the reference's, inside the
// guard band (4e-7 * N cells) where the cell is settled against the exact
// float32 boundaries; the values interpolate continuously in t.
__device__ __forceinline__ void tanh_jac(float x, float& t, float& jac) {
  float r;
  t = tanh_r(x, r);
  jac = 4.0f * r * (1.0f - r);
}

__device__ __forceinline__ float lerp_ref(float v0, float v1, float f) {
  // v_left (1-f) + v_right f  (lut.py:115), exact at f = 0 and f = 1
  return fmaf(v1, f, v0 * (1.0f - f));
}

// Grid node -1 + i*step (lut.py:82-84) in float32: one FMA with the
// float32 step 2/(N-1) (within ~1 ulp of the correctly rounded node; the
// recomputed table entries then match the float64 table to ~k^2 ulp), the
// last node forced to 1.0 like the reference.
__device__ __forceinline__ float grid_node_f(int i, int n, float step) {
  return i >= n - 1 ? 1.0f : fmaf(static_cast<float>(i), step, -1.0f);
}

// v[0..P] = B_0..B_P at x.
template <int KIND, int P>
__device__ __forceinline__ void basis_f32(float x, float (&v)[P + 1]) {
  v[0] = 1.0f;
  if constexpr (P >= 1) {
    if constexpr (KIND == kFourier) {
      static_assert(P % 2 == 0, "Fourier features come in cos/sin pairs");
      float s1, c1;
      sincospif(x, &s1, &c1);  // cos(pi x), sin(pi x)
      v[1] = c1;
      v[2] = s1;
#pragma unroll
      for (int k = 1; k < P / 2; ++k) {
        // cos((k+1)t) = cos t cos kt - sin t sin kt; sin((k+1)t) = sin t cos kt + cos t sin kt
        v[2 * k + 1] = fmaf(c1, v[2 * k - 1], -s1 * v[2 * k]);
        v[2 * k + 2] = fmaf(s1, v[2 * k - 1], c1 * v[2 * k]);
      }
    } else if constexpr (KIND == kChebTrig) {
      const float th = acosf(fminf(fmaxf(x, -1.0f), 1.0f));
#pragma unroll
      for (int k = 1; k <= P; ++k) v[k] = cosf(static_cast<float>(k) * th);
    } else {
      const float two_x = 2.0f * x;
      v[1] = KIND == kHermite ? two_x : x;
#pragma unroll
      for (int k = 1; k < P; ++k) {
        if constexpr (KIND == kCheb) {
          v[k + 1] = fmaf(two_x, v[k], -v[k - 1]);  // T_{k+1} = 2x T_k - T_{k-1}
        } else if constexpr (KIND == kLegendre) {
          // (k+1) P_{k+1} = (2k+1) x P_k - k P_{k-1}
          const float num = fmaf(static_cast<float>(2 * k + 1) * x, v[k], -static_cast<float>(k) * v[k - 1]);
          v[k + 1] = num * (1.0f / static_cast<float>(k + 1));
        } else {
          v[k + 1] = fmaf(two_x, v[k], -static_cast<float>(2 * k) * v[k - 1]);  // H_{k+1} = 2x H_k - 2k H_{k-1}
        }
      }
    }
  }
}

// dv[0..P] = dB_k/dx at x (dv[0] = 0).  Needs the values for Legendre,
// Hermite and Fourier; they are recomputed here (registers only).
template <int KIND, int P>
__device__ __forceinline__ void deriv_f32(float x, float (&dv)[P + 1]) {
  dv[0] = 0.0f;
  if constexpr (P >= 1) {
    if constexpr (KIND == kCheb || KIND == kChebTrig) {
      // T_n' = n U_{n-1}; U_0 = 1, U_1 = 2x, U_{k+1} = 2x U_k - U_{k-1}
      const float two_x = 2.0f * x;
      float up = 1.0f, uc = two_x;
      dv[1] = 1.0f;
      if constexpr (P >= 2) dv[2] = 2.0f * uc;
#pragma unroll
      for (int n = 3; n <= P; ++n) {
        const float un = fmaf(two_x, uc, -up);
        up = uc;
        uc = un;
        dv[n] = static_cast<float>(n) * uc;
      }
    } else {
      float v[P + 1];
      basis_f32<KIND, P>(x, v);
      if constexpr (KIND == kLegendre) {
        // P'_{k+1} = P'_{k-1} + (2k+1) P_k
        dv[1] = 1.0f;
#pragma unroll
        for (int k = 1; k < P; ++k) dv[k + 1] = fmaf(static_cast<float>(2 * k + 1), v[k], dv[k - 1]);
      } else if constexpr (KIND == kHermite) {
#pragma unroll
        for (int n = 1; n <= P; ++n) dv[n] = static_cast<float>(2 * n) * v[n - 1];  // H_n' = 2n H_{n-1}
      } else {
        constexpr float kPi = 3.14159265358979323846f;
#pragma unroll
        for (int k = 1; k <= P / 2; ++k) {
          const float kpi = static_cast<float>(k) * kPi;
          dv[2 * k - 1] = -kpi * v[2 * k];  // d/dx cos(k pi x)
          dv[2 * k] = kpi * v[2 * k - 1];   // d/dx sin(k pi x)
        }
      }
    }
  }
}

// --- runtime-degree basis (generic paths) -----------------------------------
// Streams B_1, B_2, ... at one point for a runtime kind (same recurrences as
// basis_f32 in ck_basis.cuh).
struct Rec {
  int kind, k;
  float x, prev, cur, c1, s1, cm, sm, th;
  __device__ __forceinline__ void init(int kind_, float x_) {
    kind = kind_;
    x = x_;
    k = 0;
    prev = 0.0f;
    cur = 1.0f;
    if (kind == kFourier) {
      sincospif(x, &s1, &c1);
      cm = 1.0f;
      sm = 0.0f;
    } else if (kind == kChebTrig) {
      th = acosf(fminf(fmaxf(x, -1.0f), 1.0f));
    }
  }
  // B_{k+1}
  __device__ __forceinline__ float next() {
    float v;
    if (kind == kFourier) {
      // features 2m-1 = cos(m pi x), 2m = sin(m pi x)
      if ((k & 1) == 0) {
        const float c = fmaf(c1, cm, -s1 * sm), s = fmaf(s1, cm, c1 * sm);
        cm = c;
        sm = s;
        v = cm;
      } else {
        v = sm;
      }
    } else if (kind == kChebTrig) {
      v = cosf(static_cast<float>(k + 1) * th);
    } else if (k == 0) {
      v = kind == kHermite ? 2.0f * x : x;
    } else if (kind == kCheb) {
      v = fmaf(2.0f * x, cur, -prev);
    } else if (kind == kLegendre) {
      v = fmaf(static_cast<float>(2 * k + 1) * x, cur, -static_cast<float>(k) * prev) *
          (1.0f / static_cast<float>(k + 1));
    } else {
      v = fmaf(2.0f * x, cur, -static_cast<float>(2 * k) * prev);
    }
    prev = cur;
    cur = v;
    ++k;
    return v;
  }
};

// v[0..P], dv[0..P] at x for a runtime kind / P (P < kMaxK).
__device__ inline void basis_deriv_rt(int kind, int P, float x, float* v, float* dv) {
  Rec r;
  r.init(kind, x);
  v[0] = 1.0f;
  for (int k = 1; k <= P; ++k) v[k] = r.next();
  if (dv == nullptr) return;
  dv[0] = 0.0f;
  if (kind == kCheb || kind == kChebTrig) {
    float up = 1.0f, uc = 2.0f * x;
    if (P >= 1) dv[1] = 1.0f;
    if (P >= 2) dv[2] = 2.0f * uc;
    for (int n = 3; n <= P; ++n) {
      const float un = fmaf(2.0f * x, uc, -up);
      up = uc;
      uc = un;
      dv[n] = static_cast<float>(n) * uc;
    }
  } else if (kind == kLegendre) {
    if (P >= 1) dv[1] = 1.0f;
    for (int k = 1; k < P; ++k) dv[k + 1] = fmaf(static_cast<float>(2 * k + 1), v[k], dv[k - 1]);
  } else if (kind == kHermite) {
    for (int n = 1; n <= P; ++n) dv[n] = static_cast<float>(2 * n) * v[n - 1];
  } else {
    constexpr float kPi = 3.14159265358979323846f;
    for (int m = 1; 2 * m <= P; ++m) {
      dv[2 * m - 1] = -static_cast<float>(m) * kPi * v[2 * m];
      dv[2 * m] = static_cast<float>(m) * kPi * v[2 * m - 1];
    }
  }
}

// --- basis planes at one element (expansion kernels, generated GEMM operand) --
// Values of features k = 1..D at one element.  kLutNodes: the two table
// entries bracketing the cell are recomputed at the (float32-rounded) grid
// nodes by the family's recurrence -- the same table entries to ~k^2 ulp,
// with no memory traffic -- then interpolated v0 (1-f) + v1 f.  kExact:
// the basis at t = tanh(x) itself.
enum PlaneSource : int { kSrcNodes = 0, kSrcExact = 1 };

template <int kSrc, int KIND, int D>
__device__ __forceinline__ void elem_planes(float xv, int n, float (&out)[D]) {
  if constexpr (kSrc == kSrcExact) {
    float v[D + 1];
    basis_f32<KIND, D>(tanhf(xv), v);
#pragma unroll
    for (int k = 1; k <= D; ++k) out[k - 1] = v[k];
  } else {
    int idx;
    float f;
    cell_f32(xv, n, idx, f);
    float v0[D + 1], v1[D + 1];
    basis_f32<KIND, D>(grid_node_f(idx, n, 2.0f / static_cast<float>(n - 1)), v0);
    basis_f32<KIND, D>(grid_node_f(idx + 1, n, 2.0f / static_cast<float>(n - 1)), v1);
#pragma unroll
    for (int k = 1; k <= D; ++k) out[k - 1] = lerp_ref(v0[k], v1[k], f);
  }
}

// Chord slopes S_k = (B_k(a) - B_k(b)) / (a - b), k = 1..D, of the family's
// features over the cell [b, a] -- the LUT slopes (values[:,1:] -
// values[:,:-1]) / step (lut.py:86, 93) -- by the divided-difference form of
// the three-term recurrence: with B_{k+1} = (A_k x + E_k) B_k - C_k B_{k-1},
//   S_{k+1} = (A_k a + E_k) S_k + A_k B_k(b) - C_k S_{k-1},
// which has no cancellation (unlike differencing two recomputed values, whose
// k^2-ulp errors divided by the step would reach 1e-3).  Endpoint rounding of
// the float32 nodes moves a chord by B''/2 * 1 ulp: <= 1e-6 relative for d <= 8.
template <int KIND, int D>
__device__ __forceinline__ void chord_slopes(float b, float a, float (&s)[D]) {
  float pv = 1.0f, cv = KIND == kHermite ? 2.0f * b : b;  // B_0(b), B_1(b)
  float sp = 0.0f, sc = KIND == kHermite ? 2.0f : 1.0f;   // S_0, S_1
  s[0] = sc;
#pragma unroll
  for (int k = 1; k < D; ++k) {
    float sn, vn;
    if constexpr (KIND == kCheb) {
      sn = fmaf(2.0f * a, sc, fmaf(2.0f, cv, -sp));
      vn = fmaf(2.0f * b, cv, -pv);
    } else if constexpr (KIND == kLegendre) {
      const float c2 = static_cast<float>(2 * k + 1), ck = static_cast<float>(k);
      const float inv = 1.0f / static_cast<float>(k + 1);
      sn = fmaf(c2, fmaf(a, sc, cv), -ck * sp) * inv;
      vn = fmaf(c2 * b, cv, -ck * pv) * inv;  // as basis_f32
    } else {
      const float c2k = static_cast<float>(2 * k);
      sn = fmaf(2.0f, fmaf(a, sc, cv), -c2k * sp);
      vn = fmaf(2.0f * b, cv, -c2k * pv);
    }
    s[k] = sn;
    sp = sc;
    sc = sn;
    pv = cv;
    cv = vn;
  }
}

}  // namespace ck
