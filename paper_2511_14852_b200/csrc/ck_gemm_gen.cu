// Forward with the basis generated in shared memory: host side (selection
// rule, coefficient reorder, launch).  The kernel is in ck_gemm_gen.cuh.
#include "ck_gemm_gen.cuh"

namespace ck {
namespace {

// Coefficients in the generated operand's order: out[o][j*64 + g*d + k-1] =
// C[k][o][j*G + g] (k = 1..d), zero for padding positions and inputs >= I.
__global__ void gen_coeff_kernel(const float* __restrict__ c, int O, int I, int d, int G, int64_t R,
                                 __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  pdl_wait();
  const int64_t n = static_cast<int64_t>(O) * R;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = e / R;
    const int q = static_cast<int>(e - o * R);
    const int j = q >> 6, pos = q & 63;
    const int gi = pos / d, k = pos - gi * d + 1;
    const int i = j * G + gi;
    float v = 0.0f;
    if (gi < G && i < I) v = c[(static_cast<int64_t>(k) * O + o) * I + i];
    __nv_bfloat16 h, l;
    split_bf16(v, h, l);
    hi[e] = h;
    lo[e] = l;
  }
}

}  // namespace

// Widest output the generated forward takes (CK_GEN_MAX_O; 0 disables it):
// prep and forward agree through this one function.
int gen_max_o() {
  static int v = [] {
    const char* e = getenv("CK_GEN_MAX_O");
    return e ? atoi(e) : 256;
  }();
  return v;
}

// Measured (tools/gen_experiment.py, batch 16384): generation costs ~13
// instructions per basis value on the SM that also feeds the tensor core, so
// it hides behind the MMAs once a stage holds enough features per input
// (d >= 4) and the reduction is long enough to amortise the fill (d*I >=
// 1536); below that the materialised planes are as fast or faster.
// CK_GEN=all drops the degree / length rule (tests).
// longest reduction (terms) the generated forward takes (CK_GEN_MAX_CHAIN
// overrides it for timing experiments; results past it are less accurate)
int gen_max_chain() {
  static int v = [] {
    const char* e = getenv("CK_GEN_MAX_CHAIN");
    return e ? atoi(e) : 8192;
  }();
  return v;
}

bool gen_layer(int I, int O, int K) {
  static const bool all = [] {
    const char* e = getenv("CK_GEN");
    return e && std::string(e) == "all";
  }();
  const int d = K - 1;
  if (skinny_layer(I, O, K) || O > gen_max_o() || gen_chunks(I, d) == 0) return false;
  // the generated forward accumulates the whole reduction in one TMEM
  // buffer (no segment folding: its epilogue warps have no registers to
  // spare), so it is limited to reductions whose biased tensor-core
  // accumulation stays <= ~3e-5 normwise (8192 terms; ck_gemm_impl.cuh,
  // kSegIters); longer ones take expand + the segmented store GEMM
  if (gen_chunks(I, d) * 64 > gen_max_chain()) return false;
  return all || (d >= 4 && static_cast<int64_t>(d) * I >= 1536);
}

int gen_chunks(int I, int d) { return d >= 1 && d <= kGenMaxD ? static_cast<int>(ceil_div(I, 64 / d)) : 0; }

bool gen_supported(const LutView& v) {
  const int d = v.K - 1;
  if (d < 1 || d > kGenMaxD) return false;
  if (v.kind == kFourier && d % 2 != 0) return false;
  if (v.kind == kChebTrig) return v.exact != 0;
  return v.kind == kCheb || v.kind == kLegendre || v.kind == kHermite || v.kind == kFourier;
}

int launch_gen_coeff(const float* coeff_doj, int I, int O, int d, __nv_bfloat16* hi, __nv_bfloat16* lo,
                     cudaStream_t s) {
  const int64_t R = static_cast<int64_t>(gen_chunks(I, d)) * 64;
  CK_CHECK(R > 0, "gen_coeff: unsupported degree");
  const int64_t n = O * R;
  const int64_t want = ceil_div(n, 256), cap = static_cast<int64_t>(num_sms()) * 8;
  LaunchScope scope(kKSplit, s);
  CK_CUDA(launch_k(gen_coeff_kernel, static_cast<int>(want < cap ? want : cap), 256, 0, s, coeff_doj, O, I, d,
                   64 / d, R, hi, lo));
  return kOk;
}

int gemm_gen_forward(const float* x, int64_t M, int I, int O, const LutView& v, const __nv_bfloat16* c_hi,
                     const __nv_bfloat16* c_lo, const float* bias0, const float* bias1, float* y, cudaStream_t s) {
  const int d = v.K - 1;
  CK_CHECK(gen_supported(v), "gemm_gen: unsupported basis");
  CK_CHECK(M < (1ll << 31), "gemm_gen: too many rows");
  const int chunks = gen_chunks(I, d);
  const int64_t R = static_cast<int64_t>(chunks) * 64;
  const int n_tile = store_ntile(O, 256, 2, false);
  CUtensorMap tb_hi, tb_lo;
  CK_TRY(make_map(&tb_hi, c_hi, R, O, 1, R, 0, n_tile / 2, 64, 0));
  CK_TRY(make_map(&tb_lo, c_lo, R, O, 1, R, 0, n_tile / 2, 64, 0));
  KArgs k{};
  k.M = static_cast<int>(M);
  k.N = O;
  k.S = 1;
  k.n_tile = n_tile;
  k.n_mma = n_tile;
  k.b_boxes = 1;
  k.stage_tx = static_cast<uint32_t>(2 * n_tile * 128);  // B hi + lo of both CTAs
  k.x = x;
  k.gen_ldx = I;
  k.gen_I = I;
  k.lutN = v.exact ? 0 : v.N;
  k.splits = 1;
  k.r_chunks = chunks;
  k.out = y;
  k.ldo = O;
  k.bias0 = bias0;
  k.bias1 = bias1;
  k.n_tiles = static_cast<int>(ceil_div(O, n_tile));
  k.m_tiles = static_cast<int>(ceil_div(M, 256));
  k.group_m = gemm_group(k.m_tiles);
  const long long total = static_cast<long long>(k.n_tiles) * k.m_tiles;
  CK_CHECK(total < (1ll << 31), "gemm_gen: too many tiles");
  k.total_tiles = static_cast<int>(total);
  const int units_max = gemm_sms() / 2;
  const int grid = 2 * static_cast<int>(total < units_max ? total : units_max);
  LaunchScope scope(kKGemmFwd, s);
  switch (v.kind) {
    case kCheb:
    case kChebTrig:
      return launch_gen_cheb(v.exact, v.kind == kChebTrig, d, k, tb_hi, tb_lo, grid, s);
    case kLegendre:
      return launch_gen_legendre(v.exact, d, k, tb_hi, tb_lo, grid, s);
    case kHermite:
      return launch_gen_hermite(v.exact, d, k, tb_hi, tb_lo, grid, s);
    default:
      return launch_gen_fourier(v.exact, d, k, tb_hi, tb_lo, grid, s);
  }
}

}  // namespace ck
