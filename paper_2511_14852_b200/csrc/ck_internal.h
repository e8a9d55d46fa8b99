// Internal (non-exported) interfaces shared by the ChebyKAN .cu files.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/chebykan.h"

struct ck_lut {
  int kind = 0;        // basis family (ck_basis_kind; tags of lut.py:35-40)
  int exact = 0;       // 1: exact evaluation handle (BasisPath.EXACT_RECURRENCE), no tables
  int degree = 0;
  int n_feat = 0;      // K = feature_count(kind, degree) (basis.py:24-34)
  int lut_size = 0;    // N (0 for exact handles)
  double step = 0.0;   // 2 / (N - 1)
  int device = 0;
  double* values64 = nullptr;  // [K][N]   float64 build-precision table (validation)
  float* values_pm = nullptr;  // [N][K]   float32, position-major (gather rows idx, idx+1)
  float* slopes_pm = nullptr;  // [N-1][K] float32 cell slopes, position-major
  // [N][dxrow_stride(K)] input-gradient rows: [0..K-2] = the cell's float32
  // slopes of features 1..K-1, [K-1] = b_i, the smallest float32 x whose
  // reference (float64) cell is >= i (-inf for i = 0, +inf sentinel for
  // i = N-1), [K] = b_{i+1}, zero padding to a 16-byte multiple.  Kernels
  // gather the slopes with 16-byte loads and, only when the float32
  // position lies near a cell edge, the two boundaries -- the exact
  // reference cell with float32 compares only.
  float* dxrows = nullptr;
};

namespace ck {

// floats per input-gradient row of a K-feature table (see ck_lut::dxrows)
__host__ __device__ constexpr int dxrow_stride(int K) { return (K + 1 + 3) & ~3; }

// Kernel classes for the launch counter / device timers (ck_timing_*).
enum KClass : int {
  kKGemmFwd = 0,
  kKGemmDx = 1,
  kKGemmDc = 2,
  kKExpand = 3,
  kKExpandT = 4,
  kKDxCombine = 5,
  kKSplit = 6,
  kKReduce = 7,
  kKLut = 8,
  kKOptim = 9,
  kKSkinny = 10,
  kKNumClasses = 11,
};

// RAII: counts one launch of class `cls` and, when timing is enabled,
// brackets it with CUDA events on `stream`.
class LaunchScope {
 public:
  LaunchScope(int cls, cudaStream_t stream);
  ~LaunchScope();

 private:
  int cls_;
  cudaStream_t stream_;
  void* ev_ = nullptr;
};

// Rows processed per internal chunk by ck_forward / ck_backward (bounds the
// workspace; chunks are processed in ascending order on one stream, so the
// accumulated dC is bit-reproducible).  Default 32768; ck_set_chunk_rows (or
// CK_CHUNK_ROWS at load) changes it process-wide, e.g. so tests run the
// multi-chunk dC accumulation of a wide layer on a small batch.
constexpr int64_t kChunkRowsDefault = 32768;
int64_t chunk_rows();

// --- LUT view passed by value to kernels ----------------------------------
struct LutView {
  const float* values_pm;
  const float* slopes_pm;
  const float* dxrows;
  int K;
  int N;
  double step;
  int kind;   // ck_basis_kind
  int exact;  // 1: evaluate the basis at t (no table)
};
inline LutView view(const ck_lut* l) {
  return LutView{l->values_pm, l->slopes_pm, l->dxrows, l->n_feat, l->lut_size, l->step, l->kind, l->exact};
}

// --- expansion (ck_expand.cu) ---------------------------------------------
// phi[r][c][k] (f32) and optional slopes[r][c][k] for every k.
int launch_expand_f32(const float* x, int64_t rows, int cols, const ck_lut* lut, float* phi,
                      float* slopes, cudaStream_t s);
// vals[e][k] (and slopes) of the basis at normalized points t[e] (no tanh)
int launch_basis_eval(const float* t, int64_t n, const ck_lut* lut, float* vals, float* slopes, cudaStream_t s);
// Split planes hi/lo [nk][rows][ld] for k = k0..K-1 (bf16, ld % 8 == 0).
int launch_expand_planes(const float* x, int64_t rows, int cols, const ck_lut* lut, int k0,
                         __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ld, int64_t plane_stride,
                         cudaStream_t s);
// dx[r][c] = J * sum_{k>=1} slope_k(cell(tanh x)) * g[k-1][r][c]
int launch_dx_combine(const float* g, int64_t g_plane_stride, const float* x, int64_t rows, int cols,
                      const ck_lut* lut, int jacobian, float* dx, cudaStream_t s);

// --- elementwise / reductions (ck_split.cu) -------------------------------
// hi/lo [z][rows][ld] <- in [z][rows][cols] (input pitch = cols)
int launch_split_rows(const float* in, int64_t nz, int64_t rows, int64_t cols, int64_t in_z_stride,
                      __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ld, int64_t out_z_stride,
                      cudaStream_t s);
// hi/lo [rows][ld] <- in [rows][cols] plus part[s][c] = float64 sum of row
// block s (rows split into `slots` equal blocks) of column c, one pass
int launch_split_rows_colsum(const float* in, int64_t rows, int64_t cols, __nv_bfloat16* hi, __nv_bfloat16* lo,
                             int64_t ld, double* part, int slots, cudaStream_t s);
// hi/lo [z][cols][ld] <- transpose of in [z][rows][cols]
int launch_split_transpose(const float* in, int64_t nz, int64_t rows, int64_t cols, int64_t in_z_stride,
                           __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ld, int64_t out_z_stride,
                           cudaStream_t s);
// Stacked input-gradient operand from DOJ fp32 [K][O][I]: row
// (i / n_i) * d * n_i + (k-1) * n_i + i % n_i holds C[k][:, i] (k = 1..d,
// d = K-1) as bf16 hi/lo with pitch ld; rows of padded inputs are zero.
int launch_split_transpose_stacked(const float* c_doj, int64_t K, int64_t O, int64_t I, int n_i, __nv_bfloat16* hi,
                                   __nv_bfloat16* lo, int64_t ld, cudaStream_t s);
// out[r] = sum_c in[r][c]  (float64 accumulation in a fixed order)
int launch_row_sum(const float* in, int64_t rows, int64_t cols, float* out, cudaStream_t s, void* hdr = nullptr,
                   const struct PrepHeader* h = nullptr);
// part[slot][c] = sum over rows of in[rows][cols]  (float64, fixed order)
int launch_col_partial(const float* in, int64_t rows, int64_t cols, double* part, int slots,
                       cudaStream_t s);
// out[c] = sum_{s<slots} part[s][c] -> float
// out[c] = sum_s part[s][c] in fixed order; bcast (nullable): also
// bcast[c][0..bcast_cols) = out[c]
int launch_col_finish(const double* part, int slots, int64_t cols, float* out, cudaStream_t s,
                      float* bcast = nullptr, int64_t bcast_cols = 0);
// A col_finish (above) folded into another reduction launch.
struct ColFinishJob {
  const double* part;
  int slots;
  int64_t cols;
  float* out;
  float* bcast;        // nullable
  int64_t bcast_cols;
};
// out[n] = (accumulate ? out[n] : 0) + sum_{s<S} partials[s * stride + n];
// fin (nullable): a col_finish job run by extra blocks of the same launch
int launch_merge(const float* partials, int S, int64_t stride, int64_t n, float* out, int accumulate,
                 cudaStream_t s, const ColFinishJob* fin = nullptr);
// out[r][c] = a[c] + b[c] (either nullable)
int launch_fill_rows(float* out, int64_t rows, int64_t cols, const float* a, const float* b,
                     cudaStream_t s);
// out[r][c] += a[c] + b[c] (either nullable)
int launch_add_rows(float* out, int64_t rows, int64_t cols, const float* a, const float* b, cudaStream_t s);

// Header at the start of an opaque coefficient-prep buffer (written by
// ck_coeff_prepare on the device; read back by ck_coeff_prep_check).
struct PrepHeader {
  uint32_t magic;     // kPrepMagic
  uint32_t version;   // layout version
  int32_t d_in, d_out, n_feat, flags;  // flags: 1 = skinny (fp32 copy), 2 = generated-forward copy
  uint64_t bytes;     // ck_coeff_prep_bytes(d_in, d_out, n_feat)
};
constexpr uint32_t kPrepMagic = 0x52504b43u;  // "CKPR"
constexpr uint32_t kPrepVersion = 3;  // 3: stacked dX tile width chosen per d_in
// The coefficient prep of a stacked-dX layer in one launch: DOJ hi/lo
// [K][O][ldI], the stacked operand (see launch_split_transpose_stacked),
// c0sum[o] = sum_i C[0][o][i] (float64, fixed order) and the header.
int launch_prep_fused(const float* c_doj, int64_t K, int64_t O, int64_t I, int n_i, __nv_bfloat16* doj_hi,
                      __nv_bfloat16* doj_lo, int64_t ldI, __nv_bfloat16* dxb_hi, __nv_bfloat16* dxb_lo, int64_t ldO,
                      float* c0sum, void* hdr, const PrepHeader& h, cudaStream_t s);
// out[0..n) = in[0..n) and the prep header, one launch
int launch_copy_with_header(const float* in, float* out, int64_t n, void* hdr, const PrepHeader& h, cudaStream_t s);

// --- skinny-output layers (ck_skinny.cu) ----------------------------------
// d_out <= 8 with n_feat * round_up_pow2(d_out) <= 32: CUDA-core kernels on
// fp32 DOJ coefficients (no basis planes, no tensor-core tiles).
constexpr int kSkinnyMaxO = 8;
constexpr int kSkinnyMaxKO = 32;
constexpr int kSkinnyMaxSlots = 128;
bool skinny_layer(int d_in, int d_out, int n_feat);
// row blocks of the skinny backward's partial reduction for this shape
int skinny_slots(int64_t rows, int d_in, int d_out, int n_feat);
int launch_skinny_forward(const float* x, int64_t rows, int I, int O, const float* c, const float* bias,
                          const ck_lut* lut, float* y, cudaStream_t s);
// dx (nullable) written directly; part_c [slots][K][O][I] float and part_b
// [slots][O] float64 partials for the ordered slot merges
int launch_skinny_backward(const float* x, const float* dy, int64_t rows, int I, int O, const float* c,
                           const ck_lut* lut, int jacobian, float* dx, float* part_c, double* part_b, int slots,
                           cudaStream_t s);

// --- tcgen05 split-precision GEMM (ck_gemm.cu) ----------------------------
// out[z][m][n] (+)= sum_{s<S} sum_r A[aseg][m][r] * B[bseg][n][r]
//   aseg = a_seg0 + s + a_seg_z * z,  bseg = b_seg0 + s + b_seg_z * z
// A and B are bf16 hi/lo pairs, K-major, row pitch lda/ldb (multiple of 8),
// segment stride a_seg_stride/b_seg_stride elements.  BF16x3: the MMA sums
// hi*hi + hi*lo + lo*hi in fp32 TMEM accumulators.
struct GemmOperand {
  const __nv_bfloat16* hi;
  const __nv_bfloat16* lo;
  int64_t rows;        // M (for A) or N (for B)
  int64_t ld;          // pitch in elements between consecutive rows (K-major) or K-rows (MN-major)
  int64_t seg_stride;  // elements between segments
  int64_t segs;        // number of segments addressable
  int mn_major = 0;    // 1: stored [K][MN] (M/N contiguous), e.g. dy [B][O] as the dC A operand
};
// Fused input-gradient epilogue (kernels.py:430-444): the GEMM's N tile
// stacks d features x n_i inputs; the epilogue folds the d accumulators
// with the cell slopes and the tanh Jacobian straight into dx.
struct DxEpilogue {
  const float* x;      // [M][cols] chunk of the layer input
  float* dx;           // [M][cols]
  LutView lut;
  int jacobian;
  int64_t cols;        // I
  int n_i;             // inputs per N tile; the MMA N is d * n_i
};
// n_i for degree d and I inputs, or 0 when the stacked layout does not fit one MMA.
int dx_tile_inputs(int d, int64_t I);

struct GemmProblem {
  GemmOperand a, b;
  int64_t R;          // reduction extent per segment
  int S;              // segments summed into each output
  int a_seg0, a_seg_z, b_seg0, b_seg_z;
  int nz;             // number of outputs along z
  float* out;
  int64_t ldo, out_z_stride;
  const float* bias0;  // nullable, added per column n
  const float* bias1;  // nullable
  int accumulate;      // out += result
  float* split_ws;     // workspace for split-R partials (nullable -> no split)
  int64_t split_ws_elems;
  int kclass = kKGemmFwd;  // timing / counting class
  int out_trans = 0;       // 1: store out[z][n][m] (row pitch ldo) -- the transposed orientation
  const DxEpilogue* dx = nullptr;  // non-null: stacked-B fused dX path
  const ColFinishJob* fin = nullptr;  // run after the GEMM (in its merge launch when it splits)
};
int gemm_bf16x3(const GemmProblem& p, cudaStream_t s);

// --- forward with the basis generated in shared memory (ck_gemm_gen.cu) -----
// 64-wide reduction chunks of 64/d whole inputs (0: degree not supported)
int gen_chunks(int I, int d);
// layers whose prepared coefficients carry the generated operand's copy
bool gen_layer(int I, int O, int K);
bool gen_supported(const LutView& v);
// coefficients [O][gen_chunks*64] bf16 hi/lo in the generated operand's order
int launch_gen_coeff(const float* coeff_doj, int I, int O, int d, __nv_bfloat16* hi, __nv_bfloat16* lo,
                     cudaStream_t s);
// y[M][O] = Φ(x) C^T + bias0 + bias1 (per column), Φ never materialised
int gemm_gen_forward(const float* x, int64_t M, int I, int O, const LutView& v, const __nv_bfloat16* c_hi,
                     const __nv_bfloat16* c_lo, const float* bias0, const float* bias1, float* y, cudaStream_t s);
// Output cells a store GEMM computes, tile padding included (orientation choice).
int64_t gemm_store_padded(int64_t M, int64_t N, bool mn_major);
// Workspace (floats) the split-R path may want for this problem shape;
// kchunks = 64-wide K chunks of the whole reduction (segments x ceil(R/64)).
int64_t gemm_split_ws_elems(int64_t M, int64_t N, int nz, int64_t kchunks);

}  // namespace ck
