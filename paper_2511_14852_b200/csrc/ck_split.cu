// Memory-bound helpers: bf16x3 operand splitting (with optional transpose),
// fixed-order reductions (the two-stage deterministic merges) and fills.
#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

constexpr int kThreads = 256;

int blocks_for(int64_t items, int per_sm = 8) {
  const int64_t want = ceil_div(items, kThreads);
  const int64_t cap = static_cast<int64_t>(num_sms()) * per_sm;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

// hi/lo [z][r][ld] from in [z][r][cols]; two columns per thread.
__global__ void split_rows_kernel(const float* __restrict__ in, int64_t nz, int64_t rows, int64_t cols,
                                  int64_t in_zs, uint32_t* __restrict__ hi, uint32_t* __restrict__ lo,
                                  int64_t ld, int64_t out_zs) {
  pdl_wait();
  const int64_t pairs = (cols + 1) >> 1;
  const int64_t n = nz * rows * pairs;
  for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < n;
       it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t z = it / (rows * pairs);
    const int64_t rem = it - z * rows * pairs;
    const int64_t r = rem / pairs;
    const int64_t c = (rem - r * pairs) * 2;
    const float* src = in + z * in_zs + r * cols + c;
    const float a = src[0];
    const float b = c + 1 < cols ? src[1] : 0.0f;
    uint32_t h2, l2;
    split_pack2(a, b, h2, l2);
    const int64_t o = (z * out_zs + r * ld + c) >> 1;
    hi[o] = h2;
    lo[o] = l2;
  }
}

// dy pass of the backward: hi/lo [r][ld] bf16 split of in [rows][cols] and,
// in the same read, float64 column sums per row block (the bias gradient's
// first stage).  grid = (slots, ceil(cols / 64)); block (s, cb) covers rows
// [s*rb, min((s+1)*rb, rows)) and columns [64 cb, 64 cb + 64): warp w takes
// rows w, w+8, ...; lane l the column pair 64 cb + 2 l.  The 8 warp partials
// are folded in warp order, so part[s][c] is deterministic.
__global__ void __launch_bounds__(256, 3) split_rows_colsum_kernel(const float* __restrict__ in, int64_t rows,
                                                                int64_t cols, int64_t rb, uint32_t* __restrict__ hi,
                                                                uint32_t* __restrict__ lo, int64_t ld,
                                                                double* __restrict__ part) {
  pdl_wait();
  __shared__ double red[8][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.y) * 64 + 2 * lane;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rb;
  const int64_t r1 = r0 + rb < rows ? r0 + rb : rows;
  double s0 = 0.0, s1 = 0.0;
  if (c < cols) {
    const bool two = c + 1 < cols;
    const bool vec = two && ((cols & 1) == 0);
    // 8 rows per iteration (independent loads in flight: 4 left the HBM
    // pipe a third full, ncu 27 % DRAM); sums in row order
    constexpr int RU = 8;
    for (int64_t rr = r0 + w; rr < r1; rr += 8 * RU) {
      float a[RU], b[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int64_t r = rr + 8 * u;
        a[u] = b[u] = 0.0f;
        if (r < r1) {
          const float* src = in + r * cols + c;
          if (vec) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(src));
            a[u] = v.x;
            b[u] = v.y;
          } else {
            a[u] = __ldg(src);
            b[u] = two ? __ldg(src + 1) : 0.0f;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int64_t r = rr + 8 * u;
        if (r >= r1) break;
        s0 += static_cast<double>(a[u]);
        s1 += static_cast<double>(b[u]);
        uint32_t h2, l2;
        split_pack2(a[u], b[u], h2, l2);
        const int64_t o = (r * ld + c) >> 1;
        hi[o] = h2;
        lo[o] = l2;
      }
    }
  }
  red[w][2 * lane] = s0;
  red[w][2 * lane + 1] = s1;
  __syncthreads();
  if (threadIdx.x < 64) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += red[j][threadIdx.x];
    const int64_t cc = static_cast<int64_t>(blockIdx.y) * 64 + threadIdx.x;
    if (cc < cols) part[static_cast<int64_t>(blockIdx.x) * cols + cc] = acc;
  }
}

// hi/lo [z][c][ld] = transpose of in [z][r][c] via 32x32 smem tiles.
__global__ void split_transpose_kernel(const float* __restrict__ in, int64_t nz, int64_t rows, int64_t cols,
                                       int64_t in_zs, __nv_bfloat16* __restrict__ hi,
                                       __nv_bfloat16* __restrict__ lo, int64_t ld, int64_t out_zs) {
  pdl_wait();
  __shared__ float tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
  const int64_t rt = ceil_div(rows, 32), ct = ceil_div(cols, 32);
  for (int64_t t = blockIdx.x; t < nz * rt * ct; t += gridDim.x) {
    const int64_t z = t / (rt * ct);
    const int64_t rem = t - z * rt * ct;
    const int64_t r0 = (rem / ct) * 32, c0 = (rem % ct) * 32;
    for (int j = ty; j < 32; j += 8) {
      const int64_t r = r0 + j, c = c0 + tx;
      tile[j][tx] = (r < rows && c < cols) ? in[z * in_zs + r * cols + c] : 0.0f;
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
      const int64_t c = c0 + j, r = r0 + tx;
      if (c < cols && r < ld) {
        __nv_bfloat16 h, l;
        split_bf16(tile[tx][j], h, l);
        const int64_t o = z * out_zs + c * ld + r;
        hi[o] = h;
        lo[o] = l;
      }
    }
    __syncthreads();
  }
}

// Stacked transpose: input tile 32 (o) x 32 (i) of plane k (>= 1); output
// row (i / n_i) * d * n_i + (k-1) * n_i + i % n_i, column o.
__global__ void split_transpose_stacked_kernel(const float* __restrict__ c, int64_t K, int64_t O, int64_t I, int n_i,
                                               __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo,
                                               int64_t ld) {
  pdl_wait();
  __shared__ float tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t d = K - 1;
  const int64_t i_pad = ceil_div(I, n_i) * n_i;
  const int64_t ot = ceil_div(O, 32), it_ = ceil_div(i_pad, 32);
  for (int64_t t = blockIdx.x; t < d * ot * it_; t += gridDim.x) {
    const int64_t k = 1 + t / (ot * it_);
    const int64_t rem = t % (ot * it_);
    const int64_t o0 = (rem / it_) * 32, i0 = (rem % it_) * 32;
    const float* src = c + k * O * I;
    for (int j = ty; j < 32; j += 8) {
      const int64_t o = o0 + j, i = i0 + tx;
      tile[j][tx] = (o < O && i < I) ? src[o * I + i] : 0.0f;
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
      const int64_t i = i0 + j, o = o0 + tx;
      if (i < i_pad && o < ld) {
        __nv_bfloat16 h, l;
        split_bf16(tile[tx][j], h, l);
        const int64_t row = (i / n_i) * d * n_i + (k - 1) * n_i + i % n_i;
        hi[row * ld + o] = h;
        lo[row * ld + o] = l;
      }
    }
    __syncthreads();
  }
}

// one warp per row, float64 lane partials combined by a fixed shuffle tree
__global__ void row_sum_kernel(const float* __restrict__ in, int64_t rows, int64_t cols, float* __restrict__ out,
                               PrepHeader* hdr, PrepHeader h) {
  pdl_wait();
  if (hdr != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *hdr = h;  // (coefficient prep: same launch)
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    double acc = 0.0;
    for (int64_t c = lane; c < cols; c += 32) acc += static_cast<double>(in[r * cols + c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = static_cast<float>(acc);
  }
}

// The whole coefficient prep of a stacked-dX layer in one launch (it was
// three: DOJ split, stacked transpose, row sums): blocks [0, sum_blocks)
// compute c0sum[o] = sum_i C[0][o][i] (one warp per row, float64 lane
// partials, fixed shuffle tree -- as row_sum_kernel); the other blocks take
// 64 (o) x 64 (i) tiles of every plane k: lanes own input pairs (8-byte
// loads, bf16x2 stores of the DOJ hi/lo copy, unit stride in i) and, for
// k >= 1, after a shared-memory transpose, output pairs of the stacked
// input-gradient operand (unit stride in o; padded inputs zeroed).  The
// stacked row of an input is computed once per warp (the index division was
// most of the kernel's instructions when every element did it).
__global__ void __launch_bounds__(256) prep_fused_kernel(const float* __restrict__ c, int64_t K, int64_t O, int64_t I,
                                                         int n_i, int sum_blocks, __nv_bfloat16* __restrict__ doj_hi,
                                                         __nv_bfloat16* __restrict__ doj_lo, int64_t ldI,
                                                         __nv_bfloat16* __restrict__ dxb_hi,
                                                         __nv_bfloat16* __restrict__ dxb_lo, int64_t ldO,
                                                         float* __restrict__ c0sum, PrepHeader* hdr, PrepHeader h) {
  pdl_wait();
  __shared__ float tile[64][65];
  if (blockIdx.x == 0 && threadIdx.x == 0) *hdr = h;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t d = K - 1;
  const int64_t i_pad = ceil_div(I, n_i) * n_i;
  const int64_t ot = ceil_div(O, 64), it_ = ceil_div(i_pad, 64);
  const int64_t tiles = K * ot * it_;
  const bool pairs = (I % 2 == 0) && (reinterpret_cast<uintptr_t>(c) & 7) == 0;
  uint32_t* dh = reinterpret_cast<uint32_t*>(doj_hi);
  uint32_t* dl = reinterpret_cast<uint32_t*>(doj_lo);
  uint32_t* xh = reinterpret_cast<uint32_t*>(dxb_hi);
  uint32_t* xl = reinterpret_cast<uint32_t*>(dxb_lo);
  for (int64_t t = blockIdx.x; t < sum_blocks + tiles; t += gridDim.x) {
    if (t < sum_blocks) {
      const int64_t o = t * 8 + w;
      if (o < O) {
        // 8 loads in flight per lane, added in index order
        double acc = 0.0;
        int64_t i = lane;
        for (; i + 7 * 32 < I; i += 8 * 32) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldg(c + o * I + i + 32 * u);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc += static_cast<double>(v[u]);
        }
        for (; i < I; i += 32) acc += static_cast<double>(c[o * I + i]);
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
        if (lane == 0) c0sum[o] = static_cast<float>(acc);
      }
      continue;
    }
    const int64_t u = t - sum_blocks;
    const int64_t k = u / (ot * it_);
    const int64_t rem = u - k * ot * it_;
    const int64_t o0 = (rem / it_) * 64, i0 = (rem % it_) * 64;
    const float* src = c + k * O * I;
    const int64_t i = i0 + 2 * lane;
    // all 8 row loads in flight before any store (the tile loop was a chain
    // of L2 round trips: ~35 % of HBM at 512^2)
    float av[8], bv[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int64_t o = o0 + w + 8 * r;
      av[r] = bv[r] = 0.0f;
      if (o < O) {
        const float* p = src + o * I + i;
        if (pairs && i < I) {
          const float2 v = __ldg(reinterpret_cast<const float2*>(p));
          av[r] = v.x;
          bv[r] = v.y;
        } else {
          av[r] = i < I ? __ldg(p) : 0.0f;
          bv[r] = i + 1 < I ? __ldg(p + 1) : 0.0f;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int ol = w + 8 * r;
      const int64_t o = o0 + ol;
      if (o < O && i < I) {  // (i + 1 = I odd: the pad element of the row gets 0)
        uint32_t h2, l2;
        split_pack2(av[r], bv[r], h2, l2);
        const int64_t q = ((k * O + o) * ldI + i) >> 1;
        dh[q] = h2;
        dl[q] = l2;
      }
      tile[ol][2 * lane] = av[r];
      tile[ol][2 * lane + 1] = bv[r];
    }
    if (k == 0) continue;  // (uniform per block: no barrier skipped by part of it)
    __syncthreads();
    const int64_t o = o0 + 2 * lane;
#pragma unroll 4
    for (int r = 0; r < 8; ++r) {
      const int il = w + 8 * r;
      const int64_t ii = i0 + il;
      if (ii >= i_pad) break;  // uniform per warp (ii grows with r)
      const int iiw = static_cast<int>(ii);  // (32-bit division: inputs < 2^31)
      const int blk = iiw / n_i;
      const int64_t row = static_cast<int64_t>(blk) * d * n_i + (k - 1) * n_i + (iiw - blk * n_i);
      if (o < ldO) {
        uint32_t h2, l2;
        split_pack2(tile[2 * lane][il], tile[2 * lane + 1][il], h2, l2);
        const int64_t q = (row * ldO + o) >> 1;
        xh[q] = h2;
        xl[q] = l2;
      }
    }
    __syncthreads();
  }
}

// fp32 copy of the coefficients (skinny layers' prep) plus the prep header
__global__ void copy_header_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n, PrepHeader* hdr,
                                   PrepHeader h) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) *hdr = h;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t e = t0; e < n4; e += stride)
    reinterpret_cast<float4*>(out)[e] = reinterpret_cast<const float4*>(in)[e];
  for (int64_t e = 4 * n4 + t0; e < n; e += stride) out[e] = in[e];
}

// part[s][c] = sum of rows [s*chunk, min((s+1)*chunk, rows)) of column c
__global__ void col_partial_kernel(const float* __restrict__ in, int64_t rows, int64_t cols, int64_t chunk,
                                   double* __restrict__ part, int slots) {
  pdl_wait();
  const int64_t n = static_cast<int64_t>(slots) * cols;
  for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < n;
       it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = it / cols, c = it - s * cols;
    const int64_t r1 = (s + 1) * chunk < rows ? (s + 1) * chunk : rows;
    double acc = 0.0;
    for (int64_t r = s * chunk; r < r1; ++r) acc += static_cast<double>(in[r * cols + c]);
    part[it] = acc;
  }
}

// out[c] = sum_s part[s][c]: block = 32 columns x 8 warps; warp w sums
// slots w, w+8, ... and the 8 partials are folded in warp order (fixed
// order for a given slot count: deterministic).
// With bcast != nullptr the block also writes bcast[c][i] = out[c] for its
// 32 columns and bcast columns i in [i0, i1) (dC_0 = db, the B_0 == 1 fold)
// -- one launch instead of a separate broadcast.  Blocks that share the 32
// columns (different broadcast ranges) recompute the same sums; only the
// first writes out[c].
__device__ __forceinline__ void col_finish_block(const double* __restrict__ part, int slots, int64_t cols,
                                                 float* __restrict__ out, float* __restrict__ bcast,
                                                 int64_t bcast_cols, int64_t cb, int64_t i0, int64_t i1,
                                                 bool write_out) {
  __shared__ double red[8][32];
  __shared__ float val[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = cb * 32;
  const int64_t c = c0 + lane;
  double acc = 0.0;
  if (c < cols) {
    int s = w;
    for (; s + 24 < slots; s += 32) {  // four loads in flight, added in slot order
      const double p0 = part[s * cols + c], p1 = part[(s + 8) * cols + c];
      const double p2 = part[(s + 16) * cols + c], p3 = part[(s + 24) * cols + c];
      acc += p0;
      acc += p1;
      acc += p2;
      acc += p3;
    }
    for (; s < slots; s += 8) acc += part[s * cols + c];
  }
  red[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += red[j][lane];
    val[lane] = static_cast<float>(t);
    if (write_out && c < cols) out[c] = static_cast<float>(t);
  }
  if (bcast == nullptr) return;
  __syncthreads();
  const int nr = cols - c0 < 32 ? static_cast<int>(cols - c0) : 32;
  for (int r = 0; r < nr; ++r) {
    float* row = bcast + (c0 + r) * bcast_cols;
    const float v = val[r];
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) row[i] = v;
  }
}

// broadcast column ranges per 32 output columns: enough blocks to fill the
// GPU (16 blocks wrote the 1 MB dC_0 of a 512 x 512 layer in 7.5 us)
int64_t bcast_split(int64_t cols, int64_t bcast_cols) {
  if (bcast_cols <= 0) return 1;
  const int64_t cb = ceil_div(cols, 32);
  int64_t by = ceil_div(static_cast<int64_t>(num_sms()) * 2, cb);
  const int64_t max_by = ceil_div(bcast_cols, 256);
  if (by > max_by) by = max_by;
  return by < 1 ? 1 : by;
}

__global__ void __launch_bounds__(256) col_finish_kernel(const double* __restrict__ part, int slots, int64_t cols,
                                                         float* __restrict__ out, float* __restrict__ bcast,
                                                         int64_t bcast_cols) {
  pdl_wait();
  const int64_t by = gridDim.y, span = ceil_div(bcast_cols, by);
  const int64_t i0 = blockIdx.y * span, i1 = i0 + span < bcast_cols ? i0 + span : bcast_cols;
  col_finish_block(part, slots, cols, out, bcast, bcast_cols, blockIdx.x, i0, i1, blockIdx.y == 0);
}

// out[n] = (acc ? out[n] : 0) + sum_s partials[s*stride + n], ascending s.
// The first `fin_blocks` blocks run a col_finish job (the bias gradient and
// dC_0 that follow a split dC GEMM) in the same launch, alongside the merge.
__global__ void merge_kernel(const float* __restrict__ partials, int S, int64_t stride, int64_t n,
                             float* __restrict__ out, int accumulate, int merge_blocks, ColFinishJob fin,
                             int64_t fin_by, int fin_blocks) {
  pdl_wait();
  if (static_cast<int>(blockIdx.x) < fin_blocks) {
    const int64_t j = blockIdx.x;
    const int64_t cb = j / fin_by, y = j - cb * fin_by;
    const int64_t span = ceil_div(fin.bcast_cols, fin_by);
    const int64_t i0 = y * span, i1 = i0 + span < fin.bcast_cols ? i0 + span : fin.bcast_cols;
    col_finish_block(fin.part, fin.slots, fin.cols, fin.out, fin.bcast, fin.bcast_cols, cb, i0, i1, y == 0);
    return;
  }
  const bool vec = (stride % 4 == 0) && (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(partials) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  const int64_t step = static_cast<int64_t>(merge_blocks) * blockDim.x;
  const int64_t t0 = (blockIdx.x - fin_blocks) * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  // the slot loads are issued 8 at a time, then added in ascending slot
  // order: a plain loop waited one L2 round trip per slot (27 slots of the
  // C2 head's dC took 11 us for 0.4 MB)
  constexpr int U = 8;
  if (vec) {
    const float4* pp = reinterpret_cast<const float4*>(partials);
    const int64_t st4 = stride / 4;
    for (int64_t i = t0; i < n / 4; i += step) {
      float4 a = accumulate ? reinterpret_cast<const float4*>(out)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      int s = 0;
      for (; s + U <= S; s += U) {
        float4 p[U];
#pragma unroll
        for (int u = 0; u < U; ++u) p[u] = __ldg(pp + (s + u) * st4 + i);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a.x += p[u].x;
          a.y += p[u].y;
          a.z += p[u].z;
          a.w += p[u].w;
        }
      }
      for (; s < S; ++s) {
        const float4 p = __ldg(pp + s * st4 + i);
        a.x += p.x;
        a.y += p.y;
        a.z += p.z;
        a.w += p.w;
      }
      reinterpret_cast<float4*>(out)[i] = a;
    }
  } else {
    for (int64_t i = t0; i < n; i += step) {
      float a = accumulate ? out[i] : 0.0f;
      int s = 0;
      for (; s + U <= S; s += U) {
        float p[U];
#pragma unroll
        for (int u = 0; u < U; ++u) p[u] = __ldg(partials + (s + u) * stride + i);
#pragma unroll
        for (int u = 0; u < U; ++u) a += p[u];
      }
      for (; s < S; ++s) a += partials[s * stride + i];
      out[i] = a;
    }
  }
}

__global__ void fill_rows_kernel(float* __restrict__ out, int64_t rows, int64_t cols, const float* __restrict__ a,
                                 const float* __restrict__ b) {
  pdl_wait();
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = i % cols;
    out[i] = (a ? a[c] : 0.0f) + (b ? b[c] : 0.0f);
  }
}

__global__ void add_rows_kernel(float* __restrict__ out, int64_t rows, int64_t cols, const float* __restrict__ a,
                                const float* __restrict__ b) {
  pdl_wait();
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = i % cols;
    out[i] += (a ? a[c] : 0.0f) + (b ? b[c] : 0.0f);
  }
}

}  // namespace

int launch_split_rows(const float* in, int64_t nz, int64_t rows, int64_t cols, int64_t in_zs, __nv_bfloat16* hi,
                      __nv_bfloat16* lo, int64_t ld, int64_t out_zs, cudaStream_t s) {
  if (nz * rows * cols == 0) return kOk;
  CK_CHECK(ld % 2 == 0 && out_zs % 2 == 0, "split_rows: pitch must be even");
  LaunchScope scope(kKSplit, s);
  CK_CUDA(launch_k((split_rows_kernel), blocks_for(nz * rows * ((cols + 1) / 2)), kThreads, 0, s, 
      in, nz, rows, cols, in_zs, reinterpret_cast<uint32_t*>(hi), reinterpret_cast<uint32_t*>(lo), ld, out_zs));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_split_rows_colsum(const float* in, int64_t rows, int64_t cols, __nv_bfloat16* hi, __nv_bfloat16* lo,
                             int64_t ld, double* part, int slots, cudaStream_t s) {
  if (cols == 0) return kOk;
  CK_CHECK(ld % 2 == 0, "split_rows_colsum: pitch must be even");
  const int64_t rb = ceil_div(rows > 0 ? rows : 1, slots);
  LaunchScope scope(kKSplit, s);
  CK_CUDA(launch_k((split_rows_colsum_kernel), dim3(static_cast<unsigned>(slots), static_cast<unsigned>(ceil_div(cols, 64))), 256, 0, s, 
      in, rows, cols, rb, reinterpret_cast<uint32_t*>(hi), reinterpret_cast<uint32_t*>(lo), ld, part));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_split_transpose(const float* in, int64_t nz, int64_t rows, int64_t cols, int64_t in_zs,
                           __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ld, int64_t out_zs, cudaStream_t s) {
  if (nz * rows * cols == 0) return kOk;
  const int64_t tiles = nz * ceil_div(rows, 32) * ceil_div(cols, 32);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  LaunchScope scope(kKSplit, s);
  CK_CUDA(launch_k((split_transpose_kernel), static_cast<int>(tiles < cap ? tiles : cap), kThreads, 0, s, in, nz, rows, cols, in_zs,
                                                                                         hi, lo, ld, out_zs));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_split_transpose_stacked(const float* c_doj, int64_t K, int64_t O, int64_t I, int n_i, __nv_bfloat16* hi,
                                   __nv_bfloat16* lo, int64_t ld, cudaStream_t s) {
  if (K < 2 || O == 0 || I == 0) return kOk;
  const int64_t i_pad = ceil_div(I, n_i) * n_i;
  const int64_t tiles = (K - 1) * ceil_div(O, 32) * ceil_div(i_pad, 32);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  LaunchScope scope(kKSplit, s);
  CK_CUDA(launch_k((split_transpose_stacked_kernel), static_cast<int>(tiles < cap ? tiles : cap), kThreads, 0, s, c_doj, K, O, I, n_i,
                                                                                                 hi, lo, ld));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_row_sum(const float* in, int64_t rows, int64_t cols, float* out, cudaStream_t s, void* hdr,
                   const PrepHeader* h) {
  if (rows == 0) return kOk;
  LaunchScope scope(kKReduce, s);
  CK_CUDA(launch_k((row_sum_kernel), blocks_for(rows * 32), kThreads, 0, s, in, rows, cols, out,
                   static_cast<PrepHeader*>(hdr), h ? *h : PrepHeader{}));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_prep_fused(const float* c_doj, int64_t K, int64_t O, int64_t I, int n_i, __nv_bfloat16* doj_hi,
                      __nv_bfloat16* doj_lo, int64_t ldI, __nv_bfloat16* dxb_hi, __nv_bfloat16* dxb_lo, int64_t ldO,
                      float* c0sum, void* hdr, const PrepHeader& h, cudaStream_t s) {
  CK_CHECK(n_i > 0 && K >= 1 && O >= 1 && I >= 1, "prep: bad stacked layout");
  const int sum_blocks = static_cast<int>(ceil_div(O, 8));
  CK_CHECK(ldI % 2 == 0 && ldO % 2 == 0, "prep: pitches must be even (bf16x2 stores)");
  const int64_t tiles = K * ceil_div(O, 64) * ceil_div(ceil_div(I, n_i) * n_i, 64);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  const int64_t want = sum_blocks + tiles;
  LaunchScope scope(kKSplit, s);
  CK_CUDA(launch_k((prep_fused_kernel), static_cast<int>(want < cap ? want : cap), kThreads, 0, s, c_doj, K, O, I, n_i,
                   sum_blocks, doj_hi, doj_lo, ldI, dxb_hi, dxb_lo, ldO, c0sum, static_cast<PrepHeader*>(hdr), h));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_copy_with_header(const float* in, float* out, int64_t n, void* hdr, const PrepHeader& h, cudaStream_t s) {
  LaunchScope scope(kKSplit, s);
  CK_CUDA(launch_k((copy_header_kernel), blocks_for(n / 4 > 0 ? n / 4 : 1), kThreads, 0, s, in, out, n,
                   static_cast<PrepHeader*>(hdr), h));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_col_partial(const float* in, int64_t rows, int64_t cols, double* part, int slots, cudaStream_t s) {
  if (cols == 0) return kOk;
  const int64_t chunk = ceil_div(rows > 0 ? rows : 1, slots);
  LaunchScope scope(kKReduce, s);
  CK_CUDA(launch_k((col_partial_kernel), blocks_for(slots * cols), kThreads, 0, s, in, rows, cols, chunk, part, slots));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_col_finish(const double* part, int slots, int64_t cols, float* out, cudaStream_t s, float* bcast,
                      int64_t bcast_cols) {
  if (cols == 0) return kOk;
  const int64_t by = bcast != nullptr ? bcast_split(cols, bcast_cols) : 1;
  LaunchScope scope(kKReduce, s);
  CK_CUDA(launch_k((col_finish_kernel), dim3(static_cast<unsigned>(ceil_div(cols, 32)), static_cast<unsigned>(by)),
                   256, 0, s, part, slots, cols, out, bcast, bcast ? bcast_cols : 0));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_merge(const float* partials, int S, int64_t stride, int64_t n, float* out, int accumulate, cudaStream_t s,
                 const ColFinishJob* fin) {
  if (n == 0) return fin ? launch_col_finish(fin->part, fin->slots, fin->cols, fin->out, s, fin->bcast,
                                             fin->bcast_cols)
                         : kOk;
  ColFinishJob f{};
  int64_t fin_blocks = 0, fin_by = 1;
  if (fin != nullptr && fin->cols > 0) {
    f = *fin;
    if (f.bcast == nullptr) f.bcast_cols = 0;
    fin_by = f.bcast ? bcast_split(f.cols, f.bcast_cols) : 1;
    fin_blocks = ceil_div(f.cols, 32) * fin_by;
  }
  const int mb = blocks_for(ceil_div(n, 4));
  LaunchScope scope(kKReduce, s);
  CK_CUDA(launch_k((merge_kernel), static_cast<unsigned>(mb + fin_blocks), kThreads, 0, s, partials, S, stride, n, out,
                   accumulate, mb, f, fin_by, static_cast<int>(fin_blocks)));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_fill_rows(float* out, int64_t rows, int64_t cols, const float* a, const float* b, cudaStream_t s) {
  if (rows * cols == 0) return kOk;
  LaunchScope scope(kKReduce, s);
  CK_CUDA(launch_k((fill_rows_kernel), blocks_for(rows * cols), kThreads, 0, s, out, rows, cols, a, b));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int launch_add_rows(float* out, int64_t rows, int64_t cols, const float* a, const float* b, cudaStream_t s) {
  if (rows * cols == 0) return kOk;
  LaunchScope scope(kKReduce, s);
  CK_CUDA(launch_k((add_rows_kernel), blocks_for(rows * cols), kThreads, 0, s, out, rows, cols, a, b));
  CK_CUDA(cudaGetLastError());
  return kOk;
}


}  // namespace ck
