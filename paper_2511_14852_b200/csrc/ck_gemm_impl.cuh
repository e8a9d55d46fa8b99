// tcgen05 split-precision (BF16x3) GEMM for the ChebyKAN contractions.
//
//   out[z][m][n] (+)= sum_{s<S} sum_r A[aseg][m][r] * B[bseg][n][r]
//
// A and B are each given as a bf16 (hi, lo) pair with v ~= hi + lo; per
// 16-wide K step the single elected MMA thread issues three
// tcgen05.mma.kind::f16 into one fp32 TMEM accumulator:
// hi*hi + hi*lo + lo*hi (the lo*lo term is below fp32 round-off).
//
// Persistent, 1 CTA/SM; CG = 2 runs CTA pairs (cta_group::2, M = 256 per
// pair tile, each CTA stages its 128 A rows and half of B).  Warp roles
// (384 threads):
//   warp 0       TMA producer (one elected lane), SWIZZLE_128B tiles, K- or
//                MN-major
//   warp 1       MMA issuer (one elected lane of the leader CTA)
//   warp 2       TMEM allocator
//   warps 4..11  epilogue: tcgen05.ld 32x32b -> registers -> store (staged
//                through shared memory, + bias) or the fused dX fold
// Pipelines: smem full/empty mbarrier ring (TMA <-> MMA), double-buffered
// TMEM accumulator with tmem-full / tmem-empty barriers (MMA <-> epilogue).
#pragma once
#include <cudaTypedefs.h>

#include <atomic>

#include <cstdlib>
#include <string>
#include <type_traits>

#include "ck_basis.cuh"
#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {

// shared host helpers (ck_gemm.cu)
int make_map(CUtensorMap* map, const __nv_bfloat16* base, int64_t R, int64_t rows, int64_t segs, int64_t ld,
             int64_t seg_stride, int box_rows, int bk, int mn_major = 0);
// fp32 output map for the TMA-store epilogue: dims (cols, rows, planes),
// 32 x 32 boxes, SWIZZLE_128B; kUnsupported when the layout does not allow it
int make_out_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t planes, int64_t ld,
                 int64_t plane_stride);
bool tma_store_enabled();
int gemm_group(int m_tiles);
// pipeline iterations per accumulation segment of the store GEMMs
// (kSegIters; CK_GEMM_SEG overrides, 0 = whole tile)
int gemm_seg();
// wave pacing (experiment, CK_GEMM_PACE = window in pipeline iterations, 0 off)
int gemm_pace();
uint32_t next_pace_tag();
// Store-GEMM N tile: a multiple of 32 (64 per CTA for MN-major B slabs) <= BN
// spreading N evenly over ceil(N/BN) tiles.
inline int store_ntile(int64_t N, int BN, int CG, bool mn_major) {
  const int gran = mn_major ? 64 * CG : 32;
  if (mn_major) {
    // coarse granule (64-wide slabs per CTA): the width with the least
    // padding, ties to the wider tile (N = 257: 3 x 128, not 2 x 256)
    int best = gran;
    for (int nt = gran; nt <= BN; nt += gran)
      if (ceil_div(N, nt) * nt <= ceil_div(N, best) * best) best = nt;
    return best;
  }
  const int64_t tiles = ceil_div(N, BN);
  const int nt = static_cast<int>(round_up(ceil_div(N, tiles), gran));
  return nt > BN ? BN : nt;
}
// fused dX GEMM with the exact-mode (analytic derivative) epilogue (ck_gemm_dx_exact.cu)
int launch_dx_exact(const struct GemmProblem& p, cudaStream_t s);
// LUT-mode fused dX with recomputed chord slopes (ck_gemm_dx_chord.cu);
// kUnsupported for kinds without a three-term recurrence
int launch_dx_chord(const struct GemmProblem& p, cudaStream_t s);

// Kernel arguments (external linkage: the per-family generated-forward
// launchers in separate translation units share this type).
struct KArgs {
  int M, N;
  int S;
  int a_seg0, a_seg_z, b_seg0, b_seg_z;
  int n_tile;      // output columns per CTA (BN, or n_i for the dx path)
  int n_mma;       // MMA N (BN, or d * n_i)
  int b_boxes;     // TMA boxes stacked along N per stage (1, or d)
  uint32_t stage_tx;
  // dx epilogue
  const float* x;
  float* dx;
  const float* dxrows;
  int lutK, lutN;
  float guard;
  int jacobian;
  int splits;      // R splits per z
  int r_chunks;    // ceil(R / kBK)
  int n_tiles, m_tiles, total_tiles;
  int group_m;     // rasterisation group (m-tiles walked per n)
  float* out;
  long long ldo, out_z_stride, out_split_stride;
  const float* bias0;
  const float* bias1;
  int accumulate;
  int out_trans;   // store out[n][m] (see GemmProblem::out_trans)
  int tma_store;   // store epilogue writes through the output tensor map (TMA bulk store / reduce-add)
  int tma_zmul;    // output map plane = split * tma_zmul + z
  // generated-operand forward (ck_gemm_gen.cu): x pitch and input count
  long long gen_ldx;
  int gen_I;
  // store GEMMs: pipeline iterations accumulated in TMEM per segment before
  // the epilogue folds the segment into fp32 registers (0: whole tile)
  int seg_iters;
  // wave pacing: units publish the window (pace_window iterations) they are
  // in; a producer does not start window w until every unit of this launch
  // reached w - pace_slack (0: off)
  int pace_window, pace_slack;
  uint32_t pace_tag;
};

// Per-unit progress of the paced GEMMs: (launch tag << 32) | window.  An
// entry of another launch counts as "not started"; a unit that finished
// writes window 0xffffffff.  Waits time out (pacing is an optimisation, never
// a dependency), so concurrent GEMMs on other streams cannot deadlock.
constexpr int kPaceSlots = 256;
__device__ unsigned long long g_pace[kPaceSlots];

__device__ __forceinline__ void pace_publish(int unit, uint32_t tag, uint32_t w) {
  *reinterpret_cast<volatile unsigned long long*>(&g_pace[unit]) = (static_cast<unsigned long long>(tag) << 32) | w;
}

__device__ __forceinline__ void pace_wait(int n_units, uint32_t tag, uint32_t need) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t lo = 0xffffffffu;
    for (int u = 0; u < n_units; ++u) {
      const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&g_pace[u]);
      const uint32_t w = (static_cast<uint32_t>(e >> 32) == tag) ? static_cast<uint32_t>(e) : 0u;
      lo = w < lo ? w : lo;
    }
    if (lo >= need) return;
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (t1 - t0 > 200000ull) return;  // 200 us: give up pacing this window
    __nanosleep(256);
  }
}

// Per-CTA timeline of the last launch (CK_GEMM_TRACE builds only; dev tool
// tools/gemm_trace.py): globaltimer at kernel entry, after the prologue
// barrier, after griddepcontrol.wait, first stage landed (MMA warp), last
// MMA committed, first accumulator drained (epilogue), last tile stored, exit.
constexpr int kTraceEvents = 8;
#ifdef CK_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[512][kTraceEvents];
__device__ __forceinline__ void gemm_trace(int ev) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (blockIdx.x < 512) g_gemm_trace[blockIdx.x][ev] = t;
}
#define CK_TRACE(ev) gemm_trace(ev)
#else
#define CK_TRACE(ev) ((void)0)
#endif

// Accumulation segments.  The tensor core's fp32 accumulation of a long
// reduction is biased (the error grows linearly with the chain: 1.06e-4
// normwise for the 32768-term C4 forward, 5.5e-5 / 2.6e-5 / 1.2e-5 with 2 /
// 4 / 8 reduction splits -- tools/accum_error.py), so store GEMMs accumulate
// kSegIters pipeline iterations (2048 reduction terms at BK = 64) in one
// TMEM buffer, then the epilogue warps add the segment into fp32 registers
// (round to nearest) while the MMAs fill the other buffer.  C4 forward
// error / time vs segment length (tools/seg_sweep.py): 16 it. 4.5e-6, +3-5 %;
// 32 it. 7.3e-6, +1-2 %; 64 it. 1.4e-5, +2 %; 128 it. 2.8e-5, +0-2 %;
// whole tile 1.06e-4.
constexpr int kSegIters = 32;

// A-operand collector reuse across the hi*hi / hi*lo MMA pair (1 = on; see
// umma_bf16_pair).  CK_BUILD_NO_COLLECTOR builds it off for comparison.
#ifdef CK_BUILD_NO_COLLECTOR
constexpr int kCollector = 0;
#else
constexpr int kCollector = 1;
#endif
__host__ __device__ inline int seg_len(int seg_iters, int iters) { return seg_iters > 0 ? seg_iters : iters; }

namespace {

constexpr int kBM = 128;
// Warpgroup 0 = control warps (TMA producer, MMA issuer, TMEM allocator),
// warpgroups 1-2 = epilogue.  The store epilogue keeps a row's 128 segment
// sums in registers (kSegIters): the control warpgroup hands registers to
// the epilogue warpgroups (setmaxnreg), 168 -> 56 / 224 per thread.
constexpr int kThreads = 384;
constexpr int kEpiWarp0 = 4;
constexpr int kCtrlRegs = 56, kEpiRegs = 224;
constexpr int kEpiWarps = 8;
// Input-gradient kernels may run EW = 16 epilogue warps (640 threads, 112
// registers each): the fused dX fold of a short-K tile is latency-bound at
// two epilogue warps per scheduler (ncu: 9 cycles per issued instruction,
// tensor pipe 28 % active at 256^2 d3), so four per scheduler overlap twice
// the gathers / tanh chains.  The store epilogue keeps 8 warps (its segment
// fold holds 128 running sums per thread).
__host__ __device__ constexpr int gemm_threads(int ew) { return 128 + 32 * ew; }
// setmaxnreg moves registers within the CTA's launch allocation (threads x
// the launch-bound register count, a multiple of 8): what the control warps
// release is all the epilogue warps can take, or their setmaxnreg.inc waits
// forever.  384 threads: 168 at launch -> 56 / 224; 640 threads: 96 -> 56 / 104.
__host__ __device__ constexpr int launch_regs(int threads) { return (65536 / threads) / 8 * 8 > 168 ? 168 : (65536 / threads) / 8 * 8; }
__host__ __device__ constexpr int epi_regs(int ew) {
  return (launch_regs(gemm_threads(ew)) * gemm_threads(ew) - 128 * kCtrlRegs) / (32 * ew) / 8 * 8;
}
static_assert(epi_regs(8) == kEpiRegs, "register budget (EW = 8)");
static_assert(epi_regs(16) == 104, "register budget (EW = 16)");
constexpr int kMaxDFused = 16;       // fused dX epilogue: degree <= 16

// BK = reduction elements per pipeline stage: 64 (128-byte rows, SWIZZLE_128B)
// or 32 (64-byte rows, SWIZZLE_64B, twice the stages for the same smem).
// CG = CTA group: 1 (one SM per 128 x BN tile) or 2 (an SM pair per 256 x BN
// tile; each CTA stages its 128 rows of A and half of the B rows).
template <int BN, int BK, int STAGES, int CG = 1>
struct Cfg {
  static constexpr int kRowBytes = BK * 2;
  static constexpr int kABytes = kBM * kRowBytes;   // one of hi / lo
  static constexpr int kBBytes = (BN / CG) * kRowBytes;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;  // double-buffered accumulator
  static constexpr int kBarrierBytes = 256;
  static constexpr int kSmemBytes = STAGES * kStageBytes + kBarrierBytes + 1024;
  static_assert(kSmemBytes <= 232448, "smem budget");
};

constexpr int kEpiStore = 0;  // out (+)= acc (+ bias)
constexpr int kEpiDx = 1;     // dx = J * sum_k slope_k * acc_k (stacked B)
constexpr int kDxmChord = 8;  // DXM offset of the chord-slope LUT epilogues


// Tile decode shared by all roles (persistent static schedule: CTA c takes
// tiles c, c + grid, ...; n fastest so co-resident CTAs share A rows in L2).
struct TileCoord {
  int n0, m0, z, split, f_begin, iters;
};

// Grouped rasterisation: consecutive tiles walk kGroupM m-tiles for one n,
// then the next n, so a wave of ~74-148 co-resident units covers a compact
// (kGroupM x ~wave/kGroupM) block and both operands are reused from L2.
__device__ __forceinline__ TileCoord decode_tile(const KArgs& p, int t, int m_tile_rows) {
  TileCoord c;
  const int nt = p.n_tiles, mt = p.m_tiles, G = p.group_m;
  const int per_z = nt * mt;
  const int zs = t / per_z;
  const int r = t - zs * per_z;
  const int group = r / (G * nt);
  const int first_m = group * G;
  const int gm = min(G, mt - first_m);  // last group may be short
  const int rr = r - group * G * nt;
  c.m0 = (first_m + rr % gm) * m_tile_rows;
  c.n0 = (rr / gm) * p.n_tile;
  c.z = zs / p.splits;
  c.split = zs % p.splits;
  // reduction splits cut the flattened (segment, K chunk) iteration space
  // into contiguous ranges (a split may cross segment boundaries)
  const long long flat = static_cast<long long>(p.S) * p.r_chunks;
  c.f_begin = static_cast<int>(static_cast<long long>(c.split) * flat / p.splits);
  c.iters = static_cast<int>(static_cast<long long>(c.split + 1) * flat / p.splits) - c.f_begin;
  return c;
}

template <int D>
struct DxBlock {
  static constexpr int K = D + 1;
  static constexpr int S = dxrow_stride(K);  // floats per dX row
  static constexpr int NS = (D + 3) / 4;     // 16-byte words holding the D slopes
  // columns per block: as many independent gathers in flight as the
  // register budget allows
  static constexpr int W = D <= 4 ? 8 : 4;
};

template <int W>
__device__ __forceinline__ void dx_load_x(const KArgs& p, const float* xr, bool row_ok, int i0, float (&xv)[W]) {
  if (W >= 4 && ((p.ldo & 3) == 0) && row_ok && i0 + W <= p.N) {
#pragma unroll
    for (int q = 0; q < W / 4; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(xr + i0 + 4 * q);
      xv[4 * q] = v.x;
      xv[4 * q + 1] = v.y;
      xv[4 * q + 2] = v.z;
      xv[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < W; ++e) xv[e] = (row_ok && i0 + e < p.N) ? xr[i0 + e] : 0.0f;
  }
}

template <int W>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[W]) {
  if constexpr (W == 8) {
    tmem_ld_32x32b_x8(taddr, r);
  } else if constexpr (W == 4) {
    tmem_ld_32x32b_x4(taddr, r);
  } else {
    tmem_ld_32x32b_x2(taddr, r);
  }
}

// Fused dX epilogue for one 128-row tile, degree D (compile time): TMEM
// column (k-1)*n_i + i holds G_k[row][n0+i] = sum_o dy[row][o] C[k][o][n0+i].
// Each thread owns one row; the two warps of a TMEM lane quarter take
// alternate column blocks of W inputs, x of the next block prefetched.  Per
// element: float32 tanh gives the position; its cell's slopes come in with
// ceil(D/4) 16-byte loads from the L2-resident dX rows.  Only when the
// float32 position lies within `guard` of a cell edge (where a 2-ulp tanhf
// error could flip the cell; ~1-3 % of elements) are the cell's
// reference boundaries {b_c, b_{c+1}} loaded and the cell corrected by one --
// the exact reference cell without float64 work.  Then fold with the d
// accumulators and apply the Jacobian.  (Each gather is one L1 wavefront per
// lane: the load count, not the bytes, bounds short-K tiles.)
template <int D, int NH = 2>
__device__ __forceinline__ void dx_epilogue(const KArgs& p, uint32_t tbase, int n0, int row, bool row_ok, int h) {
  constexpr int K = DxBlock<D>::K, S = DxBlock<D>::S, NS = DxBlock<D>::NS, W = DxBlock<D>::W;
  const int n_i = p.n_tile, N = p.lutN;
  const float* xr = p.x + static_cast<long long>(row) * p.ldo;
  float* dxr = p.dx + static_cast<long long>(row) * p.ldo;
  const bool vec = ((p.ldo & 3) == 0);
  const float hN = 0.5f * static_cast<float>(N - 1);
  const float4* rows4 = reinterpret_cast<const float4*>(p.dxrows);
  int cb = W * h;
  float xv[W];
  if (cb < n_i) dx_load_x(p, xr, row_ok, n0 + cb, xv);
#pragma unroll 1
  for (; cb < n_i; cb += NH * W) {
    uint32_t r[D][W];
#pragma unroll
    for (int k = 0; k < D; ++k) tmem_ld_cols<W>(tbase + k * n_i + cb, r[k]);
    float x_cur[W], t[W];
    int cell[W];
    bool near[W];
    float4 sl[W][NS];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      x_cur[e] = xv[e];
      const float tt = fminf(fmaxf(tanhf(xv[e]), -1.0f), 1.0f);
      t[e] = tt;
      const float pos = fmaf(tt, hN, hN);
      const int c = min(static_cast<int>(pos), N - 2);
      const float fr = pos - static_cast<float>(c);
      cell[e] = c;
      near[e] = fr < p.guard || fr > 1.0f - p.guard;
#pragma unroll
      for (int j = 0; j < NS; ++j) sl[e][j] = __ldg(rows4 + static_cast<long long>(c) * (S / 4) + j);
    }
    if (cb + NH * W < n_i) dx_load_x(p, xr, row_ok, n0 + cb + NH * W, xv);  // next block's x
#pragma unroll
    for (int e = 0; e < W; ++e) {
      if (near[e]) {
        // exact reference cell: b_c <= x < b_{c+1}; at most one step off
        const float* rw = p.dxrows + static_cast<long long>(cell[e]) * S;
        const float bl = __ldg(rw + D), bh = __ldg(rw + K);
        const bool lo = x_cur[e] < bl, hi = !(x_cur[e] < bh);
        if (lo || hi) {
          // clamped like the reference's idx = min(., N-2) (x = +inf lands past b_{N-1})
          const long long c2 = min(cell[e] + (lo ? -1 : 1), N - 2);
#pragma unroll
          for (int j = 0; j < NS; ++j) sl[e][j] = __ldg(rows4 + c2 * (S / 4) + j);
        }
      }
    }
    tmem_ld_wait();
    float acc[W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const float* f = reinterpret_cast<const float*>(sl[e]);
      float a = 0.0f;
#pragma unroll
      for (int k = 0; k < D; ++k) a = fmaf(f[k], __uint_as_float(r[k][e]), a);
      acc[e] = p.jacobian ? a * (1.0f - t[e] * t[e]) : a;
    }
    const int i0 = n0 + cb;
    if (row_ok) {
      if (W >= 4 && vec && i0 + W <= p.N) {
#pragma unroll
        for (int q = 0; q < W / 4; ++q)
          *reinterpret_cast<float4*>(dxr + i0 + 4 * q) =
              make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      } else {
#pragma unroll
        for (int e = 0; e < W; ++e)
          if (i0 + e < p.N) dxr[i0 + e] = acc[e];
      }
    }
  }
}

// LUT-mode input-gradient epilogue with recomputed chord slopes (three-term
// families): the reference cell as in dx_epilogue (float32 position, the
// cell boundaries gathered only inside the guard band), then the cell's
// slopes from chord_slopes at its float32 grid nodes -- the node recomputation
// the expansion kernels use for the values (DESIGN decision 2).  No per-element
// table gather: short-K dX tiles were bound by that gather's L2 round trip.
template <int KIND, int D, int NH = 2>
__device__ __forceinline__ void dx_epilogue_chord(const KArgs& p, uint32_t tbase, int n0, int row, bool row_ok,
                                                  int h) {
  // no slope registers to hold: 8 columns per block up to d = 8 (d = 4 with
  // the 112-register budget of 16 epilogue warps)
  constexpr int K = DxBlock<D>::K, S = DxBlock<D>::S, W = D <= (NH > 2 ? 4 : 8) ? 8 : 4;
  const int n_i = p.n_tile, N = p.lutN;
  const float* xr = p.x + static_cast<long long>(row) * p.ldo;
  float* dxr = p.dx + static_cast<long long>(row) * p.ldo;
  const bool vec = ((p.ldo & 3) == 0);
  const float hN = 0.5f * static_cast<float>(N - 1);
  const float stepf = 2.0f / static_cast<float>(N - 1);
  // columns past d_in (a ragged last tile) are skipped, not folded
  const int n_lim = min(n_i, p.N - n0);
  int cb = W * h;
  float xv[W];
  if (cb < n_lim) dx_load_x(p, xr, row_ok, n0 + cb, xv);
#pragma unroll 1
  for (; cb < n_lim; cb += NH * W) {
    uint32_t r[D][W];
#pragma unroll
    for (int k = 0; k < D; ++k) tmem_ld_cols<W>(tbase + k * n_i + cb, r[k]);
    float x_cur[W], jac[W];
    int cell[W];
    bool near[W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      x_cur[e] = xv[e];
      float tt;
      tanh_jac(xv[e], tt, jac[e]);
      const float pos = fmaf(tt, hN, hN);
      const int c = min(static_cast<int>(pos), N - 2);
      const float fr = pos - static_cast<float>(c);
      cell[e] = c;
      near[e] = fr < p.guard || fr > 1.0f - p.guard;
    }
    if (cb + NH * W < n_lim) dx_load_x(p, xr, row_ok, n0 + cb + NH * W, xv);  // next block's x
    // the block's guard-band boundary loads are all issued before any is
    // consumed (one L2 round trip per block, not per band element)
    float bl[W], bh[W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      bl[e] = bh[e] = 0.0f;
      if (near[e]) {
        const float* rw = p.dxrows + static_cast<long long>(cell[e]) * S;
        bl[e] = __ldg(rw + D);
        bh[e] = __ldg(rw + K);
      }
    }
#pragma unroll
    for (int e = 0; e < W; ++e) {
      // exact reference cell: b_c <= x < b_{c+1}; at most one step off
      if (near[e]) cell[e] = min(cell[e] + (x_cur[e] < bl[e] ? -1 : (x_cur[e] < bh[e] ? 0 : 1)), N - 2);  // x = +inf: N-2
    }
    tmem_ld_wait();
    float acc[W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      float sl[D];
      chord_slopes<KIND, D>(grid_node_f(cell[e], N, stepf), grid_node_f(cell[e] + 1, N, stepf), sl);
      float a = 0.0f;
#pragma unroll
      for (int k = 0; k < D; ++k) a = fmaf(sl[k], __uint_as_float(r[k][e]), a);
      acc[e] = p.jacobian ? a * jac[e] : a;
    }
    const int i0 = n0 + cb;
    if (row_ok) {
      if (W >= 4 && vec && i0 + W <= p.N) {
#pragma unroll
        for (int q = 0; q < W / 4; ++q)
          *reinterpret_cast<float4*>(dxr + i0 + 4 * q) =
              make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      } else {
#pragma unroll
        for (int e = 0; e < W; ++e)
          if (i0 + e < p.N) dxr[i0 + e] = acc[e];
      }
    }
  }
}

// Exact-mode input-gradient epilogue (BasisPath.EXACT_RECURRENCE): the
// slopes are the analytic derivatives derivative_rows(kind, t)
// (basis.py:155-204, kernels.py:224) at float32 t = tanh(x), recomputed in
// registers; no table and no cell.
template <int KIND, int D, int NH = 2>
__device__ __forceinline__ void dx_epilogue_exact(const KArgs& p, uint32_t tbase, int n0, int row, bool row_ok,
                                                  int h) {
  constexpr int W = D <= 8 ? 4 : 2;
  const int n_i = p.n_tile;
  const float* xr = p.x + static_cast<long long>(row) * p.ldo;
  float* dxr = p.dx + static_cast<long long>(row) * p.ldo;
  const bool vec = ((p.ldo & 3) == 0);
#pragma unroll 1
  for (int cb = W * h; cb < n_i; cb += NH * W) {
    uint32_t r[D][W];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if constexpr (W == 4) {
        tmem_ld_32x32b_x4(tbase + k * n_i + cb, r[k]);
      } else {
        tmem_ld_32x32b_x2(tbase + k * n_i + cb, r[k]);
      }
    }
    const int i0 = n0 + cb;
    float xv[W];
    if (W == 4 && vec && row_ok && i0 + 4 <= p.N) {
      const float4 v = *reinterpret_cast<const float4*>(xr + i0);
      xv[0] = v.x; xv[1] = v.y; xv[W - 2] = v.z; xv[W - 1] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < W; ++e) xv[e] = (row_ok && i0 + e < p.N) ? xr[i0 + e] : 0.0f;
    }
    float acc[W];
    float t[W];
    float dv[W][D + 1];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      t[e] = tanhf(xv[e]);
      deriv_f32<KIND, D>(t[e], dv[e]);
    }
    tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < W; ++e) {
      float a = 0.0f;
#pragma unroll
      for (int k = 0; k < D; ++k) a = fmaf(dv[e][k + 1], __uint_as_float(r[k][e]), a);
      acc[e] = p.jacobian ? a * (1.0f - t[e] * t[e]) : a;
    }
    if (row_ok) {
      if (W == 4 && vec && i0 + 4 <= p.N) {
        *reinterpret_cast<float4*>(dxr + i0) = make_float4(acc[0], acc[1], acc[W - 2], acc[W - 1]);
      } else {
#pragma unroll
        for (int e = 0; e < W; ++e)
          if (i0 + e < p.N) dxr[i0 + e] = acc[e];
      }
    }
  }
}

// Store epilogue, one 32-row x 32-column accumulator chunk of a warp (lane =
// row, r[j] = column j): staged through a warp-private 4 KB shared tile
// (16-byte slots XOR-swizzled by row, conflict-free both ways) so that each
// global store instruction writes four full 128-byte row segments instead of
// 32 scattered 16-byte pieces -- the partial-line writes made the store
// epilogue of a one-tile-per-CTA launch take ~7 us.
constexpr int kEpiTileBytes = 32 * 32 * 4;

__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}

// One 32 x 32 accumulator chunk through the TMA: the warp stages its rows
// (+ bias) in its 1 KB-aligned 4 KB tile in the SWIZZLE_128B layout of the
// output map's 32 x 32 box, and lane 0 issues one bulk tensor store (or
// reduce-add for out +=) -- the copy engine writes the 4 KB, no per-thread
// global stores.  Rows >= M / columns >= N of the box are clipped by the TMA.
// The previous chunk's bulk read of the tile must be done before it is
// rewritten (wait_group.read).
__device__ __forceinline__ void store_chunk_tma(const uint32_t (&r)[32], float* tile, int lane, int row0, int nb,
                                               int N, int plane, const CUtensorMap* map, const float* bias0,
                                               const float* bias1, int accumulate) {
  const uint32_t ts = smem_u32(tile);
  float b[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) b[e] = 0.0f;
  if (bias0 || bias1) {
    if (nb + 32 <= N) {
#pragma unroll
      for (int e4 = 0; e4 < 8; ++e4) {
        if (bias0) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(bias0 + nb) + e4);
          b[4 * e4] += q.x; b[4 * e4 + 1] += q.y; b[4 * e4 + 2] += q.z; b[4 * e4 + 3] += q.w;
        }
        if (bias1) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(bias1 + nb) + e4);
          b[4 * e4] += q.x; b[4 * e4 + 1] += q.y; b[4 * e4 + 2] += q.z; b[4 * e4 + 3] += q.w;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        if (nb + e < N) {
          if (bias0) b[e] += __ldg(bias0 + nb + e);
          if (bias1) b[e] += __ldg(bias1 + nb + e);
        }
      }
    }
  }
  if (lane == 0) bulk_wait_read_all();
  __syncwarp();
#pragma unroll
  for (int c4 = 0; c4 < 8; ++c4) {
    const int slot = c4 ^ (lane & 7);
    sts128(ts + (lane * 32 + slot * 4) * 4, __uint_as_float(r[4 * c4]) + b[4 * c4],
           __uint_as_float(r[4 * c4 + 1]) + b[4 * c4 + 1], __uint_as_float(r[4 * c4 + 2]) + b[4 * c4 + 2],
           __uint_as_float(r[4 * c4 + 3]) + b[4 * c4 + 3]);
  }
  fence_proxy_async_smem();  // generic-proxy smem writes -> the bulk copy
  __syncwarp();
  if (lane == 0) {
    if (accumulate) {
      tma_reduce_add_3d(map, ts, nb, row0, plane);
    } else {
      tma_store_3d(map, ts, nb, row0, plane);
    }
    bulk_commit();
  }
}

// One 32 x 32 accumulator chunk (this warp's 32 rows, columns nb..nb+31)
// to the output through the warp's XOR-swizzled 4 KB staging tile: each
// store instruction then writes four whole 128-byte row segments.  The
// staging tile is addressed in the shared window (ld/st.shared: generic
// accesses cost an address-space check each) and all eight row groups'
// loads are issued before the stores.
__device__ __forceinline__ void store_chunk_coalesced(const uint32_t (&r)[32], float* tile, int lane, int row0,
                                                      int M, int nb, int N, float* out, long long ldo,
                                                      const float* bias0, const float* bias1, int accumulate,
                                                      bool vec) {
  const uint32_t ts = smem_u32(tile);
#pragma unroll
  for (int c4 = 0; c4 < 8; ++c4) {
    const int slot = c4 ^ (lane & 7);
    sts128(ts + (lane * 32 + slot * 4) * 4, __uint_as_float(r[4 * c4]), __uint_as_float(r[4 * c4 + 1]),
           __uint_as_float(r[4 * c4 + 2]), __uint_as_float(r[4 * c4 + 3]));
  }
  __syncwarp();
#ifdef CK_EPI_NOSTORE
  if (M > 0) return;  // timing experiment: stage only, no global stores
#endif
  const int c4 = lane & 7;      // this lane's 4 columns
  const int rsub = lane >> 3;   // row within each group of 4
  const int n = nb + 4 * c4;
  const bool full = vec && n + 4 <= N;
  float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
  if (full) {
    if (bias0) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(bias0 + n));
      bv.x += b.x; bv.y += b.y; bv.z += b.z; bv.w += b.w;
    }
    if (bias1) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(bias1 + n));
      bv.x += b.x; bv.y += b.y; bv.z += b.z; bv.w += b.w;
    }
  }
  float4 v[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int lr = 4 * g + rsub;
    v[g] = lds128(ts + (lr * 32 + ((c4 ^ (lr & 7)) * 4)) * 4);
  }
  __syncwarp();
  float* dst = out + static_cast<long long>(row0 + rsub) * ldo + n;
  const long long step = 4 * ldo;
#pragma unroll
  for (int g = 0; g < 8; ++g, dst += step) {
    if (row0 + 4 * g + rsub >= M) continue;
    float4 w = v[g];
    if (full) {
      w.x += bv.x; w.y += bv.y; w.z += bv.z; w.w += bv.w;
      if (accumulate) {
        const float4 prev = *reinterpret_cast<const float4*>(dst);
        w.x += prev.x; w.y += prev.y; w.z += prev.z; w.w += prev.w;
      }
      *reinterpret_cast<float4*>(dst) = w;
    } else {
      const float e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (n + q < N) {
          float o = e[q];
          if (bias0) o += bias0[n + q];
          if (bias1) o += bias1[n + q];
          if (accumulate) o += dst[q];
          dst[q] = o;
        }
      }
    }
  }
}

// DXM: input-gradient epilogue flavour -- 0 = LUT slopes gathered from the
// dX rows (exact reference cell), 1 + kind = analytic derivatives of that
// basis kind (exact mode), kDxmChord + kind = LUT slopes recomputed as chords.
template <int BN, int BK, int STAGES, int EPI, int CG, int AMN, int BMN, int DXM = 0, int EW = kEpiWarps>
__global__ void __launch_bounds__(gemm_threads(EW), 1)
    gemm_bf16x3_kernel(const __grid_constant__ CUtensorMap tm_a_hi, const __grid_constant__ CUtensorMap tm_a_lo,
                       const __grid_constant__ CUtensorMap tm_b_hi, const __grid_constant__ CUtensorMap tm_b_lo,
                       const __grid_constant__ CUtensorMap tm_out, const KArgs p) {
  using C = Cfg<BN, BK, STAGES, CG>;
  constexpr int kRowBytes = C::kRowBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // layout: operand stages | store epilogue staging tiles (4 KB per warp,
  // 1 KB-aligned for the SWIZZLE_128B TMA box) | barriers
  constexpr int kTileRegion = EPI == kEpiStore ? kEpiWarps * kEpiTileBytes : 0;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes + kTileRegion);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2] accumulator ready (MMA -> epilogue)
  uint64_t* tempty = tfull + 2;      // [2] accumulator drained (epilogue -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = p.total_tiles;
  // persistent schedule over work units (a CTA, or a CTA pair for CG = 2)
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit = blockIdx.x / CG, n_units = gridDim.x / CG;
  const int row_off = static_cast<int>(rank) * kBM;  // this CTA's rows inside a pair tile
  if (threadIdx.x == 0) CK_TRACE(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a_hi);
    tma_prefetch_desc(&tm_a_lo);
    tma_prefetch_desc(&tm_b_hi);
    tma_prefetch_desc(&tm_b_lo);
    if (p.tma_store) tma_prefetch_desc(&tm_out);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG * EW);  // one arrive per epilogue warp (of both CTAs)
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      tmem_alloc_pair(tmem_slot, C::kTmemCols);
    } else {
      tmem_alloc(tmem_slot, C::kTmemCols);
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync();  // barriers of both CTAs initialised before any remote signal
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) CK_TRACE(1);
  // everything above is CTA-local; operands and outputs are touched below
  pdl_wait();
  if (threadIdx.x == 0) CK_TRACE(2);

  if (warp < kEpiWarp0) {
  reg_dealloc<kCtrlRegs>();  // (warpgroup-uniform)
  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t g = 0;  // global k-iteration counter (smem ring position)
      const int b_half = p.n_mma / CG;  // B rows this CTA stages
      for (int t = unit; t < total; t += n_units) {
        const TileCoord tc = decode_tile(p, t, kBM * CG);
        for (int it = 0; it < tc.iters; ++it, ++g) {
          if (p.pace_window > 0 && g % p.pace_window == 0) {
            const uint32_t w = g / p.pace_window;
            if (leader) pace_publish(unit, p.pace_tag, w);
            if (w > static_cast<uint32_t>(p.pace_slack)) pace_wait(n_units, p.pace_tag, w - p.pace_slack);
          }
          const int stage = g % STAGES;
          const uint32_t phase = (g / STAGES) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * C::kStageBytes;
          const int f = tc.f_begin + it;
          const int s = f / p.r_chunks;
          const int r0 = (f - s * p.r_chunks) * BK;
          const int aseg = p.a_seg0 + s + p.a_seg_z * tc.z;
          const int bseg = p.b_seg0 + s + p.b_seg_z * tc.z;
          const int arow = tc.m0 + row_off;
          int brow, bz;
          if (EPI == kEpiDx) {
            // stacked operand: the d x n_i N tile is one box of n_mma rows (per pair)
            brow = (tc.n0 / p.n_tile) * p.n_mma + static_cast<int>(rank) * b_half;
            bz = 0;
          } else {
            brow = tc.n0 + static_cast<int>(rank) * b_half;
            bz = bseg;
          }
          if constexpr (CG == 2) {
            if (leader) mbar_arrive_expect_tx(&full[stage], p.stage_tx);  // bytes of both CTAs
          } else {
            mbar_arrive_expect_tx(&full[stage], p.stage_tx);
          }
          // A: 128 rows of this CTA; B: b_half rows.  MN-major operands come
          // as 64-wide MN slabs (8 KB each for BK = 64).
          auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1, int c2) {
            if constexpr (CG == 2) {
              tma_load_3d_pair(dst, map, &full[stage], c0, c1, c2);
            } else {
              tma_load_3d(dst, map, &full[stage], c0, c1, c2);
            }
          };
          if constexpr (AMN) {
#pragma unroll
            for (int j = 0; j < kBM / 64; ++j) {
              load(st + j * 64 * kRowBytes, &tm_a_hi, arow + 64 * j, r0, aseg);
              load(st + C::kABytes + j * 64 * kRowBytes, &tm_a_lo, arow + 64 * j, r0, aseg);
            }
          } else {
            load(st, &tm_a_hi, r0, arow, aseg);
            load(st + C::kABytes, &tm_a_lo, r0, arow, aseg);
          }
          if constexpr (BMN) {
            for (int j = 0; j < b_half / 64; ++j) {
              load(st + 2 * C::kABytes + j * 64 * kRowBytes, &tm_b_hi, brow + 64 * j, r0, bz);
              load(st + 2 * C::kABytes + C::kBBytes + j * 64 * kRowBytes, &tm_b_lo, brow + 64 * j, r0, bz);
            }
          } else {
            load(st + 2 * C::kABytes, &tm_b_hi, r0, brow, bz);
            load(st + 2 * C::kABytes + C::kBBytes, &tm_b_lo, r0, brow, bz);
          }
        }
      }
      if (p.pace_window > 0 && leader) pace_publish(unit, p.pace_tag, 0xffffffffu);
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader CTA of a pair) ----------------
      const uint32_t idesc = umma_idesc_bf16_f32(kBM * CG, p.n_mma, AMN, BMN);
      uint32_t g = 0, seg = 0;
      for (int t = unit; t < total; t += n_units) {
        const TileCoord tc = decode_tile(p, t, kBM * CG);
        const int D = seg_len(p.seg_iters, tc.iters);
        for (int s0 = 0; s0 < tc.iters; s0 += D, ++seg) {
        // one accumulation segment: iterations [s0, s1) into buffer seg & 1
        const uint32_t acc = seg & 1, use = seg >> 1;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);  // epilogue has drained this buffer
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int s1 = min(s0 + D, tc.iters);
        for (int it = s0; it < s1; ++it, ++g) {
          const int stage = g % STAGES;
          const uint32_t phase = (g / STAGES) & 1;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (g == 0) CK_TRACE(3);
          const uint32_t a_hi = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t a_lo = a_hi + C::kABytes;
          const uint32_t b_hi = a_hi + 2 * C::kABytes;
          const uint32_t b_lo = b_hi + C::kBBytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // K-major: 16 bf16 = 32 bytes along the swizzled row;
            // MN-major: 16 K-rows = 2 core groups = 2048 bytes
            constexpr uint32_t kSlab = 64 * kRowBytes;
            uint64_t dah, dal, dbh, dbl;
            if constexpr (AMN) {
              dah = umma_desc_mnmajor(a_hi + kk * 2048, kSlab);
              dal = umma_desc_mnmajor(a_lo + kk * 2048, kSlab);
            } else {
              dah = umma_desc_kmajor<kRowBytes>(a_hi + kk * 32);
              dal = umma_desc_kmajor<kRowBytes>(a_lo + kk * 32);
            }
            if constexpr (BMN) {
              dbh = umma_desc_mnmajor(b_hi + kk * 2048, kSlab);
              dbl = umma_desc_mnmajor(b_lo + kk * 2048, kSlab);
            } else {
              dbh = umma_desc_kmajor<kRowBytes>(b_hi + kk * 32);
              dbl = umma_desc_kmajor<kRowBytes>(b_lo + kk * 32);
            }
            const uint32_t accum = ((it - s0) | kk) != 0 ? 1u : 0u;
            if constexpr (CG == 2) {
              umma_bf16_pair<kCollector>(d_tmem, dah, dbh, idesc, accum);
              umma_bf16_pair<kCollector ? 2 : 0>(d_tmem, dah, dbl, idesc, 1u);
              umma_bf16_pair(d_tmem, dal, dbh, idesc, 1u);
            } else {
              umma_bf16<kCollector>(d_tmem, dah, dbh, idesc, accum);
              umma_bf16<kCollector ? 2 : 0>(d_tmem, dah, dbl, idesc, 1u);
              umma_bf16(d_tmem, dal, dbh, idesc, 1u);
            }
          }
          // frees the smem slot (in both CTAs) once these MMAs retire
          if constexpr (CG == 2) {
            umma_commit_pair(&empty[stage]);
          } else {
            umma_commit(&empty[stage]);
          }
        }
        if constexpr (CG == 2) {
          umma_commit_pair(&tfull[acc]);
        } else {
          umma_commit(&tfull[acc]);
        }
        }
      }
      CK_TRACE(4);
    }
  }
  } else {
    static_assert(EW == kEpiWarps || EPI == kEpiDx, "the store epilogue runs 8 warps");
    reg_alloc<epi_regs(EW)>();
    const int q = warp & 3;                  // TMEM lane quarter this warp may access
    const int h = (warp - kEpiWarp0) >> 2;   // which half of the tile's columns
    uint32_t seg = 0;
    for (int t = unit; t < total; t += n_units) {
      const TileCoord tc = decode_tile(p, t, kBM * CG);
      const int row = tc.m0 + row_off + q * 32 + lane;
      const bool row_ok = row < p.M;
      if constexpr (EPI == kEpiDx) {
        // one segment per tile (seg_iters = 0)
        const uint32_t acc = seg & 1, use = seg >> 1;
        ++seg;
        mbar_wait(&tfull[acc], use & 1);
        tc_fence_after();
        const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
        // ------------- fused dX epilogue (degree-specialized) -------------
        if constexpr (DXM == 0) {
          switch (p.b_boxes) {
#define CK_DX_CASE(D) \
  case D:             \
    dx_epilogue<D, EW / 4>(p, tbase, tc.n0, row, row_ok, h); \
    break;
            CK_DX_CASE(1) CK_DX_CASE(2) CK_DX_CASE(3) CK_DX_CASE(4) CK_DX_CASE(5) CK_DX_CASE(6) CK_DX_CASE(7)
            CK_DX_CASE(8) CK_DX_CASE(9) CK_DX_CASE(10) CK_DX_CASE(11) CK_DX_CASE(12) CK_DX_CASE(13)
            CK_DX_CASE(14) CK_DX_CASE(15) CK_DX_CASE(16)
#undef CK_DX_CASE
            default:
              break;
          }
        } else if constexpr (DXM >= kDxmChord) {
          constexpr int KIND = DXM - kDxmChord;
          switch (p.b_boxes) {
#define CK_DX_CASE(D)                                            \
  case D:                                                        \
    dx_epilogue_chord<KIND, D, EW / 4>(p, tbase, tc.n0, row, row_ok, h); \
    break;
            CK_DX_CASE(1) CK_DX_CASE(2) CK_DX_CASE(3) CK_DX_CASE(4) CK_DX_CASE(5) CK_DX_CASE(6) CK_DX_CASE(7)
            CK_DX_CASE(8) CK_DX_CASE(9) CK_DX_CASE(10) CK_DX_CASE(11) CK_DX_CASE(12) CK_DX_CASE(13)
            CK_DX_CASE(14) CK_DX_CASE(15) CK_DX_CASE(16)
#undef CK_DX_CASE
            default:
              break;
          }
        } else {
          constexpr int KIND = DXM - 1;
          switch (p.b_boxes) {
#define CK_DX_CASE(D)                                                   \
  case D:                                                               \
    if constexpr (KIND != kFourier || D % 2 == 0) {                     \
      dx_epilogue_exact<KIND, D, EW / 4>(p, tbase, tc.n0, row, row_ok, h); \
    }                                                                   \
    break;
            CK_DX_CASE(1) CK_DX_CASE(2) CK_DX_CASE(3) CK_DX_CASE(4) CK_DX_CASE(5) CK_DX_CASE(6) CK_DX_CASE(7)
            CK_DX_CASE(8) CK_DX_CASE(9) CK_DX_CASE(10) CK_DX_CASE(11) CK_DX_CASE(12) CK_DX_CASE(13)
            CK_DX_CASE(14) CK_DX_CASE(15) CK_DX_CASE(16)
#undef CK_DX_CASE
            default:
              break;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) {
            mbar_arrive_cluster(&tempty[acc], 0);  // the leader's MMA warp waits on it
          } else {
            mbar_arrive(&tempty[acc]);
          }
        }
      } else {
        // ------------- store epilogue -------------
        float* out = p.out + static_cast<long long>(tc.z) * p.out_z_stride +
                     static_cast<long long>(tc.split) * p.out_split_stride;
        const bool vec = ((p.ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
        float* tile = reinterpret_cast<float*>(smem + STAGES * C::kStageBytes + (warp - kEpiWarp0) * kEpiTileBytes);
        const int plane = tc.split * p.tma_zmul + tc.z;
        const int row0 = tc.m0 + row_off + q * 32;
        // one 32-column chunk (this thread's row) to the output, + bias
        auto store32 = [&](const uint32_t (&v)[32], int c) {
          const int nb = tc.n0 + c;
          if (c >= p.n_tile || nb >= p.N) return;
          if (p.out_trans) {
            // transposed: column n of the tile is a row of the output; lanes
            // (= tile rows) are contiguous there, so each store is 128 bytes
            if (row_ok) {
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                const int n = nb + e;
                if (n < p.N) {
                  float o = __uint_as_float(v[e]);
                  if (p.bias0) o += p.bias0[n];
                  if (p.bias1) o += p.bias1[n];
                  float* dst = out + static_cast<long long>(n) * p.ldo + row;
                  if (p.accumulate) o += *dst;
                  *dst = o;
                }
              }
            }
          } else if (p.tma_store) {
            store_chunk_tma(v, tile, lane, row0, nb, p.N, plane, &tm_out, p.bias0, p.bias1, p.accumulate);
          } else {
            store_chunk_coalesced(v, tile, lane, row0, p.M, nb, p.N, out, p.ldo, p.bias0, p.bias1, p.accumulate, vec);
          }
        };
        auto release = [&](uint32_t acc) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) {
              mbar_arrive_cluster(&tempty[acc], 0);  // the leader's MMA warp waits on it
            } else {
              mbar_arrive(&tempty[acc]);
            }
          }
        };
        const int D = seg_len(p.seg_iters, tc.iters);
        const int nseg = (tc.iters + D - 1) / D;
        if (nseg == 1) {
          // one segment: nothing to fold -- stream 32-column chunks from TMEM
          // to the output (loads and stores interleaved; short-K tiles are
          // epilogue-bound)
          const uint32_t acc = seg & 1, use = seg >> 1;
          ++seg;
          mbar_wait(&tfull[acc], use & 1);
          tc_fence_after();
          if (seg == 1 && warp == kEpiWarp0 && lane == 0) CK_TRACE(5);
          const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
          for (int c = 32 * h; c < p.n_tile; c += 64) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tbase + c, r);
            tmem_ld_wait();
            store32(r, c);
          }
          release(acc);
        } else {
          // Fold the tile's accumulation segments into fp32 registers: this
          // thread's row, columns 32 h + 64 ch + [0, 32) (round-to-nearest
          // adds; see kSegIters).  Each drained buffer is released before the
          // next wait, so the MMAs of the following segment overlap the fold.
          constexpr int NCH = BN / 64;
          float sums[NCH][32];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int e = 0; e < 32; ++e) sums[ch][e] = 0.0f;
          for (int j = 0; j < nseg; ++j, ++seg) {
            const uint32_t acc = seg & 1, use = seg >> 1;
            mbar_wait(&tfull[acc], use & 1);
            tc_fence_after();
            const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
            // every chunk of the buffer (columns past a narrow tile's n_tile
            // are allocated and never stored), 16 columns per load
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
              for (int e0 = 0; e0 < 32; e0 += 16) {
                uint32_t r[16];
                tmem_ld_32x32b_x16(tbase + 32 * h + 64 * ch + e0, r);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 16; ++e) sums[ch][e0 + e] += __uint_as_float(r[e]);
              }
            }
            release(acc);
          }
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) store32(reinterpret_cast<const uint32_t(&)[32]>(sums[ch]), 32 * h + 64 * ch);
        }
      }
    }
  }
  if (EPI == kEpiStore && p.tma_store && warp >= kEpiWarp0 && lane == 0) bulk_wait_all();  // stores complete
  if (warp == kEpiWarp0 && lane == 0) CK_TRACE(6);
  __syncwarp();  // reconverge the role warps before the aligned barriers
  if constexpr (CG == 2) {
    tc_fence_before();
    cluster_sync();  // no CTA leaves while its peer may still signal it
    if (threadIdx.x == 0) CK_TRACE(7);
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc_pair(tmem_base, C::kTmemCols);
    }
  } else {
    __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc(tmem_base, C::kTmemCols);
    }
  }
}

// ----------------------------------------------------------------------------
// Host side: launch

template <int BN, int BK, int STAGES, int EPI, int CG, int AMN = 0, int BMN = 0, int DXM = 0, int EW = kEpiWarps>
int launch(const GemmProblem& p, int splits, float* out, long long out_split_stride, int accumulate,
           cudaStream_t s) {
  static_assert(!(AMN || BMN) || BK == 64, "MN-major operands use 128-byte (BK = 64) K slabs");
  using C = Cfg<BN, BK, STAGES, CG>;
  constexpr int kRowBytes = C::kRowBytes;
  const int r_chunks = static_cast<int>(ceil_div(p.R, BK));
  // store GEMMs: the N tile width is a runtime multiple of 32 (64 per CTA for
  // MN-major B slabs) <= BN, spreading N evenly over ceil(N/BN) tiles -- a
  // ragged N (e.g. 257) then wastes one 32-column step, not half a tile
  const int n_tile = EPI != kEpiDx ? store_ntile(p.b.rows, BN, CG, BMN) : p.dx->n_i;
  const int b_boxes = EPI == kEpiDx ? p.S : 1;
  const int n_mma = n_tile * b_boxes;
  CK_CHECK(n_mma % (8 * CG) == 0 && n_mma <= BN, "gemm: bad MMA N");
  CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
  CK_CHECK(p.a.mn_major == AMN && p.b.mn_major == BMN, "gemm: operand majorness mismatch");
  CK_TRY(make_map(&ta_hi, p.a.hi, p.R, p.a.rows, p.a.segs, p.a.ld, p.a.seg_stride, kBM, BK, AMN));
  CK_TRY(make_map(&ta_lo, p.a.lo, p.R, p.a.rows, p.a.segs, p.a.ld, p.a.seg_stride, kBM, BK, AMN));
  const int b_box = n_mma / CG;  // each CTA of a pair stages half of the B rows
  CK_CHECK(!BMN || b_box % 64 == 0, "gemm: MN-major B tile must be a multiple of 64 rows");
  CK_TRY(make_map(&tb_hi, p.b.hi, p.R, p.b.rows, p.b.segs, p.b.ld, p.b.seg_stride, b_box, BK, BMN));
  CK_TRY(make_map(&tb_lo, p.b.lo, p.R, p.b.rows, p.b.segs, p.b.ld, p.b.seg_stride, b_box, BK, BMN));
  KArgs k{};
  k.n_tile = n_tile;
  k.n_mma = n_mma;
  k.b_boxes = b_boxes;
  // bytes landing on the (leader's) full barrier per stage: A and B of all CTAs
  k.stage_tx = static_cast<uint32_t>(CG * 2 * C::kABytes + 2 * n_mma * kRowBytes);
  if (EPI == kEpiDx) {
    k.x = p.dx->x;
    k.dx = p.dx->dx;
    k.dxrows = p.dx->lut.dxrows;
    k.lutK = p.dx->lut.K;
    k.lutN = p.dx->lut.N;
    // float32 position error <= (2-ulp tanhf + fma rounding) * (N-1)/2 < 0.01
    // cells at N = 32768: inside this band the epilogue checks the cell's
    // reference boundaries (tested within 3 ulps of cell edges)
    k.guard = fminf(0.5f, fmaxf(1e-3f, 4e-7f * static_cast<float>(p.dx->lut.N)));
    k.jacobian = p.dx->jacobian;
  }
  k.M = static_cast<int>(p.a.rows);
  k.N = static_cast<int>(EPI == kEpiDx ? p.dx->cols : p.b.rows);
  k.S = EPI == kEpiDx ? 1 : p.S;
  k.a_seg0 = p.a_seg0;
  k.a_seg_z = p.a_seg_z;
  k.b_seg0 = p.b_seg0;
  k.b_seg_z = p.b_seg_z;
  k.splits = splits;
  k.r_chunks = r_chunks;
  k.out = out;
  k.ldo = p.ldo;
  k.out_z_stride = p.out_z_stride;
  k.out_split_stride = out_split_stride;
  k.bias0 = splits == 1 ? p.bias0 : nullptr;
  k.bias1 = splits == 1 ? p.bias1 : nullptr;
  k.accumulate = accumulate;
  k.seg_iters = EPI == kEpiStore ? gemm_seg() : 0;
  k.pace_window = gemm_pace();
  k.pace_slack = 2;
  k.pace_tag = k.pace_window > 0 ? next_pace_tag() : 0;
  k.out_trans = p.out_trans;
  // TMA-store epilogue for short reductions (<= 256 K chunks per tile), where
  // the last tile's store is exposed: 256^2 d3 forward 24.3 -> 21.8 us, the
  // C2 step 511 -> 501 us.  Long tiles (C4: 512 chunks) keep the per-thread
  // stores: there the store hides behind the next tile's MMAs and the bulk
  // stores, sharing the TMA unit with the operand loads, measured 0.3 %
  // slower (3 alternating runs each, profiles/r02_session3.md).  Partial
  // slots [split][z] must form one plane sequence.
  CUtensorMap to{};
  k.tma_store = 0;
  k.tma_zmul = 0;
  const int64_t chunks_per_tile = ceil_div(static_cast<int64_t>(k.S) * r_chunks, static_cast<int64_t>(splits));
  if (EPI == kEpiStore && !p.out_trans && tma_store_enabled() && chunks_per_tile <= 256 &&
      (splits == 1 || out_split_stride == static_cast<long long>(p.nz) * p.out_z_stride)) {
    const int64_t planes = static_cast<int64_t>(p.nz) * splits;
    if (make_out_map(&to, out, k.M, k.N, planes, p.ldo, planes > 1 ? p.out_z_stride : p.ldo * k.M) == kOk) {
      k.tma_store = 1;
      k.tma_zmul = splits > 1 ? p.nz : 0;
    }
  }
  auto kernel = gemm_bf16x3_kernel<BN, BK, STAGES, EPI, CG, AMN, BMN, DXM, EW>;
  // store kernels: + a 4 KB staging tile per epilogue warp
  constexpr int kSmem = C::kSmemBytes + (EPI == kEpiStore ? kEpiWarps * kEpiTileBytes : 0);
  static_assert(kSmem <= 232448, "smem budget");
  // the opt-in shared-memory size is a per-device function attribute
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  CK_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
    CK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr_set.fetch_or(bit);
  }
  k.n_tiles = static_cast<int>(ceil_div(k.N, n_tile));
  k.m_tiles = static_cast<int>(ceil_div(k.M, kBM * CG));
  k.group_m = gemm_group(k.m_tiles);
  const long long total = static_cast<long long>(k.n_tiles) * k.m_tiles * p.nz * splits;
  CK_CHECK(total < (1ll << 31), "gemm: too many tiles");
  k.total_tiles = static_cast<int>(total);
  const int units_max = gemm_sms() / CG;
  const int units = static_cast<int>(total < units_max ? total : units_max);
  LaunchScope scope(p.kclass, s);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(units * CG));
  cfg.blockDim = dim3(gemm_threads(EW));
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CG;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {  // prologue overlaps the previous kernel's tail
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  CK_CUDA(cudaLaunchKernelEx(&cfg, kernel, ta_hi, ta_lo, tb_hi, tb_lo, to, k));
  return kOk;
}

}  // namespace
}  // namespace ck
