// tcgen05 split-precision (BF16x3) GEMM for the ChebyKAN contractions.
//
//   out[z][m][n] (+)= sum_{s<S} sum_r A[aseg][m][r] * B[bseg][n][r]
//
// A and B are each given as a bf16 (hi, lo) pair with v ~= hi + lo; per
// 16-wide K step the single elected MMA thread issues three
// tcgen05.mma.kind::f16 into one fp32 TMEM accumulator:
// hi*hi + hi*lo + lo*hi (the lo*lo term is below fp32 round-off).
//
// Warp roles (256 threads, 1 CTA/SM):
//   warp 0      TMA producer (one elected lane), SWIZZLE_128B K-major tiles
//   warp 1      MMA issuer (one elected lane)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> registers -> (+bias) -> global
// Pipelines: smem full/empty mbarrier ring (TMA <-> MMA), one tmem-full
// barrier (MMA -> epilogue).
#include <cudaTypedefs.h>

#include <mutex>

#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;           // one 128-byte swizzle row of bf16
constexpr int kRowBytes = kBK * 2;
constexpr int kThreads = 256;

template <int BN, int STAGES>
struct Cfg {
  static constexpr int kABytes = kBM * kRowBytes;   // one of hi / lo
  static constexpr int kBBytes = BN * kRowBytes;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  static constexpr int kBarrierBytes = 256;
  static constexpr int kSmemBytes = STAGES * kStageBytes + kBarrierBytes + 1024;
  static_assert(kSmemBytes <= 232448, "smem budget");
};

constexpr int kEpiStore = 0;  // out (+)= acc (+ bias)
constexpr int kEpiDx = 1;     // dx = J * sum_k slope_k * acc_k (stacked B)

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
  const float* slopes_pm;
  int lutK, lutN;
  int jacobian;
  int splits;      // R splits per z
  int r_chunks;    // ceil(R / kBK)
  float* out;
  long long ldo, out_z_stride, out_split_stride;
  const float* bias0;
  const float* bias1;
  int accumulate;
};

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16x3_kernel(const __grid_constant__ CUtensorMap tm_a_hi, const __grid_constant__ CUtensorMap tm_a_lo,
                       const __grid_constant__ CUtensorMap tm_b_hi, const __grid_constant__ CUtensorMap tm_b_lo,
                       const KArgs p) {
  using C = Cfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * p.n_tile, m0 = blockIdx.y * kBM;
  const int z = blockIdx.z / p.splits, split = blockIdx.z % p.splits;
  const int c_begin = static_cast<int>(static_cast<long long>(split) * p.r_chunks / p.splits);
  const int c_end = static_cast<int>(static_cast<long long>(split + 1) * p.r_chunks / p.splits);
  const int per_seg = c_end - c_begin;
  const int iters = p.S * per_seg;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a_hi);
    tma_prefetch_desc(&tm_a_lo);
    tma_prefetch_desc(&tm_b_hi);
    tma_prefetch_desc(&tm_b_lo);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      for (int it = 0; it < iters; ++it) {
        const int stage = it % STAGES;
        const uint32_t phase = (it / STAGES) & 1;
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st = smem + stage * C::kStageBytes;
        const int s = it / per_seg;
        const int r0 = (c_begin + it % per_seg) * kBK;
        const int aseg = p.a_seg0 + s + p.a_seg_z * z;
        const int bseg = p.b_seg0 + s + p.b_seg_z * z;
        mbar_arrive_expect_tx(&full[stage], p.stage_tx);
        tma_load_3d(st, &tm_a_hi, &full[stage], r0, m0, aseg);
        tma_load_3d(st + C::kABytes, &tm_a_lo, &full[stage], r0, m0, aseg);
        if (EPI == kEpiDx) {
          // N tile = d stacked boxes of n_i rows (feature k = bseg + j)
          const uint32_t box_bytes = static_cast<uint32_t>(p.n_tile) * kRowBytes;
          for (int j = 0; j < p.b_boxes; ++j) {
            tma_load_3d(st + 2 * C::kABytes + j * box_bytes, &tm_b_hi, &full[stage], r0, n0, bseg + j);
            tma_load_3d(st + 2 * C::kABytes + C::kBBytes + j * box_bytes, &tm_b_lo, &full[stage], r0, n0, bseg + j);
          }
        } else {
          tma_load_3d(st + 2 * C::kABytes, &tm_b_hi, &full[stage], r0, n0, bseg);
          tma_load_3d(st + 2 * C::kABytes + C::kBBytes, &tm_b_lo, &full[stage], r0, n0, bseg);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc = umma_idesc_bf16_f32(kBM, p.n_mma);
      for (int it = 0; it < iters; ++it) {
        const int stage = it % STAGES;
        const uint32_t phase = (it / STAGES) & 1;
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a_hi = smem_u32(smem + stage * C::kStageBytes);
        const uint32_t a_lo = a_hi + C::kABytes;
        const uint32_t b_hi = a_hi + 2 * C::kABytes;
        const uint32_t b_lo = b_hi + C::kBBytes;
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          const uint32_t off = kk * 32;  // 16 bf16 = 32 bytes along the swizzled row
          const uint64_t dah = umma_desc_kmajor<kRowBytes>(a_hi + off);
          const uint64_t dal = umma_desc_kmajor<kRowBytes>(a_lo + off);
          const uint64_t dbh = umma_desc_kmajor<kRowBytes>(b_hi + off);
          const uint64_t dbl = umma_desc_kmajor<kRowBytes>(b_lo + off);
          umma_bf16(tmem_base, dah, dbh, idesc, (it | kk) != 0 ? 1u : 0u);
          umma_bf16(tmem_base, dah, dbl, idesc, 1u);
          umma_bf16(tmem_base, dal, dbh, idesc, 1u);
        }
        umma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
      }
      umma_commit(tmem_full);
    }
  } else if (warp >= 4 && EPI == kEpiDx) {
    // ---------------- fused dX epilogue ----------------
    // TMEM column (k-1)*n_i + i holds G_k[row][i0+i] = sum_o dy[row][o] C[k][o][i0+i]
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    const bool row_ok = row < p.M;
    const int n_i = p.n_tile, d = p.b_boxes, K = p.lutK;
    const float* xr = p.x + static_cast<long long>(row) * p.ldo;
    float* dxr = p.dx + static_cast<long long>(row) * p.ldo;
    const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
    for (int ib = 0; ib < n_i; ib += 8) {
      int idx[8];
      double tt[8];
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int i = n0 + ib + e;
        const bool ok = row_ok && i < p.N;
        double fr;
        cell_f64(ok ? xr[i] : 0.0f, p.lutN, idx[e], fr, tt[e]);
        acc[e] = 0.0f;
      }
#pragma unroll 1
      for (int kb = 0; kb < d; kb += 4) {
        uint32_t r[4][8];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (kb + kk < d) tmem_ld_32x32b_x8(tbase + (kb + kk) * n_i + ib, r[kk]);
        tmem_ld_wait();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (kb + kk < d) {
            const int k = kb + kk + 1;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              acc[e] = fmaf(__ldg(p.slopes_pm + static_cast<long long>(idx[e]) * K + k), __uint_as_float(r[kk][e]),
                            acc[e]);
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int i = n0 + ib + e;
        if (row_ok && i < p.N) {
          double v = static_cast<double>(acc[e]);
          if (p.jacobian) v *= 1.0 - tt[e] * tt[e];
          dxr[i] = static_cast<float>(v);
        }
      }
    }
    tc_fence_before();
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    float* out = p.out + static_cast<long long>(z) * p.out_z_stride +
                 static_cast<long long>(split) * p.out_split_stride;
    const bool row_ok = row < p.M;
    float* orow = out + static_cast<long long>(row) * p.ldo;
    const bool vec = ((p.ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + c, r);
      tmem_ld_wait();
      const int nb = n0 + c;
      if (!row_ok || nb >= p.N) continue;
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      if (vec && nb + 32 <= p.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          if (p.bias0) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias0 + nb + j));
            o.x += b.x; o.y += b.y; o.z += b.z; o.w += b.w;
          }
          if (p.bias1) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias1 + nb + j));
            o.x += b.x; o.y += b.y; o.z += b.z; o.w += b.w;
          }
          float4* dst = reinterpret_cast<float4*>(orow + nb + j);
          if (p.accumulate) {
            const float4 prev = *dst;
            o.x += prev.x; o.y += prev.y; o.z += prev.z; o.w += prev.w;
          }
          *dst = o;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = nb + j;
          if (n < p.N) {
            float o = v[j];
            if (p.bias0) o += p.bias0[n];
            if (p.bias1) o += p.bias1[n];
            if (p.accumulate) o += orow[n];
            orow[n] = o;
          }
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// ----------------------------------------------------------------------------
// Host side: tensor maps and launch

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
  });
  return fn;
}

int make_map(CUtensorMap* map, const __nv_bfloat16* base, int64_t R, int64_t rows, int64_t segs, int64_t ld,
             int64_t seg_stride, int box_rows) {
  auto encode = get_encode();
  if (!encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kCudaError;
  }
  CK_CHECK((reinterpret_cast<uintptr_t>(base) & 15) == 0, "gemm operand not 16-byte aligned");
  CK_CHECK(ld % 8 == 0 && seg_stride % 8 == 0, "gemm operand pitch must be a multiple of 8 elements");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(segs)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 2), static_cast<cuuint64_t>(seg_stride * 2)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(base), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with code " + std::to_string(static_cast<int>(r)));
    return kCudaError;
  }
  return kOk;
}

template <int BN, int STAGES, int EPI>
int launch(const GemmProblem& p, int splits, int r_chunks, float* out, long long out_split_stride, int accumulate,
           cudaStream_t s) {
  using C = Cfg<BN, STAGES>;
  const int n_tile = EPI == kEpiDx ? p.dx->n_i : BN;
  const int b_boxes = EPI == kEpiDx ? p.S : 1;
  const int n_mma = n_tile * b_boxes;
  CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
  CK_TRY(make_map(&ta_hi, p.a.hi, p.R, p.a.rows, p.a.segs, p.a.ld, p.a.seg_stride, kBM));
  CK_TRY(make_map(&ta_lo, p.a.lo, p.R, p.a.rows, p.a.segs, p.a.ld, p.a.seg_stride, kBM));
  CK_TRY(make_map(&tb_hi, p.b.hi, p.R, p.b.rows, p.b.segs, p.b.ld, p.b.seg_stride, n_tile));
  CK_TRY(make_map(&tb_lo, p.b.lo, p.R, p.b.rows, p.b.segs, p.b.ld, p.b.seg_stride, n_tile));
  KArgs k{};
  k.n_tile = n_tile;
  k.n_mma = n_mma;
  k.b_boxes = b_boxes;
  k.stage_tx = static_cast<uint32_t>(2 * C::kABytes + 2 * n_mma * kRowBytes);
  if (EPI == kEpiDx) {
    k.x = p.dx->x;
    k.dx = p.dx->dx;
    k.slopes_pm = p.dx->lut.slopes_pm;
    k.lutK = p.dx->lut.K;
    k.lutN = p.dx->lut.N;
    k.jacobian = p.dx->jacobian;
  }
  k.M = static_cast<int>(p.a.rows);
  k.N = static_cast<int>(p.b.rows);
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
  static bool attr_set = false;
  if (!attr_set) {
    CK_CUDA(cudaFuncSetAttribute(gemm_bf16x3_kernel<BN, STAGES, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::kSmemBytes));
    attr_set = true;
  }
  dim3 grid(static_cast<unsigned>(ceil_div(k.N, n_tile)), static_cast<unsigned>(ceil_div(k.M, kBM)),
            static_cast<unsigned>(p.nz * splits));
  LaunchScope scope(p.kclass, s);
  gemm_bf16x3_kernel<BN, STAGES, EPI><<<grid, kThreads, C::kSmemBytes, s>>>(ta_hi, ta_lo, tb_hi, tb_lo, k);
  CK_CUDA(cudaGetLastError());
  return kOk;
}

int choose_splits(int64_t M, int64_t N, int nz, int64_t R, int bn) {
  const int64_t tiles = ceil_div(M, kBM) * ceil_div(N, bn) * nz;
  const int64_t chunks = ceil_div(R, kBK);
  const int64_t sms = num_sms();
  if (tiles >= sms) return 1;
  // enough CTAs for ~2 waves, but keep >= 8 K-chunks per split
  int64_t splits = ceil_div(2 * sms, tiles);
  const int64_t max_splits = chunks / 8 > 1 ? chunks / 8 : 1;
  if (splits > max_splits) splits = max_splits;
  if (splits > 64) splits = 64;
  return static_cast<int>(splits < 1 ? 1 : splits);
}

int pick_bn(int64_t N) { return N <= 128 ? 128 : 256; }

}  // namespace

int64_t gemm_split_ws_elems(int64_t M, int64_t N, int nz, int64_t R) {
  const int splits = choose_splits(M, N, nz, R, pick_bn(N));
  return splits > 1 ? static_cast<int64_t>(splits) * nz * M * N : 0;
}

int dx_tile_inputs(int d) {
  if (d < 1) return 0;
  for (int n_i = (256 / d) / 8 * 8; n_i >= 8; n_i -= 8)
    if ((d * n_i) % 16 == 0 && d * n_i <= 256) return n_i;
  return 0;
}

int gemm_bf16x3(const GemmProblem& p, cudaStream_t s) {
  CK_CHECK(p.S >= 1 && p.nz >= 1 && p.R >= 1, "gemm: empty reduction");
  if (p.dx != nullptr) {
    // fused dX: B = d stacked boxes (S = d features), N = cols of dx
    CK_CHECK(p.nz == 1 && p.dx->n_i == dx_tile_inputs(p.S), "gemm: bad fused-dx configuration");
    const int r_chunks = static_cast<int>(ceil_div(p.R, kBK));
    return launch<256, 2, kEpiDx>(p, 1, r_chunks, nullptr, 0, 0, s);
  }
  CK_CHECK(p.a.rows >= 1 && p.b.rows >= 1, "gemm: empty output");
  CK_CHECK(p.a.rows < (1ll << 31) && p.b.rows < (1ll << 31), "gemm: extent too large");
  const int bn = pick_bn(p.b.rows);
  const int r_chunks = static_cast<int>(ceil_div(p.R, kBK));
  int splits = choose_splits(p.a.rows, p.b.rows, p.nz, p.R, bn);
  const int64_t need = static_cast<int64_t>(splits) * p.nz * p.a.rows * p.b.rows;
  if (splits > 1 && (p.split_ws == nullptr || p.split_ws_elems < need)) splits = 1;
  const bool dense_out = p.ldo == p.b.rows && p.out_z_stride == p.a.rows * p.b.rows;
  if (splits > 1 && !dense_out) splits = 1;

  float* out = p.out;
  long long split_stride = 0;
  int acc = p.accumulate;
  if (splits > 1) {
    // stage 1: per-split partial tiles (unique writer per slot), then a
    // fixed-order merge (stage 2) -- the two-stage reduction.
    out = p.split_ws;
    split_stride = p.nz * p.a.rows * p.b.rows;
    acc = 0;
  }
  GemmProblem q = p;
  // partial slot layout: [split][z][M][N]; the kernel offsets by split first
  int rc;
  if (bn == 128) {
    rc = launch<128, 3, kEpiStore>(q, splits, r_chunks, out, split_stride, acc, s);
  } else {
    rc = launch<256, 2, kEpiStore>(q, splits, r_chunks, out, split_stride, acc, s);
  }
  if (rc != kOk) return rc;
  if (splits > 1) {
    CK_TRY(launch_merge(p.split_ws, splits, split_stride, split_stride, p.out, p.accumulate, s));
    if (p.bias0 || p.bias1) {
      CK_TRY(launch_add_rows(p.out, p.nz * p.a.rows, p.b.rows, p.bias0, p.bias1, s));
    }
  }
  return kOk;
}

}  // namespace ck
