// Forward contraction with the basis generated on the fly into shared memory
// (kernel templates; instantiated per basis family in ck_gemm_gen_k*.cu)
// (the north star's subsystem (2)): y = Φ(x)·Cᵀ + bias + c0sum without the
// Φ planes ever reaching HBM.
//
// The reduction axis is input-major: the 64-wide K chunk j holds G = 64/d
// whole inputs i = jG + g, feature k at position g*d + (k-1), zero padding
// after G*d.  The coefficient operand is prepared once in that order
// (launch_gen_coeff: [O][chunks*64] bf16 hi/lo, "reordered unit-stride
// tiles") and TMA-staged; the A operand of each pipeline stage is written by
// sixteen generator warps straight into the SWIZZLE_128B K-major layout the
// tensor core reads: thread (row, quarter) evaluates elem_planes for the
// inputs covering its 16 positions (the LUT path recomputes the two bracketing table
// entries at the grid nodes, exactly as the expansion kernels), splits the
// values into bf16 hi/lo and stores two 16-byte chunks of each.
//
// Pays off when the output is narrow (d_out <= 256: one N tile, so every
// element is generated once): the materialised path writes and re-reads
// 4*d bytes of planes per element, this one reads x (4 bytes).  Wider
// outputs would regenerate the tile once per N tile.
//
// Warp roles (768 threads, CTA pairs): warp 0 TMA producer (coefficients),
// warp 1 MMA issuer (leader CTA), warp 2 TMEM allocator, warps 4..7 store
// epilogue, warps 8..23 generators (four per K quarter).
#pragma once
#include "ck_gemm_impl.cuh"

namespace ck {
namespace {

constexpr int kGenThreads = 768;
constexpr int kGenWarps = 16;
constexpr int kGenEpiWarps = 4;
constexpr int kGenMaxD = 16;

// Generator thread = (row, quarter Q): the 16 K positions [16Q, 16Q+16) of
// one row of each stage chunk j -- the inputs covering them (g_lo..g_hi),
// evaluated, split, stored as 2 x 16 bytes (hi) + 2 x 16 (lo).
template <int D, int Q>
struct GenQuarter {
  static constexpr int G = 64 / D;  // inputs per chunk
  static constexpr int P0 = 16 * Q;
  static constexpr int g_lo = P0 / D;
  static constexpr int g_hi = (P0 + 15) / D < G - 1 ? (P0 + 15) / D : G - 1;
  static constexpr int NX = g_hi >= g_lo ? g_hi - g_lo + 1 : 1;
};

template <int D, int Q>
__device__ __forceinline__ void gen_load_x(const float* xr, bool row_ok, int i_base, int I,
                                           float (&xv)[GenQuarter<D, Q>::NX]) {
  using GQ = GenQuarter<D, Q>;
#pragma unroll
  for (int g = 0; g < GQ::NX; ++g) {
    const int i = i_base + GQ::g_lo + g;
    xv[g] = (row_ok && i < I && GQ::g_lo + g <= GQ::g_hi) ? __ldg(xr + i) : 0.0f;
  }
}

template <int SRC, int KIND, int D, int Q>
__device__ __forceinline__ void gen_store(const float (&xv)[GenQuarter<D, Q>::NX], int lut_n, uint32_t row,
                                          uint8_t* a_hi, uint8_t* a_lo) {
  using GQ = GenQuarter<D, Q>;
  float vals[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) vals[p] = 0.0f;
  if constexpr (GQ::g_lo <= GQ::g_hi) {
#pragma unroll
    for (int g = GQ::g_lo; g <= GQ::g_hi; ++g) {
      float v[D];
      elem_planes<SRC, KIND, D>(xv[g - GQ::g_lo], lut_n, v);
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const int p = g * D + k - GQ::P0;
        if (p >= 0 && p < 16) vals[p] = v[k];
      }
    }
  }
  uint32_t hw[8], lw[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) split_pack2(vals[2 * j], vals[2 * j + 1], hw[j], lw[j]);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const uint32_t off = row * 128u + ((((2u * Q + c) ^ (row & 7u)) & 7u) << 4);
    *reinterpret_cast<uint4*>(a_hi + off) = make_uint4(hw[4 * c], hw[4 * c + 1], hw[4 * c + 2], hw[4 * c + 3]);
    *reinterpret_cast<uint4*>(a_lo + off) = make_uint4(lw[4 * c], lw[4 * c + 1], lw[4 * c + 2], lw[4 * c + 3]);
  }
}

// All stages of all tiles of this CTA for one generator warp; the next
// stage's x is loaded while the current one is evaluated.
template <int SRC, int KIND, int D, int Q, int STAGES, int STAGE_BYTES, int A_BYTES>
__device__ __forceinline__ void gen_loop(const KArgs& p, uint8_t* smem, uint64_t* full, uint64_t* empty,
                                         uint64_t* ready, int unit, int n_units, int row_off, uint32_t lrow,
                                         int lane) {
  constexpr int G = 64 / D;
  uint32_t g = 0;
  for (int t = unit; t < p.total_tiles; t += n_units) {
    const TileCoord tc = decode_tile(p, t, kBM * 2);
    const int row = tc.m0 + row_off + static_cast<int>(lrow);
    const bool row_ok = row < p.M;
    const float* xr = p.x + static_cast<long long>(row_ok ? row : 0) * p.gen_ldx;
    // x of stages it and it+1 in registers; stage it+2's loads are issued
    // after stage it is handed over, a full stage ahead of their use
    float xv[GenQuarter<D, Q>::NX], xn[GenQuarter<D, Q>::NX];
    gen_load_x<D, Q>(xr, row_ok, 0, p.gen_I, xv);
    if (tc.iters > 1) gen_load_x<D, Q>(xr, row_ok, G, p.gen_I, xn);
    for (int it = 0; it < tc.iters; ++it, ++g) {
      const int stage = g % STAGES;
      mbar_wait(&empty[stage], ((g / STAGES) & 1) ^ 1);
      uint8_t* st = smem + stage * STAGE_BYTES;
      gen_store<SRC, KIND, D, Q>(xv, p.lutN, lrow, st, st + A_BYTES);
      fence_proxy_async_smem();  // generic-proxy stores -> tensor-core reads
      __syncwarp();
      // leader CTA: straight onto the MMA's barrier; peer CTA: onto a local
      // barrier its signaller warp forwards (a remote release arrive costs a
      // GPU-scope membar, ~0.6 us, which must stay off the generators' path)
      if (lane == 0) mbar_arrive(row_off == 0 ? &full[stage] : &ready[stage]);
#pragma unroll
      for (int e = 0; e < GenQuarter<D, Q>::NX; ++e) xv[e] = xn[e];
      if (it + 2 < tc.iters) gen_load_x<D, Q>(xr, row_ok, (it + 2) * G, p.gen_I, xn);
    }
  }
}

template <int SRC, int KIND, int D>
__global__ void __launch_bounds__(kGenThreads, 1)
    gemm_gen_kernel(const __grid_constant__ CUtensorMap tm_b_hi, const __grid_constant__ CUtensorMap tm_b_lo,
                    const KArgs p) {
  constexpr int BN = 256, BK = 64, STAGES = 3, CG = 2;
  using C = Cfg<BN, BK, STAGES, CG>;
  constexpr int kRowBytes = C::kRowBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ready = tempty + 2;  // [STAGES] peer CTA: its generators done (-> signaller)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ready + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = p.total_tiles;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int unit = blockIdx.x / CG, n_units = gridDim.x / CG;
  const int row_off = static_cast<int>(rank) * kBM;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_b_hi);
    tma_prefetch_desc(&tm_b_lo);
    for (int s = 0; s < STAGES; ++s) {
      // the leader's barrier completes on its TMA bytes, its own generator
      // warps and the peer CTA's signaller
      mbar_init(&full[s], 1 + kGenWarps + 1);
      mbar_init(&empty[s], 1);
      mbar_init(&ready[s], kGenWarps);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG * kGenEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, C::kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: coefficient tiles ----------------
      uint32_t g = 0;
      const int b_half = p.n_mma / CG;
      for (int t = unit; t < total; t += n_units) {
        const TileCoord tc = decode_tile(p, t, kBM * CG);
        for (int it = 0; it < tc.iters; ++it, ++g) {
          const int stage = g % STAGES;
          mbar_wait(&empty[stage], ((g / STAGES) & 1) ^ 1);
          uint8_t* st = smem + stage * C::kStageBytes;
          if (leader) mbar_arrive_expect_tx(&full[stage], p.stage_tx);
          const int brow = tc.n0 + static_cast<int>(rank) * b_half;
          tma_load_3d_pair(st + 2 * C::kABytes, &tm_b_hi, &full[stage], it * BK, brow, 0);
          tma_load_3d_pair(st + 2 * C::kABytes + C::kBBytes, &tm_b_lo, &full[stage], it * BK, brow, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc = umma_idesc_bf16_f32(kBM * CG, p.n_mma);
      uint32_t g = 0, lt = 0;
      for (int t = unit; t < total; t += n_units, ++lt) {
        const TileCoord tc = decode_tile(p, t, kBM * CG);
        const uint32_t acc = lt & 1, use = lt >> 1;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int it = 0; it < tc.iters; ++it, ++g) {
          const int stage = g % STAGES;
          mbar_wait(&full[stage], (g / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_hi = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t a_lo = a_hi + C::kABytes;
          const uint32_t b_hi = a_hi + 2 * C::kABytes;
          const uint32_t b_lo = b_hi + C::kBBytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t dah = umma_desc_kmajor<kRowBytes>(a_hi + kk * 32);
            const uint64_t dal = umma_desc_kmajor<kRowBytes>(a_lo + kk * 32);
            const uint64_t dbh = umma_desc_kmajor<kRowBytes>(b_hi + kk * 32);
            const uint64_t dbl = umma_desc_kmajor<kRowBytes>(b_lo + kk * 32);
            umma_bf16_pair<kCollector>(d_tmem, dah, dbh, idesc, (it | kk) != 0 ? 1u : 0u);
            umma_bf16_pair<kCollector ? 2 : 0>(d_tmem, dah, dbl, idesc, 1u);
            umma_bf16_pair(d_tmem, dal, dbh, idesc, 1u);
          }
          umma_commit_pair(&empty[stage]);
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp == 3) {
    if (lane == 0 && !leader) {
      // ---------------- signaller (peer CTA): generators done -> leader ----------------
      uint32_t g = 0;
      for (int t = unit; t < total; t += n_units) {
        const TileCoord tc = decode_tile(p, t, kBM * CG);
        for (int it = 0; it < tc.iters; ++it, ++g) {
          const int stage = g % STAGES;
          mbar_wait(&ready[stage], (g / STAGES) & 1);
          mbar_arrive_cluster(&full[stage], 0);
        }
      }
    }
  } else if (warp >= 4 && warp < 4 + kGenEpiWarps) {
    // ---------------- store epilogue: y = acc + bias + c0sum ----------------
    const int q = warp & 3;
    uint32_t lt = 0;
    for (int t = unit; t < total; t += n_units, ++lt) {
      const TileCoord tc = decode_tile(p, t, kBM * CG);
      const uint32_t acc = lt & 1, use = lt >> 1;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      const int row = tc.m0 + row_off + q * 32 + lane;
      const bool vec = ((p.ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.out) & 15) == 0);
      float* tile = reinterpret_cast<float*>(smem + STAGES * C::kStageBytes + C::kBarrierBytes) +
                    q * (kEpiTileBytes / 4);
#pragma unroll 1
      for (int c = 0; c < p.n_tile; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tbase + c, r);
        tmem_ld_wait();
        const int nb = tc.n0 + c;
        if (nb >= p.N) continue;
        store_chunk_coalesced(r, tile, lane, row - lane, p.M, nb, p.N, p.out, p.ldo, p.bias0, p.bias1, 0, vec);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
    }
  } else if (warp >= 8) {
    // ---------------- generators: the A operand of every stage ----------------
    const int gw = warp - 8;
    const uint32_t lrow = static_cast<uint32_t>((gw & 3) * 32 + lane);  // row inside this CTA's 128
    constexpr int SB = C::kStageBytes, AB = C::kABytes;
    switch (gw >> 2) {  // quarter of the 64 K positions (warp-uniform)
      case 0:
        gen_loop<SRC, KIND, D, 0, STAGES, SB, AB>(p, smem, full, empty, ready, unit, n_units, row_off, lrow, lane);
        break;
      case 1:
        gen_loop<SRC, KIND, D, 1, STAGES, SB, AB>(p, smem, full, empty, ready, unit, n_units, row_off, lrow, lane);
        break;
      case 2:
        gen_loop<SRC, KIND, D, 2, STAGES, SB, AB>(p, smem, full, empty, ready, unit, n_units, row_off, lrow, lane);
        break;
      default:
        gen_loop<SRC, KIND, D, 3, STAGES, SB, AB>(p, smem, full, empty, ready, unit, n_units, row_off, lrow, lane);
        break;
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::kTmemCols);
  }
}

template <int SRC, int KIND, int D>
int launch_gen_kernel(const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo, int grid,
                      cudaStream_t s) {
  using C = Cfg<256, 64, 3, 2>;
  constexpr int kSmem = C::kSmemBytes + kGenEpiWarps * kEpiTileBytes;
  auto kernel = gemm_gen_kernel<SRC, KIND, D>;
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  CK_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
    CK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr_set.fetch_or(bit);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kGenThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = 2;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  CK_CUDA(cudaLaunchKernelEx(&cfg, kernel, tb_hi, tb_lo, k));
  return kOk;
}

template <int SRC, int KIND>
int launch_gen_kind(int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo, int grid,
                    cudaStream_t s) {
#define CK_GEN_CASE(D)                                                      \
  case D:                                                                   \
    if constexpr (KIND != kFourier || D % 2 == 0) {                         \
      return launch_gen_kernel<SRC, KIND, D>(k, tb_hi, tb_lo, grid, s);     \
    } else {                                                                \
      return kUnsupported;                                                  \
    }
  switch (d) {
    CK_GEN_CASE(1) CK_GEN_CASE(2) CK_GEN_CASE(3) CK_GEN_CASE(4) CK_GEN_CASE(5) CK_GEN_CASE(6) CK_GEN_CASE(7)
    CK_GEN_CASE(8) CK_GEN_CASE(9) CK_GEN_CASE(10) CK_GEN_CASE(11) CK_GEN_CASE(12) CK_GEN_CASE(13) CK_GEN_CASE(14)
    CK_GEN_CASE(15) CK_GEN_CASE(16)
    default:
      return kUnsupported;
  }
#undef CK_GEN_CASE
}

}  // namespace

// Per-family launchers (one translation unit each, compiled in parallel).
int launch_gen_cheb(int exact, int trig, int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo,
                     int grid, cudaStream_t s);
int launch_gen_legendre(int exact, int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo,
                         int grid, cudaStream_t s);
int launch_gen_hermite(int exact, int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo,
                        int grid, cudaStream_t s);
int launch_gen_fourier(int exact, int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo,
                        int grid, cudaStream_t s);

}  // namespace ck
