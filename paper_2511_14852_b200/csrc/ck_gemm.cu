// tcgen05 split-precision (BF16x3) GEMM for the ChebyKAN contractions:
// host-side tensor maps, configuration choice and dispatch.  The kernel
// itself is in ck_gemm_impl.cuh; the exact-mode input-gradient variants are
// instantiated in ck_gemm_dx_exact.cu (compiled in parallel).
#include <mutex>

#include "ck_gemm_impl.cuh"

namespace ck {
namespace {

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

}  // namespace

int make_map(CUtensorMap* map, const __nv_bfloat16* base, int64_t R, int64_t rows, int64_t segs, int64_t ld,
             int64_t seg_stride, int box_rows, int bk, int mn_major) {
  auto encode = get_encode();
  if (!encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kCudaError;
  }
  CK_CHECK((reinterpret_cast<uintptr_t>(base) & 15) == 0, "gemm operand not 16-byte aligned");
  CK_CHECK(ld % 8 == 0 && seg_stride % 8 == 0, "gemm operand pitch must be a multiple of 8 elements");
  // K-major: dims (K, rows, segs), box (bk, box_rows).  MN-major: dims
  // (rows, K, segs), box (64 MN elements = one 128-byte swizzle row, bk K-rows).
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(mn_major ? rows : R), static_cast<cuuint64_t>(mn_major ? R : rows),
                        static_cast<cuuint64_t>(segs)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 2), static_cast<cuuint64_t>(seg_stride * 2)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(mn_major ? 64 : bk), static_cast<cuuint32_t>(mn_major ? bk : box_rows),
                       1};
  cuuint32_t estr[3] = {1, 1, 1};
  // L2 promotion of the TMA requests (CK_TMA_PROMO = 0 none, 1 64B, 2 128B, 3 256B; default 256B)
  static const CUtensorMapL2promotion promo = [] {
    const char* e = getenv("CK_TMA_PROMO");
    const int v = e ? atoi(e) : 3;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                  : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                           : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(base), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                      promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with code " + std::to_string(static_cast<int>(r)));
    return kCudaError;
  }
  return kOk;
}

// Output map of the TMA-store epilogue (see store_chunk_tma).  The copy
// engine needs 16-byte aligned base and pitches; other layouts keep the
// per-thread stores.
int make_out_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t planes, int64_t ld,
                 int64_t plane_stride) {
  auto encode = get_encode();
  if (!encode || (reinterpret_cast<uintptr_t>(base) & 15) != 0 || ld % 4 != 0 || plane_stride % 4 != 0 ||
      rows < 1 || cols < 1 || planes < 1)
    return kUnsupported;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(planes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 4), static_cast<cuuint64_t>(plane_stride * 4)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? kOk : kUnsupported;
}

// CK_TMA_STORE=0: the store epilogue uses per-thread coalesced stores (A/B)
bool tma_store_enabled() {
  static const bool on = [] {
    const char* e = getenv("CK_TMA_STORE");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

namespace {

int gemm_bk() {
  static int bk = [] {
    const char* e = getenv("CK_GEMM_BK");
    return (e && std::string(e) == "32") ? 32 : 64;
  }();
  return bk;
}

}  // namespace

// Rasterisation group size (m-tiles per group) for a problem with m_tiles
// rows of tiles; CK_GEMM_GROUP overrides.  16 for tall problems (>= 128
// m-tiles: the C4 chunks of 32768 rows): the C4 training step went 517-523k
// -> 542-547k samples/s against 8 (eight interleaved runs on one box,
// profiles/r02_session3.md) -- the same work per clock at ~5 % higher
// power-capped clocks, ~9 % less L2->SM traffic for the forward and dC GEMMs
// (ncu).  8 below that (the 16384-row C1 layers: 8 measured 0.3-1.5 % faster).
int gemm_group(int m_tiles) {
  static int g = [] {
    const char* e = getenv("CK_GEMM_GROUP");
    const int v = e ? atoi(e) : 0;
    return v >= 1 && v <= 1024 ? v : 0;
  }();
  return g > 0 ? g : (m_tiles >= 128 ? 16 : 8);
}

int gemm_pace() {
  static int v = [] {
    const char* e = getenv("CK_GEMM_PACE");
    const int n = e ? atoi(e) : 0;
    return n > 0 ? n : 0;
  }();
  return v;
}

uint32_t next_pace_tag() {
  static std::atomic<uint32_t> tag{0};
  return tag.fetch_add(1) + 1;  // never 0 (the zero-initialised table)
}

int gemm_seg() {
  static int v = [] {
    const char* e = getenv("CK_GEMM_SEG");
    const int n = e ? atoi(e) : kSegIters;
    return n >= 0 ? n : kSegIters;
  }();
  return v;
}

namespace {

// LUT-mode fused dX: chord slopes recomputed in the epilogue (1, default for
// the three-term families) or gathered from the dX rows (CK_DX_CHORD=0).
int dx_chord() {
  static int v = [] {
    const char* e = getenv("CK_DX_CHORD");
    return (e && std::string(e) == "0") ? 0 : 1;
  }();
  return v;
}

bool chord_kind(int kind) { return kind == kCheb || kind == kLegendre || kind == kHermite; }

// CTA group for the GEMMs: 2 (SM pairs, default) or 1 (CK_GEMM_CG=1).
int gemm_cg() {
  static int cg = [] {
    const char* e = getenv("CK_GEMM_CG");
    return (e && std::string(e) == "1") ? 1 : 2;
  }();
  return cg;
}

// Store-GEMM tile configuration: the tile capacity BN and the CTA group.
// N <= 128: single-CTA 128x128 tiles; otherwise 256-wide tiles on CTA pairs.
// (128-wide pair tiles would fill partial waves better at some shapes, but
// measured 5-12 % slower: twice the A-operand traffic per MMA.)
struct StoreCfg {
  int bn, cg;
};

StoreCfg pick_store(int64_t N) { return N <= 128 ? StoreCfg{128, 1} : StoreCfg{256, gemm_cg()}; }

// Split-R factor for a store GEMM, from a cost model in units of one
// pipeline iteration of one tile (~0.8 us x n_tile/256 on a CTA pair):
// rounds of the persistent schedule x iterations per split, plus the
// fixed-order merge of the partials (read s, write 1 output at ~4 TB/s, and
// a launch).  Splitting fills partial waves: 80 dC tiles on 74 SM pairs
// (1024^2, d5) ran as two rounds, the second 8 % full; 8 splits run 9 rounds
// of 1/8 the length.  >= 4 K blocks per split, <= 64 splits, partials
// <= 1.5 GB.
int choose_splits(int64_t M, int64_t N, int nz, int64_t kchunks, const StoreCfg& c, bool mn_major) {
  const int nt = store_ntile(N, c.bn, c.cg, mn_major);
  const int64_t tiles = ceil_div(M, static_cast<int64_t>(kBM) * c.cg) * ceil_div(N, nt) * nz;
  const int64_t units = num_sms() / c.cg;
  const int64_t chunks = kchunks;  // 64-wide K chunks over all segments
  const double t_it = 0.8e-6 * nt / 256.0 * (c.cg == 2 ? 1.0 : 0.5);
  const double out_bytes = 4.0 * static_cast<double>(nz) * static_cast<double>(M) * static_cast<double>(N);
  int64_t max_splits = chunks / 4 > 1 ? chunks / 4 : 1;
  if (max_splits > 64) max_splits = 64;
  double best = static_cast<double>(ceil_div(tiles, units) * chunks);
  int best_s = 1;
  for (int64_t s = 2; s <= max_splits; ++s) {
    if (s * out_bytes > 1.5e9) break;
    const double work = static_cast<double>(ceil_div(tiles * s, units) * ceil_div(chunks, s));
    const double merge = ((s + 1) * out_bytes / 4e12 + 4e-6) / t_it;
    if (work + merge < 0.97 * best) {
      best = work + merge;
      best_s = static_cast<int>(s);
    }
  }
  return best_s;
}

}  // namespace

// CK_GEMM_SPLITS=s forces s reduction splits on every store GEMM whose
// workspace allows it (accuracy / traffic experiments; 0 = cost model).
int forced_splits() {
  static int v = [] {
    const char* e = getenv("CK_GEMM_SPLITS");
    const int s = e ? atoi(e) : 0;
    return s >= 1 && s <= 64 ? s : 0;
  }();
  return v;
}

int64_t gemm_split_ws_elems(int64_t M, int64_t N, int nz, int64_t kchunks) {
  // the larger of the two operand majornesses' choices (the workspace is
  // sized before the caller knows which GEMM runs)
  int splits = forced_splits() > 0 ? forced_splits() : 1;
  for (bool mn : {false, true}) {
    const int sp = choose_splits(M, N, nz, kchunks, pick_store(N), mn);
    if (sp > splits) splits = sp;
  }
  return splits > 1 ? static_cast<int64_t>(splits) * nz * M * N : 0;
}

int64_t gemm_store_padded(int64_t M, int64_t N, bool mn_major) {
  const StoreCfg c = pick_store(N);
  const int nt = store_ntile(N, c.bn, c.cg, mn_major);
  return ceil_div(M, static_cast<int64_t>(kBM) * c.cg) * kBM * c.cg * (ceil_div(N, nt) * nt);
}

// Inputs per stacked dX tile: a multiple of 8 with d * n_i <= 256 (one MMA,
// a multiple of 16) chosen for the layer width -- the fewest padded columns
// plus a per-tile overhead of 8 columns (I = 256, d = 3: 4 tiles of 64, not
// 4 x 80 with a 16-wide last tile; I = 512, d = 5: 11 x 48).
int dx_tile_inputs(int d, int64_t I) {
  if (d < 1 || d > kMaxDFused) return 0;
  int best = 0;
  int64_t best_cost = 0;
  for (int n_i = (256 / d) / 8 * 8; n_i >= 8; n_i -= 8) {
    if ((d * n_i) % 16 != 0 || d * n_i > 256) continue;
    const int64_t cost = ceil_div(I, n_i) * (n_i + 8);
    if (best == 0 || cost < best_cost) {
      best = n_i;
      best_cost = cost;
    }
  }
  return best;
}

int gemm_bf16x3(const GemmProblem& p, cudaStream_t s) {
  CK_CHECK(p.S >= 1 && p.nz >= 1 && p.R >= 1, "gemm: empty reduction");
  if (p.dx != nullptr) {
    // fused dX: B = d stacked boxes (S = d features), N = cols of dx
    CK_CHECK(p.nz == 1 && p.dx->n_i == dx_tile_inputs(p.S, p.dx->cols), "gemm: bad fused-dx configuration");
    if (p.dx->lut.exact) return launch_dx_exact(p, s);
    const bool bk64 = gemm_bk() == 64;
    if (dx_chord() && bk64 && gemm_cg() == 2 && chord_kind(p.dx->lut.kind)) return launch_dx_chord(p, s);
    if (gemm_cg() == 2)
      return bk64 ? launch<256, 64, 3, kEpiDx, 2>(p, 1, nullptr, 0, 0, s)
                  : launch<256, 32, 6, kEpiDx, 2>(p, 1, nullptr, 0, 0, s);
    return bk64 ? launch<256, 64, 2, kEpiDx, 1>(p, 1, nullptr, 0, 0, s)
                : launch<256, 32, 4, kEpiDx, 1>(p, 1, nullptr, 0, 0, s);
  }
  CK_CHECK(p.a.rows >= 1 && p.b.rows >= 1, "gemm: empty output");
  CK_CHECK(p.a.rows < (1ll << 31) && p.b.rows < (1ll << 31), "gemm: extent too large");
  const bool mn = p.a.mn_major || p.b.mn_major;
  const StoreCfg cfg = pick_store(p.b.rows);
  int splits = choose_splits(p.a.rows, p.b.rows, p.nz, p.S * ceil_div(p.R, 64), cfg, mn);
  if (forced_splits() > 0) splits = forced_splits();  // experiments (CK_GEMM_SPLITS)
  const int64_t need = static_cast<int64_t>(splits) * p.nz * p.a.rows * p.b.rows;
  if (splits > 1 && (p.split_ws == nullptr || p.split_ws_elems < need)) splits = 1;
  const bool dense_out = p.ldo == (p.out_trans ? p.a.rows : p.b.rows) && p.out_z_stride == p.a.rows * p.b.rows;
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
  const bool bk64 = gemm_bk() == 64;
  if (mn) {
    CK_CHECK(p.a.mn_major && p.b.mn_major, "gemm: mixed-majorness store GEMM not instantiated");
    if (cfg.bn == 128) {
      rc = launch<128, 64, 3, kEpiStore, 1, 1, 1>(q, splits, out, split_stride, acc, s);
    } else if (cfg.cg == 2) {
      rc = launch<256, 64, 3, kEpiStore, 2, 1, 1>(q, splits, out, split_stride, acc, s);
    } else {
      rc = launch<256, 64, 2, kEpiStore, 1, 1, 1>(q, splits, out, split_stride, acc, s);
    }
  } else if (cfg.bn == 128) {
    rc = bk64 ? launch<128, 64, 3, kEpiStore, 1>(q, splits, out, split_stride, acc, s)
              : launch<128, 32, 6, kEpiStore, 1>(q, splits, out, split_stride, acc, s);
  } else if (cfg.cg == 2) {
    rc = bk64 ? launch<256, 64, 3, kEpiStore, 2>(q, splits, out, split_stride, acc, s)
              : launch<256, 32, 6, kEpiStore, 2>(q, splits, out, split_stride, acc, s);
  } else {
    rc = bk64 ? launch<256, 64, 2, kEpiStore, 1>(q, splits, out, split_stride, acc, s)
              : launch<256, 32, 4, kEpiStore, 1>(q, splits, out, split_stride, acc, s);
  }
  if (rc != kOk) return rc;
  if (splits > 1) {
    const bool bias = p.bias0 || p.bias1;
    CK_TRY(launch_merge(p.split_ws, splits, split_stride, split_stride, p.out, p.accumulate, s, bias ? nullptr : p.fin));
    if (bias) {
      CK_TRY(launch_add_rows(p.out, p.nz * p.a.rows, p.b.rows, p.bias0, p.bias1, s));
    }
    if (bias && p.fin) {
      CK_TRY(launch_col_finish(p.fin->part, p.fin->slots, p.fin->cols, p.fin->out, s, p.fin->bcast, p.fin->bcast_cols));
    }
  } else if (p.fin) {
    CK_TRY(launch_col_finish(p.fin->part, p.fin->slots, p.fin->cols, p.fin->out, s, p.fin->bcast, p.fin->bcast_cols));
  }
  return kOk;
}

}  // namespace ck

// Timeline of the last GEMM launch (CK_GEMM_TRACE builds; 0 = not built in).
extern "C" int ck_debug_gemm_trace(unsigned long long* out, int max_ctas) {
#ifdef CK_GEMM_TRACE
  const int n = max_ctas < 512 ? max_ctas : 512;
  CK_CUDA(cudaMemcpyFromSymbol(out, ck::g_gemm_trace, sizeof(unsigned long long) * ck::kTraceEvents * n));
  return n;
#else
  (void)out;
  (void)max_ctas;
  return 0;
#endif
}
