// extern "C" entry points (include/chebykan.h): argument validation with
// the reference's error wording, workspace carving, and the orchestration of
// the forward / backward kernels on the caller's stream.
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {

namespace {
thread_local std::string g_error;

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// Opaque coefficient-prep buffer: a PrepHeader slot; bf16 hi/lo DOJ
// [K][O][ldI] (forward B operand); the input-gradient B operand, either
// "stacked" -- rows (i-tile, k, i) so one TMA box feeds a d x n_i N tile --
// or plain DJO [K][I][ldO] when the degree is too large to stack; and
// c0sum[O].  Skinny layers keep only an fp32 DOJ copy after the header.
struct PrepLayout {
  int64_t ldI, ldO;
  int n_i;             // inputs per stacked tile (0: DJO layout)
  int64_t dxb_rows;    // rows of the input-gradient operand
  bool skinny;         // d_out <= 8: only an fp32 DOJ copy (at f32)
  bool gen;            // narrow output: + the generated forward's coefficient copy
  int64_t gen_elems;   // O * gen_chunks * 64 per hi / lo
  size_t hdr, f32, doj_hi, doj_lo, dxb_hi, dxb_lo, c0sum, gen_hi, gen_lo, total;
  PrepLayout(int I, int O, int K) {
    skinny = skinny_layer(I, O, K);
    gen = false;
    gen_elems = 0;
    gen_hi = gen_lo = 0;
    hdr = 0;
    f32 = 0;
    if (skinny) {
      ldI = I;
      ldO = O;
      n_i = 0;
      dxb_rows = 0;
      doj_hi = doj_lo = dxb_hi = dxb_lo = c0sum = 0;
      f32 = kAlign;
      total = f32 + align_up(sizeof(float) * K * O * static_cast<size_t>(I));
      return;
    }
    ldI = round_up(I, 8);
    ldO = round_up(O, 8);
    const int d = K - 1;
    n_i = dx_tile_inputs(d, I);
    dxb_rows = n_i > 0 ? ceil_div(I, n_i) * d * n_i : static_cast<int64_t>(K) * I;
    const size_t doj = align_up(sizeof(__nv_bfloat16) * K * O * ldI);
    const size_t dxb = align_up(sizeof(__nv_bfloat16) * dxb_rows * ldO);
    doj_hi = kAlign;
    doj_lo = doj_hi + doj;
    dxb_hi = doj_lo + doj;
    dxb_lo = dxb_hi + dxb;
    c0sum = dxb_lo + dxb;
    total = c0sum + align_up(sizeof(float) * O);
    gen = gen_layer(I, O, K);
    if (gen) {
      gen_elems = static_cast<int64_t>(O) * gen_chunks(I, d) * 64;
      gen_hi = total;
      gen_lo = gen_hi + align_up(sizeof(__nv_bfloat16) * gen_elems);
      total = gen_lo + align_up(sizeof(__nv_bfloat16) * gen_elems);
    }
  }
};

// Host-side record of every prep buffer ck_coeff_prepare has filled: device
// address -> (I, O, K).  ck_forward / ck_backward reject a buffer prepared
// for another layer shape (or never prepared) before any kernel reads it.
struct PrepShape {
  int d_in, d_out, n_feat;
};
std::mutex g_prep_mu;
std::unordered_map<uintptr_t, PrepShape> g_preps;

int check_prep(const void* prep, size_t prep_bytes, int d_in, int d_out, int n_feat) {
  CK_CHECK(prep != nullptr, "coefficient prep is NULL");
  const size_t need = PrepLayout(d_in, d_out, n_feat).total + kAlign;
  if (prep_bytes < need) {
    set_error("coefficient prep buffer too small: " + std::to_string(prep_bytes) + " bytes, the layer needs " +
              std::to_string(need));
    return kInvalidArgument;
  }
  std::lock_guard<std::mutex> lk(g_prep_mu);
  auto it = g_preps.find(reinterpret_cast<uintptr_t>(prep));
  if (it == g_preps.end()) {
    set_error("coefficient prep buffer was not filled by ck_coeff_prepare");
    return kInvalidArgument;
  }
  const PrepShape& p = it->second;
  if (p.d_in != d_in || p.d_out != d_out || p.n_feat != n_feat) {
    set_error("coefficient prep was prepared for (d_in, d_out, n_feat) = (" + std::to_string(p.d_in) + ", " +
              std::to_string(p.d_out) + ", " + std::to_string(p.n_feat) + "), not (" + std::to_string(d_in) + ", " +
              std::to_string(d_out) + ", " + std::to_string(n_feat) + ")");
    return kInvalidArgument;
  }
  return kOk;
}

std::atomic<int64_t> g_chunk_rows{[] {
  const char* e = getenv("CK_CHUNK_ROWS");
  const long long v = e ? atoll(e) : 0;
  return static_cast<int64_t>(v >= 1 ? v : kChunkRowsDefault);
}()};

// Basis planes of one chunk: Φ_k hi/lo for k = 1..d, [d][chunk][ldI] bf16.
// The forward writes them; the backward's dC GEMM reads them as its MN-major
// B operand.  With a caller-provided cache the planes of every chunk persist
// from forward to backward (no re-expansion); else they live in workspace.
struct BasisLayout {
  int64_t chunk, n_chunks, ldI, plane;
  size_t half, per_chunk, total;
  BasisLayout(int64_t B, int I, int K) {
    const int64_t cr = chunk_rows();
    chunk = B < cr ? B : cr;
    if (chunk < 1) chunk = 1;
    n_chunks = ceil_div(B > 0 ? B : 1, chunk);
    ldI = round_up(I, 16);  // 32-byte rows: whole-sector plane stores (I = 257: 2.5 -> 4.8 TB/s)
    plane = chunk * ldI;
    const int d = K - 1;
    half = align_up(sizeof(__nv_bfloat16) * (d > 0 ? d : 0) * plane);
    per_chunk = 2 * half;
    total = per_chunk * n_chunks + kAlign;
  }
};

struct FwdLayout {
  int64_t chunk, ldI;
  size_t planes, split, total;
  int64_t split_elems;
  FwdLayout(int64_t B, int I, int O, int K) {
    const BasisLayout L(B, I, K);
    chunk = L.chunk;
    ldI = L.ldI;
    const int d = K - 1;
    planes = 0;
    split_elems = d > 0 ? gemm_split_ws_elems(chunk, O, 1, d * ceil_div(I, 64)) : 0;
    split = planes + L.per_chunk;
    total = split + align_up(sizeof(float) * split_elems) + kAlign;
  }
};

constexpr int kDbSlots = 64;  // bias-gradient row blocks per chunk

struct BwdLayout {
  int64_t chunk, n_chunks, ldO;
  bool fused_dx;
  size_t dy_hi, dy_lo, g, planes, db_part, db_tmp, split, total;
  int64_t split_elems;
  BwdLayout(int64_t B, int I, int O, int K) {
    const BasisLayout L(B, I, K);
    chunk = L.chunk;
    n_chunks = L.n_chunks;
    ldO = round_up(O, 16);  // 32-byte rows (whole-sector stores)
    const int64_t d = K - 1;
    const size_t dy = align_up(sizeof(__nv_bfloat16) * chunk * ldO);
    fused_dx = dx_tile_inputs(static_cast<int>(d), I) > 0;
    const size_t gb = fused_dx ? 0 : align_up(sizeof(float) * d * chunk * I);
    const size_t dbp = align_up(sizeof(double) * n_chunks * kDbSlots * O);
    int64_t s1 = d > 0 ? gemm_split_ws_elems(chunk, I, static_cast<int>(d), ceil_div(O, 64)) : 0;
    int64_t s2 = d > 0 ? gemm_split_ws_elems(O, I, static_cast<int>(d), ceil_div(chunk, 64)) : 0;
    const int64_t s3 = d > 0 ? gemm_split_ws_elems(I, O, static_cast<int>(d), ceil_div(chunk, 64)) : 0;  // transposed dC
    if (s3 > s2) s2 = s3;
    split_elems = s1 > s2 ? s1 : s2;
    dy_hi = 0;
    dy_lo = dy_hi + dy;
    g = dy_lo + dy;
    planes = g + gb;  // basis planes when no cache is given
    db_part = planes + L.per_chunk;
    db_tmp = db_part + dbp;
    split = db_tmp + align_up(sizeof(float) * O);
    total = split + align_up(sizeof(float) * split_elems) + kAlign;
  }
};

template <typename T>
T* at(void* base, size_t off) {
  uintptr_t b = (reinterpret_cast<uintptr_t>(base) + kAlign - 1) / kAlign * kAlign;
  return reinterpret_cast<T*>(b + off);
}

int check_dims(int64_t batch, int d_in, int d_out, const ck_lut* lut) {
  CK_CHECK(lut != nullptr, "LUT mode requires a LutTable");
  CK_CHECK(batch >= 0, "batch must be >= 0");
  CK_CHECK(d_in >= 1 && d_out >= 1, "d_in and d_out must be >= 1");
  CK_CHECK(batch * static_cast<int64_t>(d_in) < (int64_t(1) << 40), "input too large");
  return kOk;
}

}  // namespace

// ---------------------------------------------------------------------------
// Launch counter and optional per-class device timers.

namespace {
std::atomic<long long> g_launches{0};
std::atomic<int> g_timing{0};
std::mutex g_timing_mu;
struct TimedLaunch {
  int cls;
  cudaEvent_t a, b;
};
std::vector<TimedLaunch> g_pending;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

LaunchScope::LaunchScope(int cls, cudaStream_t stream) : cls_(cls), stream_(stream) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_timing.load(std::memory_order_relaxed)) {
    std::lock_guard<std::mutex> lk(g_timing_mu);
    cudaEvent_t a = take_event();
    cudaEvent_t b = take_event();
    cudaEventRecord(a, stream_);
    g_pending.push_back({cls_, a, b});
    ev_ = b;
  }
}

LaunchScope::~LaunchScope() {
  if (ev_) cudaEventRecord(static_cast<cudaEvent_t>(ev_), stream_);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("CK_PDL");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

void set_error(const std::string& msg) { g_error = msg; }
const char* last_error() { return g_error.c_str(); }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

int64_t chunk_rows() { return g_chunk_rows.load(std::memory_order_relaxed); }

namespace {
std::atomic<int> g_sm_reserve{0};
}

int gemm_sms() {
  const int n = num_sms() - g_sm_reserve.load(std::memory_order_relaxed);
  return n >= 2 ? n : 2;
}

}  // namespace ck

using ck::kOk;

extern "C" long long ck_launch_count(void) { return ck::g_launches.load(); }

extern "C" int ck_timing_enable(int on) {
  ck::g_timing.store(on ? 1 : 0);
  return kOk;
}

extern "C" int ck_timing_collect(double* ms_per_class, long long* launches_per_class, int n_classes) {
  CK_CHECK(n_classes >= 0, "ck_timing_collect: bad class count");
  std::vector<ck::TimedLaunch> pending;
  {
    std::lock_guard<std::mutex> lk(ck::g_timing_mu);
    pending.swap(ck::g_pending);
  }
  for (int c = 0; c < n_classes; ++c) {
    if (ms_per_class) ms_per_class[c] = 0.0;
    if (launches_per_class) launches_per_class[c] = 0;
  }
  int rc = kOk;
  for (auto& t : pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(t.b) != cudaSuccess || cudaEventElapsedTime(&ms, t.a, t.b) != cudaSuccess) {
      ck::set_error("ck_timing_collect: event query failed");
      rc = ck::kCudaError;
    }
    if (t.cls >= 0 && t.cls < n_classes) {
      if (ms_per_class) ms_per_class[t.cls] += ms;
      if (launches_per_class) launches_per_class[t.cls] += 1;
    }
  }
  std::lock_guard<std::mutex> lk(ck::g_timing_mu);
  for (auto& t : pending) {
    ck::g_event_pool.push_back(t.a);
    ck::g_event_pool.push_back(t.b);
  }
  return rc;
}

extern "C" int ck_version(void) { return 1 * 10000 + 0 * 100 + 0; }

extern "C" const char* ck_last_error(void) { return ck::last_error(); }

extern "C" int ck_device_supported(int device) {
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device) != cudaSuccess) return 0;
  return (major == 10 && minor == 0) ? 1 : 0;
}

extern "C" int ck_expand(const float* x, int64_t rows, int cols, const ck_lut* lut, float* phi, float* slopes,
                         void* stream) {
  CK_TRY(ck::check_dims(rows, cols, 1, lut));
  CK_CHECK(rows == 0 || (x != nullptr && phi != nullptr), "ck_expand: NULL tensor");
  return ck::launch_expand_f32(x, rows, cols, lut, phi, slopes, static_cast<cudaStream_t>(stream));
}

extern "C" int ck_basis_eval(const float* t, int64_t n, const ck_lut* lut, float* values, float* slopes,
                             void* stream) {
  CK_CHECK(lut != nullptr, "ck_basis_eval: NULL basis handle");
  CK_CHECK(n >= 0, "ck_basis_eval: negative size");
  CK_CHECK(n == 0 || (t != nullptr && values != nullptr), "ck_basis_eval: NULL tensor");
  return ck::launch_basis_eval(t, n, lut, values, slopes, static_cast<cudaStream_t>(stream));
}

extern "C" size_t ck_coeff_prep_bytes(int d_in, int d_out, int n_feat) {
  if (d_in < 1 || d_out < 1 || n_feat < 1) return 0;
  return ck::PrepLayout(d_in, d_out, n_feat).total + ck::kAlign;
}

extern "C" int ck_coeff_prepare(const float* coeff_doj, int d_in, int d_out, int n_feat, void* prep,
                                size_t prep_bytes, void* stream) {
  CK_CHECK(d_in >= 1 && d_out >= 1, "d_in and d_out must be >= 1");
  CK_CHECK(n_feat >= 1, "degree must be >= 0");
  CK_CHECK(coeff_doj != nullptr && prep != nullptr, "ck_coeff_prepare: NULL tensor");
  CK_CHECK(prep_bytes >= ck_coeff_prep_bytes(d_in, d_out, n_feat), "coefficient prep buffer too small");
  auto s = static_cast<cudaStream_t>(stream);
  const ck::PrepLayout L(d_in, d_out, n_feat);
  const int64_t I = d_in, O = d_out, K = n_feat;
  {
    // forget the buffer's previous shape until it is rewritten
    std::lock_guard<std::mutex> lk(ck::g_prep_mu);
    ck::g_preps.erase(reinterpret_cast<uintptr_t>(prep));
  }
  ck::PrepHeader h{ck::kPrepMagic, ck::kPrepVersion, d_in, d_out, n_feat, (L.skinny ? 1 : 0) | (L.gen ? 2 : 0),
                   static_cast<uint64_t>(ck_coeff_prep_bytes(d_in, d_out, n_feat))};
  if (L.skinny) {
    // the fp32 copy and the header in one launch
    CK_TRY(ck::launch_copy_with_header(coeff_doj, ck::at<float>(prep, L.f32), K * O * I, ck::at<void>(prep, L.hdr), h,
                                       s));
  } else if (L.n_i > 0) {
    // DOJ copies, the stacked input-gradient operand, c0sum and the header: one launch
    CK_TRY(ck::launch_prep_fused(coeff_doj, K, O, I, L.n_i, ck::at<__nv_bfloat16>(prep, L.doj_hi),
                                 ck::at<__nv_bfloat16>(prep, L.doj_lo), L.ldI, ck::at<__nv_bfloat16>(prep, L.dxb_hi),
                                 ck::at<__nv_bfloat16>(prep, L.dxb_lo), L.ldO, ck::at<float>(prep, L.c0sum),
                                 ck::at<void>(prep, L.hdr), h, s));
    if (L.gen) {
      CK_TRY(ck::launch_gen_coeff(coeff_doj, d_in, d_out, n_feat - 1, ck::at<__nv_bfloat16>(prep, L.gen_hi),
                                  ck::at<__nv_bfloat16>(prep, L.gen_lo), s));
    }
  } else {
    // DOJ copies: rows (k,o), unit stride in i
    CK_TRY(ck::launch_split_rows(coeff_doj, 1, K * O, I, 0, ck::at<__nv_bfloat16>(prep, L.doj_hi),
                                 ck::at<__nv_bfloat16>(prep, L.doj_lo), L.ldI, 0, s));
    if (L.n_i > 0) {
      // stacked input-gradient operand (k = 1..d), padded inputs zeroed
      CK_TRY(ck::launch_split_transpose_stacked(coeff_doj, K, O, I, L.n_i, ck::at<__nv_bfloat16>(prep, L.dxb_hi),
                                                ck::at<__nv_bfloat16>(prep, L.dxb_lo), L.ldO, s));
    } else {
      // DJO copies: per k, transpose [O][I] -> [I][O]
      CK_TRY(ck::launch_split_transpose(coeff_doj, K, O, I, O * I, ck::at<__nv_bfloat16>(prep, L.dxb_hi),
                                        ck::at<__nv_bfloat16>(prep, L.dxb_lo), L.ldO, I * L.ldO, s));
    }
    // k = 0 term: T_0 == 1 so its contribution is the per-output constant
    CK_TRY(ck::launch_row_sum(coeff_doj, O, I, ck::at<float>(prep, L.c0sum), s, ck::at<void>(prep, L.hdr), &h));
    if (L.gen) {
      CK_TRY(ck::launch_gen_coeff(coeff_doj, d_in, d_out, n_feat - 1, ck::at<__nv_bfloat16>(prep, L.gen_hi),
                                  ck::at<__nv_bfloat16>(prep, L.gen_lo), s));
    }
  }
  std::lock_guard<std::mutex> lk(ck::g_prep_mu);
  ck::g_preps[reinterpret_cast<uintptr_t>(prep)] = ck::PrepShape{d_in, d_out, n_feat};
  return kOk;
}

extern "C" int ck_coeff_prep_check(const void* prep, size_t prep_bytes, int d_in, int d_out, int n_feat) {
  CK_TRY(ck::check_prep(prep, prep_bytes, d_in, d_out, n_feat));
  // the device-side header as well (synchronous read; validation mode)
  ck::PrepHeader h{};
  CK_CUDA(cudaMemcpy(&h, ck::at<void>(const_cast<void*>(prep), 0), sizeof(h), cudaMemcpyDeviceToHost));
  if (h.magic != ck::kPrepMagic || h.version != ck::kPrepVersion || h.d_in != d_in || h.d_out != d_out ||
      h.n_feat != n_feat || h.bytes != ck_coeff_prep_bytes(d_in, d_out, n_feat)) {
    ck::set_error("coefficient prep header does not match (d_in, d_out, n_feat) = (" + std::to_string(d_in) + ", " +
                  std::to_string(d_out) + ", " + std::to_string(n_feat) + ")");
    return ck::kInvalidArgument;
  }
  return kOk;
}

extern "C" int ck_set_gemm_sm_reserve(int sms) {
  CK_CHECK(sms >= 0 && sms < ck::num_sms(), "ck_set_gemm_sm_reserve: 0 <= sms < SM count");
  return ck::g_sm_reserve.exchange(sms);
}

extern "C" int64_t ck_set_chunk_rows(int64_t rows) {
  return ck::g_chunk_rows.exchange(rows >= 1 ? rows : ck::kChunkRowsDefault);
}

extern "C" size_t ck_forward_workspace_bytes(int64_t batch, int d_in, int d_out, int n_feat) {
  if (d_in < 1 || d_out < 1 || n_feat < 1 || batch < 0) return 0;
  if (ck::skinny_layer(d_in, d_out, n_feat)) return ck::kAlign;
  return ck::FwdLayout(batch, d_in, d_out, n_feat).total;
}

extern "C" size_t ck_basis_cache_bytes(int64_t batch, int d_in, int d_out, int n_feat) {
  if (d_in < 1 || d_out < 1 || n_feat < 1 || batch < 0) return 0;
  if (ck::skinny_layer(d_in, d_out, n_feat)) return 0;
  return ck::BasisLayout(batch, d_in, n_feat).total;
}

extern "C" int ck_forward(const float* x, int64_t batch, int d_in, int d_out, const ck_lut* lut, const void* prep,
                          size_t prep_bytes, const float* bias, float* y, void* workspace, size_t workspace_bytes,
                          void* basis_cache, size_t basis_cache_bytes, void* stream) {
  CK_TRY(ck::check_dims(batch, d_in, d_out, lut));
  CK_CHECK(prep != nullptr && (batch == 0 || (x != nullptr && y != nullptr)), "ck_forward: NULL tensor");
  const int K = lut->n_feat, d = K - 1;
  CK_TRY(ck::check_prep(prep, prep_bytes, d_in, d_out, K));
  if (ck::skinny_layer(d_in, d_out, K)) {
    // d_out <= 8: CUDA-core dot products on the fp32 copy in prep
    const ck::PrepLayout P(d_in, d_out, K);
    return ck::launch_skinny_forward(x, batch, d_in, d_out, ck::at<float>(const_cast<void*>(prep), P.f32), bias, lut,
                                     y, static_cast<cudaStream_t>(stream));
  }
  const ck::FwdLayout W(batch, d_in, d_out, K);
  const ck::BasisLayout L(batch, d_in, K);
  if (workspace_bytes < W.total) {
    ck::set_error("forward workspace too small: need " + std::to_string(W.total) + " bytes");
    return ck::kWorkspace;
  }
  if (basis_cache != nullptr && basis_cache_bytes < L.total) {
    ck::set_error("basis cache too small: need " + std::to_string(L.total) + " bytes");
    return ck::kWorkspace;
  }
  if (batch == 0) return kOk;
  auto s = static_cast<cudaStream_t>(stream);
  const ck::PrepLayout P(d_in, d_out, K);
  void* pv = const_cast<void*>(prep);
  const float* c0sum = ck::at<float>(pv, P.c0sum);
  if (basis_cache == nullptr && d > 0 && P.gen && ck::gen_supported(ck::view(lut))) {
    // narrow output, no planes wanted by a backward: the basis is generated
    // in shared memory inside the GEMM (one launch for the whole batch)
    return ck::gemm_gen_forward(x, batch, d_in, d_out, ck::view(lut), ck::at<__nv_bfloat16>(pv, P.gen_hi),
                                ck::at<__nv_bfloat16>(pv, P.gen_lo), bias, c0sum, y, s);
  }
  int64_t ci = 0;
  for (int64_t r0 = 0; r0 < batch; r0 += W.chunk, ++ci) {
    const int64_t rows = batch - r0 < W.chunk ? batch - r0 : W.chunk;
    float* yc = y + r0 * d_out;
    if (d == 0) {
      CK_TRY(ck::launch_fill_rows(yc, rows, d_out, bias, c0sum, s));
      continue;
    }
    // planes: this chunk's slot of the cache, or the workspace
    auto* phi_hi = basis_cache ? ck::at<__nv_bfloat16>(basis_cache, ci * L.per_chunk)
                               : ck::at<__nv_bfloat16>(workspace, W.planes);
    auto* phi_lo = phi_hi + L.half / sizeof(__nv_bfloat16);
    CK_TRY(ck::launch_expand_planes(x + r0 * d_in, rows, d_in, lut, 1, phi_hi, phi_lo, L.ldI, L.plane, s));
    ck::GemmProblem g{};
    g.a = {phi_hi, phi_lo, rows, L.ldI, L.plane, d};
    g.b = {ck::at<__nv_bfloat16>(pv, P.doj_hi), ck::at<__nv_bfloat16>(pv, P.doj_lo), d_out, P.ldI,
           static_cast<int64_t>(d_out) * P.ldI, K};
    g.R = d_in;
    g.S = d;           // k = 1..d; the k = 0 term is c0sum (T_0 == 1)
    g.a_seg0 = 0;
    g.b_seg0 = 1;
    g.nz = 1;
    g.out = yc;
    g.ldo = d_out;
    g.out_z_stride = rows * d_out;
    g.bias0 = bias;
    g.bias1 = c0sum;
    g.split_ws = ck::at<float>(workspace, W.split);
    g.split_ws_elems = W.split_elems;
    CK_TRY(ck::gemm_bf16x3(g, s));
  }
  return kOk;
}

namespace ck {
namespace {
// skinny backward workspace: part_c [slots][K][O][I] float, part_b [slots][O] double
struct SkinnyBwdLayout {
  int slots;
  size_t part_c, part_b, total;
  SkinnyBwdLayout(int64_t B, int I, int O, int K) {
    slots = skinny_slots(B, I, O, K);
    part_c = 0;
    part_b = align_up(sizeof(float) * slots * static_cast<size_t>(K) * O * I);
    total = part_b + align_up(sizeof(double) * slots * O) + kAlign;
  }
};
}  // namespace
}  // namespace ck

extern "C" size_t ck_backward_workspace_bytes(int64_t batch, int d_in, int d_out, int n_feat) {
  if (d_in < 1 || d_out < 1 || n_feat < 1 || batch < 0) return 0;
  if (ck::skinny_layer(d_in, d_out, n_feat)) return ck::SkinnyBwdLayout(batch, d_in, d_out, n_feat).total;
  return ck::BwdLayout(batch, d_in, d_out, n_feat).total;
}

extern "C" int ck_backward(const float* x, const float* dy, int64_t batch, int d_in, int d_out, const ck_lut* lut,
                           const void* prep, size_t prep_bytes, int include_tanh_jacobian, float* dx, float* dc_doj,
                           float* db, void* workspace, size_t workspace_bytes, const void* basis_cache,
                           size_t basis_cache_bytes, void* grads_ready, void* stream) {
  CK_TRY(ck::check_dims(batch, d_in, d_out, lut));
  CK_CHECK(prep != nullptr && (batch == 0 || (x != nullptr && dy != nullptr)), "ck_backward: NULL tensor");
  const int K = lut->n_feat, d = K - 1;
  CK_TRY(ck::check_prep(prep, prep_bytes, d_in, d_out, K));
  if (ck::skinny_layer(d_in, d_out, K)) {
    auto s = static_cast<cudaStream_t>(stream);
    const ck::SkinnyBwdLayout SW(batch, d_in, d_out, K);
    if (workspace_bytes < SW.total) {
      ck::set_error("backward workspace too small: need " + std::to_string(SW.total) + " bytes");
      return ck::kWorkspace;
    }
    const int64_t n = static_cast<int64_t>(K) * d_out * d_in;
    if (batch == 0) {
      if (dc_doj) CK_CUDA(cudaMemsetAsync(dc_doj, 0, sizeof(float) * n, s));
      if (db) CK_CUDA(cudaMemsetAsync(db, 0, sizeof(float) * d_out, s));
      if (grads_ready != nullptr) CK_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(grads_ready), s));
      return kOk;
    }
    float* part_c = ck::at<float>(workspace, SW.part_c);
    double* part_b = ck::at<double>(workspace, SW.part_b);
    const ck::PrepLayout P(d_in, d_out, K);
    CK_TRY(ck::launch_skinny_backward(x, dy, batch, d_in, d_out, ck::at<float>(const_cast<void*>(prep), P.f32), lut,
                                      include_tanh_jacobian, dx, part_c, part_b, SW.slots, s));
    // second stage: ordered slot merges (kernels.py:438-442 order semantics)
    // (db's ordered slot fold runs in the same launch as the dC merge)
    const ck::ColFinishJob fin{part_b, SW.slots, d_out, db, nullptr, 0};
    if (dc_doj) {
      CK_TRY(ck::launch_merge(part_c, SW.slots, n, n, dc_doj, 0, s, db ? &fin : nullptr));
    } else if (db) {
      CK_TRY(ck::launch_col_finish(part_b, SW.slots, d_out, db, s));
    }
    if (grads_ready != nullptr) CK_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(grads_ready), s));
    return kOk;
  }
  const ck::BwdLayout W(batch, d_in, d_out, K);
  const ck::BasisLayout L(batch, d_in, K);
  if (workspace_bytes < W.total) {
    ck::set_error("backward workspace too small: need " + std::to_string(W.total) + " bytes");
    return ck::kWorkspace;
  }
  if (basis_cache != nullptr && basis_cache_bytes < L.total) {
    ck::set_error("basis cache too small: need " + std::to_string(L.total) + " bytes");
    return ck::kWorkspace;
  }
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t I = d_in, O = d_out;
  if (batch == 0) {
    if (dc_doj) CK_CUDA(cudaMemsetAsync(dc_doj, 0, sizeof(float) * K * O * I, s));
    if (db) CK_CUDA(cudaMemsetAsync(db, 0, sizeof(float) * O, s));
    if (grads_ready != nullptr) CK_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(grads_ready), s));
    return kOk;
  }
  const ck::PrepLayout P(d_in, d_out, K);
  void* pv = const_cast<void*>(prep);
  auto* dy_hi = ck::at<__nv_bfloat16>(workspace, W.dy_hi);
  auto* dy_lo = ck::at<__nv_bfloat16>(workspace, W.dy_lo);
  float* g = ck::at<float>(workspace, W.g);
  double* db_part = ck::at<double>(workspace, W.db_part);
  float* split_ws = ck::at<float>(workspace, W.split);
  // db is needed for dC_0 as well; keep a private copy when the caller skips it
  const bool need_db = db != nullptr || dc_doj != nullptr;

  bool event_done = false;
  // db, and dC_0 = db (T_0 == 1), from the row-block partials: one job, run
  // by the last chunk's dC GEMM (inside its split merge launch when it
  // splits) or on its own
  float* dbo = db != nullptr ? db : ck::at<float>(workspace, W.db_tmp);
  const ck::ColFinishJob fin_job{db_part, static_cast<int>(W.n_chunks * ck::kDbSlots), O, dbo, dc_doj, I};
  bool db_done = !need_db;
  auto finish_db = [&]() -> int {
    if (db_done) return kOk;
    CK_TRY(ck::launch_col_finish(fin_job.part, fin_job.slots, O, dbo, s, dc_doj, I));
    db_done = true;
    return kOk;
  };
  int64_t ci = 0;
  for (int64_t r0 = 0; r0 < batch; r0 += W.chunk, ++ci) {
    const int64_t rows = batch - r0 < W.chunk ? batch - r0 : W.chunk;
    const float* xc = x + r0 * I;
    const float* dyc = dy + r0 * O;
    double* dbp = db_part + ci * ck::kDbSlots * O;
    if (d == 0) {
      if (need_db) CK_TRY(ck::launch_col_partial(dyc, rows, O, dbp, ck::kDbSlots, s));
      if (dx) CK_CUDA(cudaMemsetAsync(dx + r0 * I, 0, sizeof(float) * rows * I, s));
      continue;
    }
    // dy hi/lo [rows][ldO]: K-major A of the dX GEMM and MN-major A of the dC
    // GEMM; the same pass leaves the bias gradient's per-block column sums
    if (dx || dc_doj) {
      CK_TRY(ck::launch_split_rows_colsum(dyc, rows, O, dy_hi, dy_lo, W.ldO, dbp, ck::kDbSlots, s));
    } else if (need_db) {
      CK_TRY(ck::launch_col_partial(dyc, rows, O, dbp, ck::kDbSlots, s));
    }
    // the input gradient and the coefficient gradient of this chunk
    auto run_dx = [&]() -> int {
      if (dx && W.fused_dx) {
        // one GEMM: N tile = d features x n_i inputs, slope combine + Jacobian in the epilogue
        ck::DxEpilogue epi{xc, dx + r0 * I, ck::view(lut), include_tanh_jacobian, I, P.n_i};
        ck::GemmProblem gx{};
        gx.a = {dy_hi, dy_lo, rows, W.ldO, rows * W.ldO, 1};
        gx.b = {ck::at<__nv_bfloat16>(pv, P.dxb_hi), ck::at<__nv_bfloat16>(pv, P.dxb_lo), P.dxb_rows, P.ldO,
                P.dxb_rows * P.ldO, 1};
        gx.R = O;
        gx.S = d;
        gx.nz = 1;
        gx.ldo = I;
        gx.kclass = ck::kKGemmDx;
        gx.dx = &epi;
        CK_TRY(ck::gemm_bf16x3(gx, s));
      } else if (dx) {
        ck::GemmProblem gx{};
        gx.a = {dy_hi, dy_lo, rows, W.ldO, rows * W.ldO, 1};
        gx.b = {ck::at<__nv_bfloat16>(pv, P.dxb_hi), ck::at<__nv_bfloat16>(pv, P.dxb_lo), I, P.ldO, I * P.ldO, K};
        gx.R = O;
        gx.S = 1;
        gx.b_seg0 = 1;   // z = k - 1
        gx.b_seg_z = 1;
        gx.nz = d;
        gx.out = g;
        gx.ldo = I;
        gx.out_z_stride = rows * I;
        gx.split_ws = split_ws;
        gx.split_ws_elems = W.split_elems;
        gx.kclass = ck::kKGemmDx;
        CK_TRY(ck::gemm_bf16x3(gx, s));
        CK_TRY(ck::launch_dx_combine(g, rows * I, xc, rows, d_in, lut, include_tanh_jacobian, dx + r0 * I, s));
      }
      return kOk;
    };
    auto run_dc = [&]() -> int {
      if (dc_doj) {
        const __nv_bfloat16* ph;
        if (basis_cache != nullptr) {
          ph = ck::at<__nv_bfloat16>(const_cast<void*>(basis_cache), ci * L.per_chunk);  // from the forward
        } else {
          auto* w = ck::at<__nv_bfloat16>(workspace, W.planes);
          CK_TRY(ck::launch_expand_planes(xc, rows, d_in, lut, 1, w, w + L.half / sizeof(__nv_bfloat16), L.ldI,
                                          L.plane, s));
          ph = w;
        }
        const __nv_bfloat16* pl = ph + L.half / sizeof(__nv_bfloat16);
        // dC_k[o][i] = sum_b dy[b][o] Φ_k[b][i]: both operands MN-major (batch = K).
        // Orientation: M = O (dy as A) or, when that pads fewer output cells,
        // M = I (planes as A) with a transposed store into the same [k][O][I].
        ck::GemmProblem gc{};
        const bool trans = ck::gemm_store_padded(I, O, true) < ck::gemm_store_padded(O, I, true);
        if (trans) {
          gc.a = {ph, pl, I, L.ldI, L.plane, d, 1};
          gc.b = {dy_hi, dy_lo, O, W.ldO, rows * W.ldO, 1, 1};
          gc.a_seg_z = 1;  // plane z holds k = z + 1
          gc.out_trans = 1;
        } else {
          gc.a = {dy_hi, dy_lo, O, W.ldO, rows * W.ldO, 1, 1};
          gc.b = {ph, pl, I, L.ldI, L.plane, d, 1};
          gc.b_seg_z = 1;  // plane z holds k = z + 1
        }
        gc.R = rows;
        gc.S = 1;
        gc.nz = d;
        gc.out = dc_doj + O * I;
        gc.ldo = I;
        gc.out_z_stride = O * I;
        gc.accumulate = ci > 0 ? 1 : 0;  // ascending chunk order: reproducible
        gc.split_ws = split_ws;
        gc.split_ws_elems = W.split_elems;
        gc.kclass = ck::kKGemmDc;
        const bool fold_db = !db_done && r0 + rows >= batch;  // the last chunk: db partials are complete
        if (fold_db) gc.fin = &fin_job;
        CK_TRY(ck::gemm_bf16x3(gc, s));
        if (fold_db) db_done = true;
      }
      return kOk;
    };
    if (grads_ready != nullptr && r0 + rows >= batch) {
      // last chunk with a grads-ready event: dC and db first, the event, then
      // the input-gradient GEMM -- a gradient exchange on another stream can
      // start while dX is computed
      CK_TRY(run_dc());
      CK_TRY(finish_db());
      CK_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(grads_ready), s));
      event_done = true;
      CK_TRY(run_dx());
    } else {
      CK_TRY(run_dx());
      CK_TRY(run_dc());
    }
  }
  CK_TRY(finish_db());
  if (grads_ready != nullptr && !event_done) CK_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(grads_ready), s));
  return kOk;
}

extern "C" int ck_merge(const float* partials, int num_partials, int64_t stride, int64_t n, float* out,
                        int accumulate, void* stream) {
  CK_CHECK(num_partials >= 0 && n >= 0 && stride >= n, "ck_merge: bad extents");
  CK_CHECK(out != nullptr && (partials != nullptr || num_partials == 0), "ck_merge: NULL tensor");
  return ck::launch_merge(partials, num_partials, stride, n, out, accumulate, static_cast<cudaStream_t>(stream));
}
