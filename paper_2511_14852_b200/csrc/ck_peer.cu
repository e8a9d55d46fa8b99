// Deterministic cross-rank gradient sum over peer memory (CUDA IPC over
// NVLink / NVSwitch, or two processes sharing one device).  Every rank maps
// every other rank's flat gradient buffer; rank r owns the contiguous shard
// r of the elements, sums it over ranks 0..R-1 in ascending order and stores
// the result into the same shard of every rank's buffer -- a fixed-order
// reduce-scatter and an all-gather by peer stores in one kernel, in place.
// Each element is summed by exactly one rank in one order, so all ranks hold
// bit-identical gradients, run to run, independent of NCCL's algorithm
// choice ("deterministic variant").
//
// Preconditions (the host helper enforces them with barriers): every rank's
// local gradient is complete before any rank launches, and no rank reads the
// result before every rank's kernel has finished.
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

constexpr int kMaxPeers = 8;
}  // namespace
constexpr int kFlagWordsPublic = 32;  // uint64 flag words per rank (3 * 8 used)
namespace {

struct PeerPtrs {
  float* p[kMaxPeers];
};

__global__ void __launch_bounds__(256) allreduce_peers_kernel(PeerPtrs bufs, int ranks, int64_t lo, int64_t hi) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  // vector part: shard bounds are multiples of 4 elements (host rounds them)
  const int64_t n4 = (hi - lo) >> 2;
  for (int64_t i = t0; i < n4; i += stride) {
    const int64_t e = lo + 4 * i;
    float4 acc = *reinterpret_cast<const float4*>(bufs.p[0] + e);
    for (int r = 1; r < ranks; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(bufs.p[r] + e);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    for (int r = 0; r < ranks; ++r) *reinterpret_cast<float4*>(bufs.p[r] + e) = acc;
  }
  for (int64_t e = lo + 4 * n4 + t0; e < hi; e += stride) {
    float acc = bufs.p[0][e];
    for (int r = 1; r < ranks; ++r) acc += bufs.p[r][e];
    for (int r = 0; r < ranks; ++r) bufs.p[r][e] = acc;
  }
}

// ---------------------------------------------------------------------------
// Flag-synchronised variant: no host barriers.  Each rank owns a small array
// of 64-bit flags inside its IPC-mapped exchange buffer (kFlagWords words):
//   [kReady + q]  epoch at which rank q's gradients for this exchange are complete
//   [kDone + q]   epoch at which rank q has stored its reduced shard everywhere
//   [kCounter]    blocks of this rank's kernel finished (local)
// Epochs grow by one per exchange and every rank issues its exchanges in
// the same order, so a flag value >= epoch means "this exchange".  Waits
// give up after kSpinLimitNs with a trap: a missing peer becomes a CUDA
// error on the next synchronisation instead of a hang.
constexpr int kReady = 0, kDone = kMaxPeers, kCounter = 2 * kMaxPeers;
constexpr unsigned long long kSpinLimitNs = 20ull * 1000 * 1000 * 1000;

struct PeerFlags {
  unsigned long long* f[kMaxPeers];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// one thread: until every rank's flag slot [base + q] reached epoch
__device__ void wait_all(const unsigned long long* mine, int base, int ranks, unsigned long long epoch) {
  const unsigned long long t0 = globaltimer();
  for (int q = 0; q < ranks; ++q) {
    while (ld_acquire_sys(mine + base + q) < epoch) {
      if (globaltimer() - t0 > kSpinLimitNs) __trap();
      __nanosleep(200);
    }
  }
}

__global__ void __launch_bounds__(512) allreduce_flags_kernel(PeerPtrs bufs, PeerFlags flags, int ranks, int rank,
                                                             int64_t lo, int64_t hi, unsigned long long epoch) {
  unsigned long long* mine = flags.f[rank];
  // (this rank's gradients are complete: the kernel runs after the producing
  // kernels on the stream)
  if (blockIdx.x == 0 && threadIdx.x < ranks) st_release_sys(flags.f[threadIdx.x] + kReady + rank, epoch);
  if (threadIdx.x == 0) wait_all(mine, kReady, ranks, epoch);
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t n4 = (hi - lo) >> 2;
  for (int64_t i = t0; i < n4; i += stride) {
    const int64_t e = lo + 4 * i;
    float4 acc = __ldcv(reinterpret_cast<const float4*>(bufs.p[0] + e));
    for (int r = 1; r < ranks; ++r) {
      const float4 v = __ldcv(reinterpret_cast<const float4*>(bufs.p[r] + e));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    for (int r = 0; r < ranks; ++r) *reinterpret_cast<float4*>(bufs.p[r] + e) = acc;
  }
  for (int64_t e = lo + 4 * n4 + t0; e < hi; e += stride) {
    float acc = __ldcv(bufs.p[0] + e);
    for (int r = 1; r < ranks; ++r) acc += __ldcv(bufs.p[r] + e);
    for (int r = 0; r < ranks; ++r) bufs.p[r][e] = acc;
  }
  // the last block to finish publishes DONE to every rank, then waits until
  // every rank's DONE arrived: when this kernel ends, all shards are stored
  // in this rank's buffer and no peer still reads it
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long prev = atomicAdd(mine + kCounter, 1ull);
    if (prev == gridDim.x - 1) {
      mine[kCounter] = 0;
      __threadfence_system();
      for (int q = 0; q < ranks; ++q) st_release_sys(flags.f[q] + kDone + rank, epoch);
      wait_all(mine, kDone, ranks, epoch);
    }
  }
}

PFN_cuMemGetAddressRange_v3020 get_range_fn() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(ptr);
  });
  return fn;
}

}  // namespace
}  // namespace ck

extern "C" int ck_ipc_handle(const void* ptr, void* handle_out, int64_t* offset_out) {
  CK_CHECK(ptr && handle_out && offset_out, "ck_ipc_handle: NULL argument");
  auto range = ck::get_range_fn();
  if (!range) {
    ck::set_error("cuMemGetAddressRange unavailable");
    return ck::kCudaError;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) {
    ck::set_error("ck_ipc_handle: pointer is not device memory");
    return ck::kInvalidArgument;
  }
  cudaIpcMemHandle_t h;
  CK_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return ck::kOk;
}

extern "C" int ck_ipc_open(const void* handle, int64_t offset, void** ptr_out) {
  CK_CHECK(handle && ptr_out, "ck_ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  CK_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr_out = static_cast<char*>(base) + offset;
  return ck::kOk;
}

extern "C" int ck_ipc_close(void* ptr, int64_t offset) {
  CK_CHECK(ptr, "ck_ipc_close: NULL pointer");
  CK_CUDA(cudaIpcCloseMemHandle(static_cast<char*>(ptr) - offset));
  return ck::kOk;
}

extern "C" int ck_allreduce_peers(float* const* bufs, int ranks, int rank, int64_t n, void* stream) {
  CK_CHECK(ranks >= 1 && ranks <= ck::kMaxPeers, "ck_allreduce_peers: 1..8 ranks");
  CK_CHECK(rank >= 0 && rank < ranks, "ck_allreduce_peers: rank out of range");
  CK_CHECK(n >= 0 && bufs != nullptr, "ck_allreduce_peers: bad arguments");
  ck::PeerPtrs pp{};
  for (int r = 0; r < ranks; ++r) {
    CK_CHECK(bufs[r] != nullptr && (reinterpret_cast<uintptr_t>(bufs[r]) & 15) == 0,
             "ck_allreduce_peers: buffers must be 16-byte aligned");
    pp.p[r] = bufs[r];
  }
  // shard r = [lo, hi), boundaries rounded to 4 elements
  const int64_t per = ck::round_up(ck::ceil_div(n, ranks), 4);
  const int64_t lo = rank * per < n ? rank * per : n;
  const int64_t hi = lo + per < n ? lo + per : n;
  if (hi <= lo) return ck::kOk;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t want = ck::ceil_div(ck::ceil_div(hi - lo, 4), 256);
  const int64_t cap = static_cast<int64_t>(ck::num_sms()) * 4;
  ck::LaunchScope scope(ck::kKReduce, s);
  ck::allreduce_peers_kernel<<<static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap)), 256, 0, s>>>(pp, ranks,
                                                                                                       lo, hi);
  CK_CUDA(cudaGetLastError());
  return ck::kOk;
}

extern "C" int ck_peer_flag_words(void) { return ck::kFlagWordsPublic; }

extern "C" int ck_allreduce_peers_flags(float* const* bufs, unsigned long long* const* flags, int ranks, int rank,
                                        int64_t lo, int64_t n, unsigned long long epoch, int max_blocks,
                                        void* stream) {
  CK_CHECK(ranks >= 1 && ranks <= ck::kMaxPeers, "ck_allreduce_peers_flags: 1..8 ranks");
  CK_CHECK(rank >= 0 && rank < ranks, "ck_allreduce_peers_flags: rank out of range");
  CK_CHECK(lo >= 0 && n >= 0 && bufs != nullptr && flags != nullptr && epoch >= 1,
           "ck_allreduce_peers_flags: bad arguments");
  ck::PeerPtrs pp{};
  ck::PeerFlags pf{};
  for (int r = 0; r < ranks; ++r) {
    CK_CHECK(bufs[r] != nullptr && flags[r] != nullptr && (reinterpret_cast<uintptr_t>(bufs[r]) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(flags[r]) & 7) == 0,
             "ck_allreduce_peers_flags: buffers must be 16-byte and flags 8-byte aligned");
    pp.p[r] = bufs[r];
    pf.f[r] = flags[r];
  }
  CK_CHECK(lo % 4 == 0, "ck_allreduce_peers_flags: range start must be a multiple of 4 elements");
  // shard `rank` of [lo, lo + n), boundaries on 4-element multiples
  const int64_t per = ck::round_up(ck::ceil_div(n, ranks), 4);
  const int64_t a = lo + (rank * per < n ? rank * per : n);
  const int64_t b = (a + per < lo + n) ? a + per : lo + n;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t want = ck::ceil_div(ck::ceil_div(b > a ? b - a : 1, 4), 512);
  int64_t cap = max_blocks > 0 ? max_blocks : static_cast<int64_t>(ck::num_sms()) * 2;
  const int blocks = static_cast<int>(want < cap ? want : cap);
  ck::LaunchScope scope(ck::kKReduce, s);
  // (an empty shard still takes part in the flag exchange)
  ck::allreduce_flags_kernel<<<blocks < 1 ? 1 : blocks, 512, 0, s>>>(pp, pf, ranks, rank, a, b > a ? b : a, epoch);
  CK_CUDA(cudaGetLastError());
  return ck::kOk;
}
