// Optimizer step on the device: Adam with bias correction, the update rule
// of the reference trainer (adam_step, model.py:247-266), elementwise over
// one parameter tensor and its moment buffers.  HBM-bound: reads p, g, m, v
// and writes p, m, v (28 bytes per element).
#include <cmath>

#include "ck_common.cuh"
#include "ck_internal.h"

namespace ck {
namespace {

constexpr int kThreads = 256;

struct AdamArgs {
  float lr, b1, omb1, b2, omb2, bc1, bc2, eps;
  const float* bc_dev;  // nullable: {bc1, bc2} read from device memory (graph-capturable form)
};

// m = m*b1 + (1-b1)*g; v = v*b2 + (1-b2)*g*g; p -= lr * (m/bc1) / (sqrt(v/bc2) + eps)
// with the reference's operation order and no FMA contraction.
__device__ __forceinline__ void adam_one(float& p, float g, float& m, float& v, const AdamArgs& a) {
  m = __fadd_rn(__fmul_rn(m, a.b1), __fmul_rn(a.omb1, g));
  v = __fadd_rn(__fmul_rn(v, a.b2), __fmul_rn(a.omb2, __fmul_rn(g, g)));
  const float mh = __fdiv_rn(m, a.bc1), vh = __fdiv_rn(v, a.bc2);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(a.lr, mh), __fadd_rn(__fsqrt_rn(vh), a.eps)));
}

__global__ void __launch_bounds__(kThreads) adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                                                        float* __restrict__ m, float* __restrict__ v, int64_t n,
                                                        AdamArgs a) {
  pdl_wait();
  if (a.bc_dev) {
    a.bc1 = a.bc_dev[0];
    a.bc2 = a.bc_dev[1];
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(m) |
                     reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  if (vec) {
    const int64_t n4 = n >> 2;
    for (int64_t i = t0; i < n4; i += stride) {
      float4 pp = reinterpret_cast<float4*>(p)[i];
      const float4 gg = reinterpret_cast<const float4*>(g)[i];
      float4 mm = reinterpret_cast<float4*>(m)[i];
      float4 vv = reinterpret_cast<float4*>(v)[i];
      adam_one(pp.x, gg.x, mm.x, vv.x, a);
      adam_one(pp.y, gg.y, mm.y, vv.y, a);
      adam_one(pp.z, gg.z, mm.z, vv.z, a);
      adam_one(pp.w, gg.w, mm.w, vv.w, a);
      reinterpret_cast<float4*>(p)[i] = pp;
      reinterpret_cast<float4*>(m)[i] = mm;
      reinterpret_cast<float4*>(v)[i] = vv;
    }
    for (int64_t i = (n4 << 2) + t0; i < n; i += stride) adam_one(p[i], g[i], m[i], v[i], a);
  } else {
    for (int64_t i = t0; i < n; i += stride) adam_one(p[i], g[i], m[i], v[i], a);
  }
}

// Several tensors in one launch (a training step's whole parameter list):
// the tensors are cut into chunks of kMultiChunk elements, a block walks
// chunks grid-stride and finds its tensor in the chunk prefix table.
constexpr int kMultiMax = 32;
constexpr int kMultiChunk = 2048;

struct MultiTensors {
  int count;
  float* p[kMultiMax];
  const float* g[kMultiMax];
  float* m[kMultiMax];
  float* v[kMultiMax];
  int64_t n[kMultiMax];
  int64_t chunk0[kMultiMax + 1];  // first chunk of each tensor; chunk0[count] = total
};

__global__ void __launch_bounds__(kThreads) adam_multi_kernel(const __grid_constant__ MultiTensors T, AdamArgs a) {
  pdl_wait();
  if (a.bc_dev) {
    a.bc1 = a.bc_dev[0];
    a.bc2 = a.bc_dev[1];
  }
  const int64_t total = T.chunk0[T.count];
  for (int64_t c = blockIdx.x; c < total; c += gridDim.x) {
    int t = 0;
    while (t + 1 < T.count && T.chunk0[t + 1] <= c) ++t;
    const int64_t e0 = (c - T.chunk0[t]) * kMultiChunk;
    const int64_t e1 = e0 + kMultiChunk < T.n[t] ? e0 + kMultiChunk : T.n[t];
    float* p = T.p[t];
    const float* g = T.g[t];
    float* m = T.m[t];
    float* v = T.v[t];
    const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                       reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0 &&
                     e1 - e0 == kMultiChunk;
    if (vec) {
      for (int64_t i = e0 / 4 + threadIdx.x; i < e1 / 4; i += blockDim.x) {
        float4 pp = reinterpret_cast<float4*>(p)[i];
        const float4 gg = reinterpret_cast<const float4*>(g)[i];
        float4 mm = reinterpret_cast<float4*>(m)[i];
        float4 vv = reinterpret_cast<float4*>(v)[i];
        adam_one(pp.x, gg.x, mm.x, vv.x, a);
        adam_one(pp.y, gg.y, mm.y, vv.y, a);
        adam_one(pp.z, gg.z, mm.z, vv.z, a);
        adam_one(pp.w, gg.w, mm.w, vv.w, a);
        reinterpret_cast<float4*>(p)[i] = pp;
        reinterpret_cast<float4*>(m)[i] = mm;
        reinterpret_cast<float4*>(v)[i] = vv;
      }
    } else {
      for (int64_t i = e0 + threadIdx.x; i < e1; i += blockDim.x) adam_one(p[i], g[i], m[i], v[i], a);
    }
  }
}

// step += 1; bc = {1 - b1^step, 1 - b2^step} (float64 pow, model.py:262-263)
__global__ void adam_begin_kernel(int64_t* step, float* bc, double b1, double b2) {
  pdl_wait();
  const int64_t t = ++(*step);
  bc[0] = static_cast<float>(1.0 - pow(b1, static_cast<double>(t)));
  bc[1] = static_cast<float>(1.0 - pow(b2, static_cast<double>(t)));
}

int adam_launch(float* param, const float* grad, float* m, float* v, int64_t n, const AdamArgs& a, cudaStream_t s) {
  const int64_t want = ceil_div(ceil_div(n, 4), kThreads);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  const int blocks = static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
  LaunchScope scope(kKOptim, s);
  CK_CUDA(launch_k((adam_kernel), blocks, kThreads, 0, s, param, grad, m, v, n, a));
  CK_CUDA(cudaGetLastError());
  return kOk;
}

// ---------------------------------------------------------------------------
// Mean squared error (model.py:184-218 mse: mean((p - t)^2), gradient
// 2 (p - t) / n) in one pass: each block sums its (p - t)^2 in float64 over a
// fixed grid-stride partition and a fixed shared-memory tree; the last block
// to finish (a counter in the workspace, reset by that block) adds the block
// partials in block order -- deterministic for a given n and device.  The
// gradient, optionally times a device scalar (autograd's grad_output), is
// written in the same pass.
constexpr int kMseThreads = 256;

__global__ void __launch_bounds__(kMseThreads) mse_kernel(const float* __restrict__ pred,
                                                          const float* __restrict__ target, int64_t n,
                                                          float* __restrict__ loss, float* __restrict__ grad,
                                                          const float* __restrict__ grad_scale,
                                                          double* __restrict__ part, unsigned int* counter) {
  pdl_wait();
  __shared__ double red[kMseThreads];
  __shared__ bool last;
  const float gscale = (grad_scale ? grad_scale[0] : 1.0f);
  const float nf = static_cast<float>(n);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  double acc = 0.0;
  const bool vec = ((reinterpret_cast<uintptr_t>(pred) | reinterpret_cast<uintptr_t>(target) |
                     reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
  const bool want_grad = grad != nullptr;
  auto one = [&](float p, float t) -> float {
    const float d = p - t;
    acc += static_cast<double>(d) * static_cast<double>(d);
    // 2 * diff / n (model.py order), x grad_out
    return want_grad ? __fmul_rn(__fdiv_rn(__fmul_rn(2.0f, d), nf), gscale) : 0.0f;
  };
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t i = t0; i < n4; i += stride) {
    const float4 p = __ldg(reinterpret_cast<const float4*>(pred) + i);
    const float4 t = __ldg(reinterpret_cast<const float4*>(target) + i);
    float4 g;
    g.x = one(p.x, t.x);
    g.y = one(p.y, t.y);
    g.z = one(p.z, t.z);
    g.w = one(p.w, t.w);
    if (grad) reinterpret_cast<float4*>(grad)[i] = g;
  }
  for (int64_t i = 4 * n4 + t0; i < n; i += stride) {
    const float g = one(pred[i], target[i]);
    if (grad) grad[i] = g;
  }
  if (loss == nullptr) return;
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kMseThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = red[0];
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // the last block folds the block partials: thread j sums partials j, j +
  // 256, ... in order, then the same fixed tree (a serial fold of ~600
  // partials took 30 us of L2 round trips)
  __threadfence();
  double s = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += kMseThreads) s += __ldcg(part + b);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kMseThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *loss = static_cast<float>(red[0] / static_cast<double>(n));
    *counter = 0u;  // ready for the next call
  }
}

int mse_blocks(int64_t n) {
  const int64_t want = ceil_div(ceil_div(n > 0 ? n : 1, 4), kMseThreads);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 4;
  return static_cast<int>(want < cap ? want : cap);
}

}  // namespace
}  // namespace ck

extern "C" size_t ck_mse_workspace_bytes(int64_t n) {
  // block partials (float64) + the completion counter
  (void)n;  // the partials are per block; the grid is capped at 4 blocks per SM
  return sizeof(double) * static_cast<size_t>(ck::num_sms()) * 4 + 16;
}

extern "C" int ck_mse_loss(const float* pred, const float* target, int64_t n, float* loss, float* grad,
                           const float* grad_scale, void* workspace, size_t workspace_bytes, void* stream) {
  CK_CHECK(n >= 1, "ck_mse_loss: empty input");
  CK_CHECK(pred && target && (loss || grad), "ck_mse_loss: NULL tensor");
  CK_CHECK(loss == nullptr || (workspace != nullptr && workspace_bytes >= ck_mse_workspace_bytes(n)),
           "ck_mse_loss: workspace too small");
  CK_CHECK((reinterpret_cast<uintptr_t>(workspace) & 15) == 0, "ck_mse_loss: workspace must be 16-byte aligned");
  auto s = static_cast<cudaStream_t>(stream);
  const int blocks = ck::mse_blocks(n);
  double* part = static_cast<double*>(workspace);
  unsigned int* counter = loss ? reinterpret_cast<unsigned int*>(part + static_cast<size_t>(ck::num_sms()) * 4) : nullptr;
  ck::LaunchScope scope(ck::kKOptim, s);
  CK_CUDA(ck::launch_k((ck::mse_kernel), blocks, ck::kMseThreads, 0, s, pred, target, n, loss, grad, grad_scale, part,
                       counter));
  CK_CUDA(cudaGetLastError());
  return ck::kOk;
}

extern "C" int ck_adam_step(float* param, const float* grad, float* m, float* v, int64_t n, double lr,
                            double beta1, double beta2, double eps, int64_t step, void* stream) {
  CK_CHECK(n >= 0, "ck_adam_step: negative size");
  CK_CHECK(step >= 1, "ck_adam_step: step counts from 1");
  if (n == 0) return ck::kOk;
  CK_CHECK(param && grad && m && v, "ck_adam_step: NULL tensor");
  ck::AdamArgs a;
  a.lr = static_cast<float>(lr);
  a.b1 = static_cast<float>(beta1);
  a.omb1 = static_cast<float>(1.0 - beta1);
  a.b2 = static_cast<float>(beta2);
  a.omb2 = static_cast<float>(1.0 - beta2);
  // bias corrections 1 - beta^t in float64 on the host (model.py:262-263)
  a.bc1 = static_cast<float>(1.0 - std::pow(beta1, static_cast<double>(step)));
  a.bc2 = static_cast<float>(1.0 - std::pow(beta2, static_cast<double>(step)));
  a.eps = static_cast<float>(eps);
  a.bc_dev = nullptr;
  return ck::adam_launch(param, grad, m, v, n, a, static_cast<cudaStream_t>(stream));
}

extern "C" int ck_adam_begin(int64_t* step_dev, float* bc_dev, double beta1, double beta2, void* stream) {
  CK_CHECK(step_dev && bc_dev, "ck_adam_begin: NULL pointer");
  auto s = static_cast<cudaStream_t>(stream);
  ck::LaunchScope scope(ck::kKOptim, s);
  CK_CUDA(ck::launch_k((ck::adam_begin_kernel), 1, 1, 0, s, step_dev, bc_dev, beta1, beta2));
  CK_CUDA(cudaGetLastError());
  return ck::kOk;
}

extern "C" int ck_adam_step_dev(float* param, const float* grad, float* m, float* v, int64_t n, double lr,
                                double beta1, double beta2, double eps, const float* bc_dev, void* stream) {
  CK_CHECK(n >= 0, "ck_adam_step_dev: negative size");
  if (n == 0) return ck::kOk;
  CK_CHECK(param && grad && m && v && bc_dev, "ck_adam_step_dev: NULL tensor");
  ck::AdamArgs a;
  a.lr = static_cast<float>(lr);
  a.b1 = static_cast<float>(beta1);
  a.omb1 = static_cast<float>(1.0 - beta1);
  a.b2 = static_cast<float>(beta2);
  a.omb2 = static_cast<float>(1.0 - beta2);
  a.bc1 = a.bc2 = 1.0f;
  a.eps = static_cast<float>(eps);
  a.bc_dev = bc_dev;
  return ck::adam_launch(param, grad, m, v, n, a, static_cast<cudaStream_t>(stream));
}

extern "C" int ck_adam_step_multi(int count, float* const* params, const float* const* grads, float* const* m,
                                  float* const* v, const int64_t* sizes, double lr, double beta1, double beta2,
                                  double eps, int64_t step, const float* bc_dev, void* stream) {
  CK_CHECK(count >= 0, "ck_adam_step_multi: negative count");
  CK_CHECK(count == 0 || (params && grads && m && v && sizes), "ck_adam_step_multi: NULL array");
  CK_CHECK(bc_dev != nullptr || step >= 1, "ck_adam_step_multi: step counts from 1");
  ck::AdamArgs a;
  a.lr = static_cast<float>(lr);
  a.b1 = static_cast<float>(beta1);
  a.omb1 = static_cast<float>(1.0 - beta1);
  a.b2 = static_cast<float>(beta2);
  a.omb2 = static_cast<float>(1.0 - beta2);
  a.bc1 = bc_dev ? 1.0f : static_cast<float>(1.0 - std::pow(beta1, static_cast<double>(step)));
  a.bc2 = bc_dev ? 1.0f : static_cast<float>(1.0 - std::pow(beta2, static_cast<double>(step)));
  a.eps = static_cast<float>(eps);
  a.bc_dev = bc_dev;
  auto s = static_cast<cudaStream_t>(stream);
  // batches of up to kMultiMax non-empty tensors; the next batch resumes at
  // the first tensor this one did not take (zero-size ones are skipped, not
  // counted, so a fixed stride would revisit tensors)
  for (int t = 0; t < count;) {
    ck::MultiTensors T{};
    int k = 0;
    int64_t chunks = 0;
    for (; t < count && k < ck::kMultiMax; ++t) {
      CK_CHECK(sizes[t] >= 0, "ck_adam_step_multi: negative size");
      if (sizes[t] == 0) continue;
      CK_CHECK(params[t] && grads[t] && m[t] && v[t], "ck_adam_step_multi: NULL tensor");
      T.p[k] = params[t];
      T.g[k] = grads[t];
      T.m[k] = m[t];
      T.v[k] = v[t];
      T.n[k] = sizes[t];
      T.chunk0[k] = chunks;
      chunks += ck::ceil_div(sizes[t], static_cast<int64_t>(ck::kMultiChunk));
      ++k;
    }
    if (k == 0) continue;
    T.count = k;
    T.chunk0[k] = chunks;
    const int64_t cap = static_cast<int64_t>(ck::num_sms()) * 8;
    ck::LaunchScope scope(ck::kKOptim, s);
    CK_CUDA(ck::launch_k((ck::adam_multi_kernel), static_cast<int>(chunks < cap ? chunks : cap), ck::kThreads, 0, s,
                         T, a));
    CK_CUDA(cudaGetLastError());
  }
  return ck::kOk;
}
