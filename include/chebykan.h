/*
 * chebykan.h -- C ABI of the B200-native fused Chebyshev-KAN layer.
 *
 * Drop-in boundary for the hot path of PolyKAN (arxiv 2511.14852).  The
 * reference's operator API is Python/NumPy (package `polykan`, citations
 * below are relative to /root/reference/pkg/src/polykan/); each entry point
 * states the reference interface it replaces.  All tensors are plain device
 * pointers owned by the caller (torch tensors on the host side), fp32 unless
 * noted, row-major, contiguous.  Calls are asynchronous on the given stream.
 * Return value: 0 = ok, otherwise a ck_status code; ck_last_error() returns
 * the (thread-local) message.  No exceptions cross the ABI.
 *
 * Coefficient layout: DOJ = [K][O][I] (order, output, input; input innermost),
 * the kernel layout of tensor.py:26-28 / doj_index tensor.py:72-74.
 * K = feature count (degree + 1; 2*degree + 1 for Fourier).
 */
#ifndef CHEBYKAN_H_
#define CHEBYKAN_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CK_API __attribute__((visibility("default")))
#else
#define CK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CK_OK = 0,
  CK_INVALID_ARGUMENT = 1, /* reference raises ValueError (kernels.py:245-260, 281-282, 395-408) */
  CK_CUDA_ERROR = 2,
  CK_UNSUPPORTED = 3,
  CK_WORKSPACE_TOO_SMALL = 4
} ck_status;

typedef struct ck_lut ck_lut; /* device-resident LUT (LutTable, lut.py:43-73) */

/* Library version (major*10000 + minor*100 + patch). */
CK_API int ck_version(void);
/* Message of the last failing call on this host thread. */
CK_API const char* ck_last_error(void);
/* 1 when the current device is sm_100 (B200) and the kernels can launch. */
CK_API int ck_device_supported(int device);

/* --- Basis families -----------------------------------------------------
 * Values are the reference's PKLT basis tags (lut.py:35-40, BasisKind
 * basis.py:17-21).  Feature count K = degree + 1, or 2*degree + 1 for
 * Fourier (feature_count, basis.py:24-34).  CK_BASIS_CHEBYSHEV_TRIG is the
 * exact-only cos(k*acos t) evaluation (trig_rows basis.py:144-152, the
 * reference_forward(trig=True) path kernels.py:450-478). */
typedef enum {
  CK_BASIS_CHEBYSHEV = 0,
  CK_BASIS_LEGENDRE = 1,
  CK_BASIS_HERMITE = 2,
  CK_BASIS_FOURIER = 3,
  CK_BASIS_CHEBYSHEV_TRIG = 4
} ck_basis_kind;

/* --- LUT ------------------------------------------------------------------
 * ck_lut_build replaces lut_build(kind, degree, lut_size) (lut.py:76-94):
 * float64 grid -1 + i*step with the last node forced to 1.0, values by the
 * family's three-term recurrence (basis.py:87-119; Fourier by the
 * angle-addition identities, basis.py:100-110), slopes = float64 first
 * differences / step rounded to float32.  Values are built in float64 with
 * the reference's operation order (bit-identical table) and kept on the
 * device as float32 position-major copies for the kernels.  Errors as
 * lut.py:78-81.
 */
CK_API int ck_lut_build(int kind, int degree, int lut_size, int device, ck_lut** out);
/* Wrap a caller-provided table (e.g. a PKLT file, load_lut lut.py:180-206):
 * values[K][N] float64 and slopes[K][N-1] float32, host memory. */
CK_API int ck_lut_create(int kind, int degree, int lut_size, const double* values_host, const float* slopes_host,
                  int device, ck_lut** out);
/* Exact-evaluation handle (BasisPath.EXACT_RECURRENCE, kernels.py:30-32,
 * 219-224): no table; the kernels evaluate basis_rows / derivative_rows
 * (basis.py:87-119, 155-204) at t = tanh(x) in float32.  Accepted wherever a
 * ck_lut is (ck_expand, ck_forward, ck_backward). */
CK_API int ck_basis_exact(int kind, int degree, int device, ck_lut** out);
CK_API void ck_lut_destroy(ck_lut* lut);
/* degree, lut_size and step of a table (LutTable fields, lut.py:52-56). */
CK_API int ck_lut_info(const ck_lut* lut, int* degree, int* lut_size, double* step);
/* kind, feature count and exact flag of a handle. */
CK_API int ck_lut_kind(const ck_lut* lut, int* kind, int* n_feat, int* exact);
/* Copy the float64 values [K][N] and float32 slopes [K][N-1] to host memory
 * (either pointer may be NULL); synchronous. */
CK_API int ck_lut_read(const ck_lut* lut, double* values_host, float* slopes_host);

/* --- Basis expansion ---------------------------------------------------------
 * phi[b][i][k] = interp of B_k at tanh(x[b][i]) and, when slopes != NULL,
 * slopes[b][i][k] = the active cell's slope: interp_rows_with_slope
 * (lut.py:97-123) applied to np.tanh(x) (kernels.py:288, 414).  The cell
 * (clip, idx, frac, snap) is computed in float64 so it matches the
 * reference's choice exactly; values are interpolated in float32.  With an
 * exact handle: phi = basis_rows, slopes = derivative_rows at tanh(x)
 * (kernels.py:219-224). */
CK_API int ck_expand(const float* x, int64_t rows, int cols, const ck_lut* lut, float* phi, float* slopes,
              void* stream);

/* Basis at normalized points t (no tanh): values[e][k] and (nullable)
 * slopes[e][k].  Table handles: lut_interp / lut_interp_with_slope
 * (lut.py:126-140, float64 cell as the reference); exact handles:
 * eval_basis / eval_basis_derivative / eval_basis_trig (basis.py:122-141,
 * 207-212) in float32. */
CK_API int ck_basis_eval(const float* t, int64_t n, const ck_lut* lut, float* values, float* slopes, void* stream);

/* --- Coefficient preparation (reorder_to_doj consumer, tensor.py:77-82) ---
 * Converts fp32 DOJ coefficients into the kernels' tensor-core operands:
 * bf16 hi/lo split copies in DOJ [K][O][I] (forward, unit stride in i) and
 * DJO [K][I][O] (input-gradient GEMM), plus sum_i C[0][o][i]; narrow layers
 * (d_out <= 256, d >= 4) also get an input-major copy for the forward that
 * generates the basis in shared memory.  Call once
 * per parameter update (any write to the coefficients, including in-place
 * writes the caller makes, needs a new ck_coeff_prepare before the next
 * forward/backward); `prep` is an opaque caller-owned device buffer of
 * ck_coeff_prep_bytes(...) bytes.  The buffer starts with a header
 * {magic, version, d_in, d_out, n_feat, flags, bytes}; the library also
 * records (host side) the shape each buffer was prepared for, and
 * ck_forward / ck_backward return CK_INVALID_ARGUMENT for a buffer that is
 * too small, was never prepared, or was prepared for another shape. */
CK_API size_t ck_coeff_prep_bytes(int d_in, int d_out, int n_feat);
CK_API int ck_coeff_prepare(const float* coeff_doj, int d_in, int d_out, int n_feat, void* prep,
                     size_t prep_bytes, void* stream);
/* Validation (synchronous): the host record and the device header of `prep`
 * match (d_in, d_out, n_feat); CK_INVALID_ARGUMENT otherwise. */
CK_API int ck_coeff_prep_check(const void* prep, size_t prep_bytes, int d_in, int d_out, int n_feat);

/* --- Forward: replaces fused_forward (kernels.py:351-371) ------------------
 * y[b][o] = sum_i sum_k T_k(tanh x[b][i]) C[k][o][i] + bias[o]
 * x [B][I], y [B][O]; bias nullable.  Workspace: ck_forward_workspace_bytes.
 * basis_cache (nullable, ck_basis_cache_bytes): when given, the forward keeps
 * the expanded basis planes there and ck_backward reuses them (the backward of
 * the same x then skips the expansion).  0 bytes = the layer does not use
 * basis planes (d_out <= 8 runs on the CUDA-core skinny kernels).  Without a
 * cache, narrow layers (see ck_coeff_prepare) never materialise the planes:
 * the GEMM's generator warps write the basis into shared memory. */
CK_API size_t ck_forward_workspace_bytes(int64_t batch, int d_in, int d_out, int n_feat);
CK_API size_t ck_basis_cache_bytes(int64_t batch, int d_in, int d_out, int n_feat);
CK_API int ck_forward(const float* x, int64_t batch, int d_in, int d_out, const ck_lut* lut, const void* prep,
               size_t prep_bytes, const float* bias, float* y, void* workspace, size_t workspace_bytes,
               void* basis_cache, size_t basis_cache_bytes, void* stream);

/* --- The two stages separately: forward_partial (kernels.py:263-318) and
 * combine (kernels.py:321-348), for callers of the partial buffer itself.
 * partial[to][ti][b][ty] = sum_{j in input tile ti} sum_k B_k(tanh x[b][j])
 * C[k][to*tile_out+ty][j] (PartialBuffer layout, kernels.py:108-137; g_x =
 * ceil(d_in/tile_in), g_y = ceil(d_out/tile_out); slots of padding lanes are
 * not written).  ck_combine folds the input tiles in ascending order and adds
 * bias (nullable).  fp32 CUDA-core arithmetic; ck_forward is the fast path.
 * write_counts (nullable, int64 per partial slot): every store the kernel
 * makes adds 1 to its slot's counter (atomically) -- the unique-writer
 * instrumentation of PartialBuffer.write_counts (kernels.py:123, 313-314). */
CK_API int ck_forward_partial(const float* x, int64_t batch, int d_in, int d_out, const ck_lut* lut,
                       const float* coeff_doj, int tile_in, int tile_out, float* partial, long long* write_counts,
                       void* stream);
CK_API int ck_combine(const float* partial, int64_t batch, int d_out, int g_x, int tile_out, const float* bias,
               float* y, void* stream);

/* --- Backward: replaces backward_fused (kernels.py:374-447) plus the bias
 * gradient of Layer.backward (model.py:147) --------------------------------
 * dc_doj[k][o][i] = sum_b dy[b][o] T_k(tanh x[b][i])
 * dx[b][i] = J * sum_o sum_{k>=1} dy[b][o] C[k][o][i] slope_k(b,i),
 *            J = 1 - tanh^2 x when include_tanh_jacobian (KernelMode, kernels.py:35-44)
 * db[o] = sum_b dy[b][o]
 * Any of dx / dc_doj / db may be NULL to skip.  dc is reduced by a
 * fixed-order two-stage merge: bit-reproducible run to run.
 * grads_ready_event (nullable cudaEvent_t): recorded on `stream` as soon as
 * dc_doj and db are final -- before the last input-gradient GEMM, which then
 * runs after it -- so a gradient exchange waiting on the event overlaps dX. */
CK_API size_t ck_backward_workspace_bytes(int64_t batch, int d_in, int d_out, int n_feat);
CK_API int ck_backward(const float* x, const float* dy, int64_t batch, int d_in, int d_out, const ck_lut* lut,
                const void* prep, size_t prep_bytes, int include_tanh_jacobian, float* dx, float* dc_doj,
                float* db, void* workspace, size_t workspace_bytes, const void* basis_cache,
                size_t basis_cache_bytes, void* grads_ready_event, void* stream);

/* Rows per internal batch chunk of ck_forward / ck_backward (default 32768;
 * CK_CHUNK_ROWS in the environment at load).  Chunks run in ascending order
 * on the caller's stream and dC accumulates over them in that order.
 * Process-wide; workspace and basis-cache sizes follow it, so change it only
 * between layer calls, never between a forward and the backward that reuses
 * its basis cache.  rows <= 0 restores the default.  Returns the previous
 * value. */
CK_API int64_t ck_set_chunk_rows(int64_t rows);

/* SMs the persistent GEMMs leave free (process-wide, default 0), for a
 * gradient exchange kernel running concurrently on another stream.  Results
 * do not depend on it (tiles are independent of the CTA computing them).
 * Returns the previous value. */
CK_API int ck_set_gemm_sm_reserve(int sms);

/* --- Deterministic merge: replaces combine's ordered fold (kernels.py:321-348)
 * and the ordered x-grad merge (kernels.py:438-442) as a standalone op.
 * out[n] = (accumulate ? out[n] : 0) + sum_{s=0}^{S-1} partials[s*stride + n],
 * summed in ascending s. */
CK_API int ck_merge(const float* partials, int num_partials, int64_t stride, int64_t n, float* out,
             int accumulate, void* stream);

/* --- Optimizer: replaces adam_step (model.py:247-266) -----------------------
 * In place on one fp32 parameter tensor and its moments (all n elements):
 * m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
 * p -= lr (m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps).
 * lr already includes any schedule scale (cosine decay, model.py:447-451);
 * step counts from 1 (AdamState.step after increment). */
CK_API int ck_adam_step(float* param, const float* grad, float* m, float* v, int64_t n, double lr, double beta1,
                 double beta2, double eps, int64_t step, void* stream);
/* Graph-capturable form (the step counter lives on the device): ck_adam_begin
 * increments *step_dev and writes bc_dev = {1-b1^step, 1-b2^step}; then
 * ck_adam_step_dev updates each tensor reading bc_dev.  A captured CUDA graph
 * of a training step then advances the bias correction on every replay. */
CK_API int ck_adam_begin(int64_t* step_dev, float* bc_dev, double beta1, double beta2, void* stream);
/* The same update for `count` tensors in one launch (a step's whole parameter
 * list): arrays of device pointers and sizes (host memory).  bc_dev != NULL:
 * bias corrections from the device (capturable, `step` ignored); else from
 * `step` like ck_adam_step. */
CK_API int ck_adam_step_multi(int count, float* const* params, const float* const* grads, float* const* m,
                              float* const* v, const int64_t* sizes, double lr, double beta1, double beta2,
                              double eps, int64_t step, const float* bc_dev, void* stream);
CK_API int ck_adam_step_dev(float* param, const float* grad, float* m, float* v, int64_t n, double lr,
                     double beta1, double beta2, double eps, const float* bc_dev, void* stream);

/* --- Deterministic cross-rank gradient sum over peer memory ----------------
 * The data-parallel exchange without NCCL: each rank exports its
 * flat fp32 gradient buffer (ck_ipc_handle: 64-byte cudaIpcMemHandle of the
 * enclosing allocation + byte offset), opens every peer's (ck_ipc_open), and
 * ck_allreduce_peers(bufs[ranks], rank, n) sums shard `rank` of the n
 * elements over ranks 0..R-1 in ascending order and writes it into every
 * rank's buffer (reduce-scatter + all-gather by peer stores, in place).
 * Bit-identical on all ranks and run to run.  Caller brackets it with
 * cross-rank barriers (inputs complete before; results read after). */
CK_API int ck_ipc_handle(const void* device_ptr, void* handle_out /*64 bytes*/, int64_t* offset_out);
CK_API int ck_ipc_open(const void* handle /*64 bytes*/, int64_t offset, void** device_ptr_out);
CK_API int ck_ipc_close(void* device_ptr, int64_t offset);
CK_API int ck_allreduce_peers(float* const* bufs /*host array of ranks device pointers*/, int ranks, int rank,
                       int64_t n, void* stream);
/* The same exchange for elements [lo, lo + n) with device-side
 * synchronisation instead of host barriers: flags[q] is rank q's array of
 * ck_peer_flag_words() uint64 flags (zero-initialised, IPC-mapped like the
 * buffers).  The kernel publishes "rank's gradients ready" to every rank,
 * waits until every rank's arrived, reduces its shard in ascending rank
 * order, stores it everywhere, publishes "done" and returns only when every
 * rank is done -- so it can be enqueued behind the producing kernels on any
 * stream with no host round trip.  `epoch` increases by one per call and
 * all ranks issue the same calls in the same order.  A rank that never
 * arrives turns into a device trap after 20 s (no hang).  max_blocks caps
 * the grid (0 = two per SM). */
CK_API int ck_peer_flag_words(void);
CK_API int ck_allreduce_peers_flags(float* const* bufs, unsigned long long* const* flags, int ranks, int rank,
                                    int64_t lo, int64_t n, unsigned long long epoch, int max_blocks,
                                    void* stream);

/* --- Loss ---------------------------------------------------------------------
 * ck_mse_loss: the trainer's mean squared error (model.py:184-218): loss =
 * mean((pred - target)^2) (float64 sums, deterministic) and/or grad = 2 (pred
 * - target) / n, times *grad_scale when given (a device scalar, e.g.
 * autograd's grad_output), in one pass; either output may be NULL.  The
 * workspace (ck_mse_workspace_bytes, 16-byte aligned) must be zero-filled
 * before its first use; each call leaves it ready for the next on the same
 * stream. */
CK_API size_t ck_mse_workspace_bytes(int64_t n);
CK_API int ck_mse_loss(const float* pred, const float* target, int64_t n, float* loss, float* grad,
                       const float* grad_scale, void* workspace, size_t workspace_bytes, void* stream);

/* --- Diagnostics --------------------------------------------------------------
 * ck_launch_count: kernels this library has launched in the process.
 * ck_timing_enable(1): bracket every launch with CUDA events on its stream;
 * ck_timing_collect waits for them and returns the summed device time (ms)
 * and launch count per kernel class, then clears the record.  Classes:
 * 0 GEMM forward, 1 GEMM input-grad, 2 GEMM coeff-grad, 3 expand,
 * 4 expand (transposed), 5 dx combine, 6 split, 7 reduce/merge/fill, 8 lut,
 * 9 optimizer, 10 skinny-output layer (d_out <= 8, CUDA cores). */
#define CK_NUM_KERNEL_CLASSES 11
CK_API long long ck_launch_count(void);
CK_API int ck_timing_enable(int on);
CK_API int ck_timing_collect(double* ms_per_class, long long* launches_per_class, int n_classes);
/* ck_debug_gemm_trace: per-CTA globaltimer stamps (8 per CTA) of the last
 * tensor-core GEMM launch, copied to out[max_ctas][8]; returns the CTA rows
 * copied, 0 when the library was built without CK_GEMM_TRACE (the default). */
CK_API int ck_debug_gemm_trace(unsigned long long* out, int max_ctas);

#ifdef __cplusplus
}
#endif

#endif /* CHEBYKAN_H_ */
