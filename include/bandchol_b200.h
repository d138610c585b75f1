/*
 * bandchol_b200.h -- C ABI of the B200-native fp64 band Cholesky library
 * (libbandchol_b200.so).  Plain pointers and sizes; no torch or CUDA types.
 *
 * Storage: LAPACK lower band AB(ldab, n), element (i,j), j <= i <= min(n-1, j+kd),
 * at ab[j*ldab + (i-j)] -- the reference's BandedMatrix layout
 * (pkg/src/bandchol/core.py:1-19, :34-44).  Padding slots are never written.
 *
 * All pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) on the
 * current device; every call is asynchronous on `stream` (a cudaStream_t, NULL =
 * legacy default stream) and returns once the work is enqueued.
 *
 * Return codes: 0 = enqueued; -i = argument i is illegal (LAPACK style,
 * 1-based); > 0 = a CUDA error code.  bcg_last_error() gives the message
 * (thread-local).  Numerical outcomes are reported through the device `info`
 * array, LAPACK convention: 0 = success, c+1 = the pivot of global column c was
 * not > 0 (NaN counts as failure) for dpbtrf -> the reference's
 * NotPositiveDefinite(c) (reference.py:56-57, errors.py:31-39); for dpbtrs
 * c+1 = diagonal of L at column c is <= 0 -> SingularFactor (core.py:227-230),
 * in which case b is left untouched.
 */
#ifndef BANDCHOL_B200_H
#define BANDCHOL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Library ABI version (major*100 + minor). */
int bcg_version(void);

/* Thread-local message describing the last non-zero return. */
const char* bcg_last_error(void);

/* Workspace bytes bcg_dpbtrf needs for an (n, kd) matrix (0 when the single
 * matrix runs in one CTA).  Holds the per-tile ready flags of the multi-CTA kernel.
 * The caller owns it (no allocation on the hot path); its contents on entry are
 * ignored: every launch clears it in stream order, so one workspace may serve calls
 * that are ordered on one stream, but concurrent calls need distinct workspaces. */
size_t bcg_dpbtrf_workspace_size(int64_t n, int64_t kd, int64_t ldab);

/* In-place lower band Cholesky A = L L^T of ONE matrix, using the whole GPU.
 * Replaces the reference engines factor_blocked_serial
 * (pkg/src/bandchol/blocked.py:363-385) and factor_blocked_parallel
 * (pkg/src/bandchol/parallel.py:130-166); info: device int32[1]. */
int bcg_dpbtrf(int64_t n, int64_t kd, double* ab, int64_t ldab, int32_t* info,
               void* workspace, size_t workspace_bytes, void* stream);

/* Workspace bytes bcg_dpbtrf_batched / bcg_dpbsv_batched need: 0 when every matrix is
 * factored by one CTA (its band window fits in shared memory), else the whole-GPU
 * kernel's flags, reused matrix after matrix (same contract as above). */
size_t bcg_dpbtrf_batched_workspace_size(int64_t n, int64_t kd, int64_t ldab, int64_t batch);

/* In-place factorization of `batch` independent matrices of the same (n, kd,
 * ldab) stored stride_ab doubles apart; info: device int32[batch].  Each matrix
 * follows the same contract as one bcg_dpbtrf call (the batched interior-point
 * use case of BASELINE.json config C5). */
int bcg_dpbtrf_batched(int64_t n, int64_t kd, double* ab, int64_t ldab, int64_t stride_ab,
                       int64_t batch, int32_t* info, void* workspace, size_t workspace_bytes,
                       void* stream);

/* Solve L L^T X = B in place (B -> X) with the factor from bcg_dpbtrf; nrhs
 * right-hand sides stored ldb doubles apart, all served by one pass over L per
 * group of up to 16.  Replaces solve_with_factor (pkg/src/bandchol/core.py:216-240).
 * info: device int32[1]; a diagonal entry <= 0 gives info = its column + 1 and B
 * untouched (SingularFactor, core.py:227-230). */
int bcg_dpbtrs(int64_t n, int64_t kd, const double* ab, int64_t ldab, double* b, int64_t ldb,
               int64_t nrhs, int32_t* info, void* stream);

/* Batched solve: matrix i uses ab + i*stride_ab and its single right-hand side
 * b + i*stride_b; info: device int32[batch]. */
int bcg_dpbtrs_batched(int64_t n, int64_t kd, const double* ab, int64_t ldab, int64_t stride_ab,
                       double* b, int64_t stride_b, int64_t batch, int32_t* info, void* stream);

/* Batched multi-right-hand-side solve: matrix i has nrhs right-hand sides, column r at
 * b + i*stride_b + r*ldb (the repeated solves of an interior-point iteration).  One pass
 * over each L serves up to 16 right-hand sides. */
int bcg_dpbtrs_batched_nrhs(int64_t n, int64_t kd, const double* ab, int64_t ldab, int64_t stride_ab,
                            double* b, int64_t ldb, int64_t stride_b, int64_t nrhs, int64_t batch,
                            int32_t* info, void* stream);

/* Workspace bytes of bcg_dpbsv_batched: batch * n doubles (the forward sweep's y, one row
 * per matrix) when the fused path applies -- 32 <= kd and the band window fits one CTA's
 * shared memory -- else bcg_dpbtrf_batched_workspace_size.  A smaller (or NULL) workspace is
 * accepted: the call then runs the unfused path (factorization, two-sweep solve). */
size_t bcg_dpbsv_batched_workspace_size(int64_t n, int64_t kd, int64_t ldab, int64_t batch);

/* Batched factor + solve (config C5): on return ab holds L and b holds x.  Stream-ordered
 * on `stream`: the batched factorization -- with the forward sweep L y = b fused in (the
 * factorization kernel solves each 16-row block right behind its panel, from shared memory,
 * y to the workspace) -- then the backward sweep of the matrices that factored.
 * info: device int32[batch] with the dpbtrf convention; a matrix that fails keeps its b
 * untouched (LAPACK dpbsv) and its ab partially overwritten (as after a failed reference
 * factorization).  Replaces factor_blocked_serial (pkg/src/bandchol/blocked.py:363-385)
 * followed by solve_with_factor (pkg/src/bandchol/core.py:216-240) per matrix. */
int bcg_dpbsv_batched(int64_t n, int64_t kd, double* ab, int64_t ldab, int64_t stride_ab,
                      double* b, int64_t stride_b, int64_t batch, int32_t* info,
                      void* workspace, size_t workspace_bytes, void* stream);

/* The two halves of bcg_dpbsv_batched's fused path, callable (and timed) on their own.
 * bcg_dpbtrf_fwd_batched: in-place factorization of the batch with the forward sweep
 *   L y = b fused in; b is only read, y (device, batch * n doubles, row i = matrix i) is
 *   written for the matrices -- and up to the block -- that factored.  Needs 32 <= kd and a
 *   band window that fits one CTA's shared memory (else a negative argument code).
 * bcg_dpbtrs_bwd_batched: L^T x = y for the matrices with info[i] == 0 (the others are left
 *   alone), x to x + i*stride_x.  Together they replace factor_blocked_serial
 *   (pkg/src/bandchol/blocked.py:363-385) + solve_with_factor (pkg/src/bandchol/core.py:216-240),
 *   whose forward loop (:231-235) and backward loop (:236-239) they split. */
int bcg_dpbtrf_fwd_batched(int64_t n, int64_t kd, double* ab, int64_t ldab, int64_t stride_ab,
                           const double* b, int64_t stride_b, int64_t batch, int32_t* info,
                           double* y, void* stream);
int bcg_dpbtrs_bwd_batched(int64_t n, int64_t kd, const double* ab, int64_t ldab, int64_t stride_ab,
                           const double* y, double* x, int64_t stride_x, int64_t batch,
                           int32_t* info, void* stream);

/* Diagnostics: per-step phase timestamps of the whole-GPU factorization, the
 * analogue of the reference's per-task trace (pkg/src/bandchol/parallel.py:54-62).
 * Subsequent bcg_dpbtrf launches on the multi-CTA path write uint64 %globaltimer
 * nanoseconds into device_buffer: [0] = steps recorded, then 8 stamps per block
 * step (potrf start/end, L published, waits done, loads done, updates done,
 * next panel published).  NULL disables tracing. */
int bcg_set_trace(void* device_buffer, size_t bytes);

/* Backward error ||A - L L^T||_F / ||A||_F over the band, on the device: the GPU
 * restatement of the reference's residual_norm (pkg/src/bandchol/core.py:186-213) --
 * off-diagonal entries weighted twice, result 0 for A = 0 = L L^T, +inf for A = 0 != L L^T.
 * a: the original matrix (lda), l: its factor (ldl), both device AB storage; *result
 * (device) receives the residual.  Deterministic (fixed-order reductions in workspace,
 * >= bcg_band_residual_workspace_size() bytes).  Asynchronous on stream. */
size_t bcg_band_residual_workspace_size(void);
int bcg_band_residual(int64_t n, int64_t kd, const double* a, int64_t lda, const double* l, int64_t ldl,
                      double* result, void* workspace, size_t workspace_bytes, void* stream);

/* Batched backward error: result[i] (device double[batch]) = the residual of matrix i,
 * a + i*stride_a against l + i*stride_l (the all-members parity gate of config C5).
 * Deterministic; workspace >= bcg_band_residual_batched_workspace_size(batch) bytes;
 * batch <= 65535.  Asynchronous on stream. */
size_t bcg_band_residual_batched_workspace_size(int64_t batch);
int bcg_band_residual_batched(int64_t n, int64_t kd, const double* a, int64_t lda, int64_t stride_a,
                              const double* l, int64_t ldl, int64_t stride_l, int64_t batch,
                              double* result, void* workspace, size_t workspace_bytes, void* stream);

/* Measurement utility (bench.py): FP64 FMA-pipe peak of the current device in
 * TFLOP/s, from a register-only DFMA loop over every SM (synchronous, ~10 ms).
 * The roofline denominator for the FP64-bound configs. */
int bcg_probe_fp64_peak(double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* BANDCHOL_B200_H */
