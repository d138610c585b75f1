// bandchol_b200.cu -- kernels and C ABI of libbandchol_b200.so (see include/bandchol_b200.h).
//
// Entry points replace the reference's factorization engines and solve:
//   bcg_dpbtrf / bcg_dpbtrf_batched  <- factor_blocked_serial (pkg/src/bandchol/blocked.py:363-385),
//                                       factor_blocked_parallel (pkg/src/bandchol/parallel.py:130-166)
//   bcg_dpbtrs / bcg_dpbtrs_batched(_nrhs)  <- solve_with_factor (pkg/src/bandchol/core.py:216-240),
//                                       up to 16 right-hand sides per pass over L
//   bcg_dpbsv_batched                <- factor + solve of config C5: the batched factorization
//                                       kernel, then the streamed solve kernel
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/bandchol_b200.h"
#include "band_cta.cuh"
#include "band_solve.cuh"
#include "band_sweep.cuh"
#include "band_residual.cuh"
#include "band_multi.cuh"

namespace bcg {

// One CTA per matrix (grid-stride over the batch).
template <int NB, int KD>
__global__ void __launch_bounds__(kCtaThreads, 2)
pbtrf_cta_kernel(double* ab0, int64_t stride_ab, int batch, CtaGeom g, int32_t* info, const double* b0,
                 int64_t stride_b, double* y0) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) unsigned long long bars[1];
  __shared__ int s_sp[kCtaWarps];
  __shared__ __align__(8) unsigned long long sig[5];
  if (threadIdx.x == 0) mbar_init(&bars[0], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  unsigned phase = 0;
  for (int mat = blockIdx.x; mat < batch; mat += gridDim.x) {
    CtaBand<NB, KD> w{g};
    w.bars = bars;
    w.phase = phase;
    w.set_roles(s_sp);
    w.tr = (blockIdx.x == 0 && mat == 0) ? g_trace : nullptr;
    w.ab = ab0 + (int64_t)mat * stride_ab;
    double* p = smem;
    w.win = p; p += (size_t)g.nslot * g.lds;
    w.P = p; p += cta_panel_doubles(NB, g);
    w.D = p; p += 2 * NB * (NB + 4);
    w.lbuf = p; p += NB;
    w.fws = p;
    if (b0) {  // fused forward sweep (dpbsv): y to the caller's workspace, n doubles per matrix
      w.fb = b0 + (int64_t)mat * stride_b;
      w.fy = y0 + (int64_t)mat * g.n;
    }
    w.sig = sig;
    const int fail = w.factor();
    phase = w.phase;
    if (threadIdx.x == 0) info[mat] = fail < 0 ? 0 : fail + 1;
    __syncthreads();
  }
}

}  // namespace bcg

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
namespace {

thread_local char g_err[512] = "";

int fail_arg(int idx, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return -idx;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
  return (int)e;
}

// Device attributes of the CURRENT device (the one every launch goes to), cached per
// device ordinal.
constexpr int kMaxDevices = 64;

int device_attr(cudaDeviceAttr attr, int fallback, int (&cache)[kMaxDevices]) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return fallback;
  int v = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess || v <= 0) return fallback;
    __atomic_store_n(&cache[dev], v, __ATOMIC_RELAXED);
  }
  return v;
}

int smem_optin() {
  static int cache[kMaxDevices];
  return device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 48 * 1024, cache);
}

int sm_count() {
  static int cache[kMaxDevices];
  return device_attr(cudaDevAttrMultiProcessorCount, 148, cache);
}

bcg::CtaGeom make_geom(int n, int kd, int ldab, int nb) {
  bcg::CtaGeom g;
  g.n = n;
  g.kd = kd;
  g.ldab = ldab;
  g.lds = ldab;  // ring slots mirror the global columns (bulk copies move whole columns)
  int ns = kd + nb;
  if (ns & 1) ++ns;
  g.nslot = ns;
  // >= kd rows, = 4 (mod 16): conflict-free DMMA fragment loads.  The tile GEMM reads (and
  // discards) up to 12 rows past kd, i.e. into the next column or the buffer after P.
  int pld = kd + ((4 - kd % 16) + 16) % 16;
  g.pld = pld;
  return g;
}

// Block size for the one-CTA-per-matrix kernel (NB = 16) when its window fits two
// CTAs per SM, else one; 0 if the window does not fit at all.
int cta_block(int n, int kd, int ldab, bcg::CtaGeom* out) {
  const size_t limit = (size_t)smem_optin();
  const size_t half = 113 * 1024 - 512;  // two CTAs per SM: 228 KB less 1 KB per CTA and the static smem
  for (size_t cap : {half, limit}) {
    const int nb = 16;
    bcg::CtaGeom g = make_geom(n, kd, ldab, nb);
    if (bcg::cta_smem_bytes(nb, g) > cap) continue;
    *out = g;
    return nb;
  }
  return 0;
}

int launch_cta(double* ab, int64_t sab, int batch, const bcg::CtaGeom& g, int32_t* info, cudaStream_t st,
               const double* b = nullptr, int64_t sb = 0, double* y = nullptr) {
  constexpr int NB = 16;
  const size_t smem = bcg::cta_smem_bytes(NB, g);
  // common band widths get a compile-time-geometry instantiation (constant strides: C5
  // 3.67 -> 3.51 ms for 1024 matrices); other widths keep the runtime geometry
  // (a small set of band widths, each ~4-5 % faster than the runtime geometry; ldab = kd + 1)
  auto k = bcg::pbtrf_cta_kernel<NB, 0>;
  if (bcg::GeomFixed<100>::matches(g)) k = bcg::pbtrf_cta_kernel<NB, 100>;
  else if (bcg::GeomFixed<50>::matches(g)) k = bcg::pbtrf_cta_kernel<NB, 50>;
  else if (bcg::GeomFixed<64>::matches(g)) k = bcg::pbtrf_cta_kernel<NB, 64>;
  else if (bcg::GeomFixed<128>::matches(g)) k = bcg::pbtrf_cta_kernel<NB, 128>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
  k<<<batch, bcg::kCtaThreads, smem, st>>>(ab, sab, batch, g, info, b, sb, y);
  return cuda_status(cudaGetLastError(), "pbtrf_cta_kernel launch");
}

int check_geom(int64_t n, int64_t kd, int64_t ldab) {
  if (n < 1 || n > INT_MAX / 2) return fail_arg(1, "n=%lld out of range", (long long)n);
  if (kd < 0 || kd >= n) return fail_arg(2, "kd=%lld invalid for n=%lld", (long long)kd, (long long)n);
  if (ldab < kd + 1 || ldab > INT_MAX / 2) return fail_arg(4, "ldab=%lld < kd+1", (long long)ldab);
  return 0;
}

}  // namespace

// Streamed solve (band_sweep.cuh): a ring of nbuf 16-column buffers, the deepest ring that
// keeps two CTAs per SM (else one); 0 when not even four buffers fit (wide bands), where
// the direct-from-L2 kernel runs instead.
static bcg::SweepGeom sweep_geom(int n, int kd, int ldab, int R) {
  bcg::SweepGeom g;
  g.n = n;
  g.kd = kd;
  g.ldab = ldab;
  g.nblk = (n + 15) / 16;
  g.nx = 16 * ((kd + 16 + 15) / 16);
  g.nbuf = 0;
  // per-CTA budgets for two and one CTAs per SM (228 KB less 1 KB per CTA and the static
  // shared memory)
  const size_t two = (size_t)(112 * 1024), one = (size_t)smem_optin() - 1024;
  for (size_t cap : {two, one}) {
    for (int nb = 8; nb >= 4; --nb) {
      g.nbuf = nb;
      if (bcg::sweep_smem_doubles(g, R) * sizeof(double) <= cap) return g;
    }
  }
  g.nbuf = 0;
  return g;
}

// right-hand sides per CTA: 1 and 2 on the FMA path; 3..8 one 8-wide DMMA n-tile (measured
// faster for 4 than the FMA path), more: 16 per CTA (two n-tiles)
static int sweep_r(int64_t nrhs) { return nrhs <= 1 ? 1 : nrhs <= 2 ? 2 : nrhs <= 8 ? 8 : 16; }

template <int R>
static int launch_sweep_t(const double* ab, int64_t sab, double* b, int64_t ldb, int64_t sb, int nrhs, int batch,
                          const bcg::SweepGeom& g, int32_t* info, cudaStream_t st, const int32_t* skip,
                          const double* y, int64_t sy) {
  const size_t smem = bcg::sweep_smem_doubles(g, R) * sizeof(double);
  auto k = bcg::pbtrs_sweep_kernel<R>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(pbtrs_sweep)");
  const int groups = (nrhs + R - 1) / R;
  k<<<(unsigned)((int64_t)batch * groups), bcg::kSweepThreads, smem, st>>>(ab, sab, b, ldb, sb, nrhs, groups, g, info,
                                                                           skip, skip ? 0 : 1, y, sy);
  return cuda_status(cudaGetLastError(), "pbtrs_sweep_kernel launch");
}

// Solve `batch` systems, each with nrhs right-hand sides (column r of matrix m at
// b + m*sb + r*ldb).  skip (device, may be NULL): matrices with skip[m] != 0 are left alone
// (their factorization failed); with skip the diagonal check is not repeated.
// y (device, may be NULL; nrhs = 1 only): the forward sweep is already done -- y of matrix m at
// y + m*sy (the fused factorization wrote it) -- and only the backward sweep runs, x to b.
static int launch_solve(const double* ab, int64_t sab, double* b, int64_t ldb, int64_t sb, int nrhs, int batch,
                        int n, int kd, int ldab, int32_t* info, cudaStream_t st, const int32_t* skip = nullptr,
                        const double* y = nullptr, int64_t sy = 0) {
  const int R = sweep_r(nrhs);
  const bcg::SweepGeom g = sweep_geom(n, kd, ldab, R);
  if (g.nbuf) {
    switch (R) {
      case 1: return launch_sweep_t<1>(ab, sab, b, ldb, sb, nrhs, batch, g, info, st, skip, y, sy);
      case 2: return launch_sweep_t<2>(ab, sab, b, ldb, sb, nrhs, batch, g, info, st, skip, y, sy);
      case 8: return launch_sweep_t<8>(ab, sab, b, ldb, sb, nrhs, batch, g, info, st, skip, y, sy);
      default: return launch_sweep_t<16>(ab, sab, b, ldb, sb, nrhs, batch, g, info, st, skip, y, sy);
    }
  }
  if (y) return fail_arg(0, "internal: backward-only solve needs the streamed kernel");
  // wide bands: one CTA per right-hand side straight from L2
  bcg::pbtrs_kernel<<<(unsigned)((int64_t)batch * nrhs), bcg::kCtaThreads, 0, st>>>(ab, sab, b, ldb, sb, nrhs, n, kd,
                                                                                     ldab, info, skip);
  return cuda_status(cudaGetLastError(), "pbtrs_kernel launch");
}

extern "C" {

int bcg_version(void) { return 200; }

const char* bcg_last_error(void) { return g_err; }

// Single matrices: one CTA when the window fits in shared memory, else the
// whole-GPU dataflow kernel (which needs the caller's workspace).
static bool single_uses_multi(int n, int kd, int ldab) {
  bcg::CtaGeom g;
  return cta_block(n, kd, ldab, &g) == 0 || bcg::use_multi(n, kd);
}

size_t bcg_dpbtrf_workspace_size(int64_t n, int64_t kd, int64_t ldab) {
  if (check_geom(n, kd, ldab) != 0) return 0;
  if (!single_uses_multi((int)n, (int)kd, (int)ldab)) return 0;
  return bcg::multi_workspace_bytes((int)n, (int)kd);
}

int bcg_dpbtrf(int64_t n, int64_t kd, double* ab, int64_t ldab, int32_t* info, void* workspace,
               size_t workspace_bytes, void* stream) {
  if (int r = check_geom(n, kd, ldab)) return r;
  if (!ab) return fail_arg(3, "ab is NULL");
  if (!info) return fail_arg(5, "info is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  if (single_uses_multi((int)n, (int)kd, (int)ldab)) {
    const size_t need = bcg::multi_workspace_bytes((int)n, (int)kd);
    if (!workspace || workspace_bytes < need)
      return fail_arg(6, "workspace of %zu bytes required (got %zu)", need, workspace_bytes);
    return bcg::launch_multi(ab, (int)n, (int)kd, (int)ldab, info, workspace, sm_count(), st, g_err, sizeof g_err);
  }
  bcg::CtaGeom g;
  cta_block((int)n, (int)kd, (int)ldab, &g);
  return launch_cta(ab, 0, 1, g, info, st);
}

// Batched matrices whose window does not fit one CTA: one whole-GPU factorization
// after another, on the caller's workspace (cleared by every launch, stream-ordered).
static int batched_multi(int n, int kd, int ldab, double* ab, int64_t stride_ab, int batch, int32_t* info,
                         void* ws, cudaStream_t st) {
  int rc = 0;
  for (int i = 0; i < batch && rc == 0; ++i)
    rc = bcg::launch_multi(ab + (int64_t)i * stride_ab, n, kd, ldab, info + i, ws, sm_count(), st, g_err,
                           sizeof g_err);
  return rc;
}

static bool batched_uses_multi(int n, int kd, int ldab) {
  bcg::CtaGeom g;
  return cta_block(n, kd, ldab, &g) == 0;
}

size_t bcg_dpbtrf_batched_workspace_size(int64_t n, int64_t kd, int64_t ldab, int64_t batch) {
  if (check_geom(n, kd, ldab) != 0 || batch <= 0) return 0;
  if (!batched_uses_multi((int)n, (int)kd, (int)ldab)) return 0;
  return bcg::multi_workspace_bytes((int)n, (int)kd);
}

// fused path of bcg_dpbsv_batched: pipelined one-CTA factorization (32 <= kd, window in shared
// memory) and the streamed solve kernel both apply
static bool dpbsv_fused(int n, int kd, int ldab, bcg::CtaGeom* g) {
  return kd >= 32 && cta_block(n, kd, ldab, g) != 0 && sweep_geom(n, kd, ldab, 1).nbuf != 0;
}

size_t bcg_dpbsv_batched_workspace_size(int64_t n, int64_t kd, int64_t ldab, int64_t batch) {
  if (check_geom(n, kd, ldab) != 0 || batch <= 0) return 0;
  bcg::CtaGeom g;
  if (dpbsv_fused((int)n, (int)kd, (int)ldab, &g)) return (size_t)batch * (size_t)n * sizeof(double);
  return bcg_dpbtrf_batched_workspace_size(n, kd, ldab, batch);
}

int bcg_dpbtrf_batched(int64_t n, int64_t kd, double* ab, int64_t ldab, int64_t stride_ab, int64_t batch,
                       int32_t* info, void* workspace, size_t workspace_bytes, void* stream) {
  if (int r = check_geom(n, kd, ldab)) return r;
  if (!ab) return fail_arg(3, "ab is NULL");
  if (stride_ab < ldab * n) return fail_arg(5, "stride_ab < ldab*n");
  if (batch < 0 || batch > INT_MAX) return fail_arg(6, "batch out of range");
  if (!info) return fail_arg(7, "info is NULL");
  if (batch == 0) return 0;
  bcg::CtaGeom g;
  if (cta_block((int)n, (int)kd, (int)ldab, &g) == 0) {
    const size_t need = bcg::multi_workspace_bytes((int)n, (int)kd);
    if (!workspace || workspace_bytes < need)
      return fail_arg(8, "workspace of %zu bytes required (got %zu)", need, workspace_bytes);
    return batched_multi((int)n, (int)kd, (int)ldab, ab, stride_ab, (int)batch, info, workspace,
                         (cudaStream_t)stream);
  }
  return launch_cta(ab, stride_ab, (int)batch, g, info, (cudaStream_t)stream);
}


static int check_dpbsv_args(int64_t n, int64_t kd, const double* ab, int64_t ldab, int64_t stride_ab, const double* b,
                            int64_t stride_b, int64_t batch, const int32_t* info) {
  if (int r = check_geom(n, kd, ldab)) return r;
  if (!ab) return fail_arg(3, "ab is NULL");
  if (stride_ab < ldab * n) return fail_arg(5, "stride_ab < ldab*n");
  if (!b) return fail_arg(6, "b is NULL");
  if (stride_b < n) return fail_arg(7, "stride_b < n");
  if (batch < 0 || batch > INT_MAX) return fail_arg(8, "batch out of range");
  if (!info) return fail_arg(9, "info is NULL");
  return 0;
}

int bcg_dpbtrf_fwd_batched(int64_t n, int64_t kd, double* ab, int64_t ldab, int64_t stride_ab, const double* b,
                           int64_t stride_b, int64_t batch, int32_t* info, double* y, void* stream) {
  if (int r = check_dpbsv_args(n, kd, ab, ldab, stride_ab, b, stride_b, batch, info)) return r;
  if (!y || (((uintptr_t)y) & 7)) return fail_arg(10, "y is NULL or misaligned");
  bcg::CtaGeom g;
  if (!dpbsv_fused((int)n, (int)kd, (int)ldab, &g))
    return fail_arg(2, "fused factorization + forward sweep needs 32 <= kd and a band window that fits one CTA");
  if (batch == 0) return 0;
  return launch_cta(ab, stride_ab, (int)batch, g, info, (cudaStream_t)stream, b, stride_b, y);
}

int bcg_dpbtrs_bwd_batched(int64_t n, int64_t kd, const double* ab, int64_t ldab, int64_t stride_ab, const double* y,
                           double* x, int64_t stride_x, int64_t batch, int32_t* info, void* stream) {
  if (int r = check_dpbsv_args(n, kd, ab, ldab, stride_ab, x, stride_x, batch, info)) return r;
  if (!y) return fail_arg(6, "y is NULL");
  if (sweep_geom((int)n, (int)kd, (int)ldab, 1).nbuf == 0)
    return fail_arg(2, "the backward-only sweep needs a band whose 16-column ring fits shared memory");
  if (batch == 0) return 0;
  return launch_solve(ab, stride_ab, x, n, stride_x, 1, (int)batch, (int)n, (int)kd, (int)ldab, info,
                      (cudaStream_t)stream, info, y, n);
}

int bcg_dpbsv_batched(int64_t n, int64_t kd, double* ab, int64_t ldab, int64_t stride_ab, double* b,
                      int64_t stride_b, int64_t batch, int32_t* info, void* workspace, size_t workspace_bytes,
                      void* stream) {
  if (int r = check_dpbsv_args(n, kd, ab, ldab, stride_ab, b, stride_b, batch, info)) return r;
  if (batch == 0) return 0;
  // With a workspace for y: the factorization kernel's light warp runs the forward sweep
  // L y = b right behind each panel, from shared memory (y to the workspace: b stays untouched
  // until the matrix is known to have factored), and the solve kernel only sweeps backward,
  // skipping the matrices that failed.
  bcg::CtaGeom g;
  if (dpbsv_fused((int)n, (int)kd, (int)ldab, &g) && workspace &&
      workspace_bytes >= (size_t)batch * (size_t)n * sizeof(double) && !(((uintptr_t)workspace) & 7)) {
    double* y = (double*)workspace;
    if (int rc = bcg_dpbtrf_fwd_batched(n, kd, ab, ldab, stride_ab, b, stride_b, batch, info, y, stream)) return rc;
    return bcg_dpbtrs_bwd_batched(n, kd, ab, ldab, stride_ab, y, b, stride_b, batch, info, stream);
  }
  // otherwise: the batched factorization, then the two-sweep solve, which skips the matrices
  // whose factorization failed (their b stays untouched, as LAPACK dpbsv leaves B when info > 0)
  if (int rc = bcg_dpbtrf_batched(n, kd, ab, ldab, stride_ab, batch, info, workspace, workspace_bytes, stream))
    return rc;
  return launch_solve(ab, stride_ab, b, n, stride_b, 1, (int)batch, (int)n, (int)kd, (int)ldab, info,
                      (cudaStream_t)stream, info);
}

int bcg_dpbtrs(int64_t n, int64_t kd, const double* ab, int64_t ldab, double* b, int64_t ldb, int64_t nrhs,
               int32_t* info, void* stream) {
  if (int r = check_geom(n, kd, ldab)) return r;
  if (!ab) return fail_arg(3, "ab is NULL");
  if (!b) return fail_arg(5, "b is NULL");
  if (nrhs < 0 || nrhs > INT_MAX) return fail_arg(7, "nrhs out of range");
  if (nrhs > 1 && ldb < n) return fail_arg(6, "ldb < n");
  if (!info) return fail_arg(8, "info is NULL");
  if (nrhs == 0) return 0;
  return launch_solve(ab, 0, b, ldb, 0, (int)nrhs, 1, (int)n, (int)kd, (int)ldab, info, (cudaStream_t)stream);
}

int bcg_dpbtrs_batched(int64_t n, int64_t kd, const double* ab, int64_t ldab, int64_t stride_ab, double* b,
                       int64_t stride_b, int64_t batch, int32_t* info, void* stream) {
  return bcg_dpbtrs_batched_nrhs(n, kd, ab, ldab, stride_ab, b, n, stride_b, 1, batch, info, stream);
}

int bcg_dpbtrs_batched_nrhs(int64_t n, int64_t kd, const double* ab, int64_t ldab, int64_t stride_ab, double* b,
                            int64_t ldb, int64_t stride_b, int64_t nrhs, int64_t batch, int32_t* info, void* stream) {
  if (int r = check_geom(n, kd, ldab)) return r;
  if (!ab) return fail_arg(3, "ab is NULL");
  if (stride_ab < ldab * n) return fail_arg(5, "stride_ab < ldab*n");
  if (!b) return fail_arg(6, "b is NULL");
  if (nrhs > 1 && ldb < n) return fail_arg(7, "ldb < n");
  if (stride_b < (nrhs > 1 ? ldb * (nrhs - 1) + n : n)) return fail_arg(8, "stride_b smaller than one matrix's rhs");
  if (nrhs < 0 || nrhs > INT_MAX) return fail_arg(9, "nrhs out of range");
  if (batch < 0 || batch > INT_MAX || batch * ((nrhs + 15) / 16) > INT_MAX) return fail_arg(10, "batch out of range");
  if (!info) return fail_arg(11, "info is NULL");
  if (batch == 0 || nrhs == 0) return 0;
  return launch_solve(ab, stride_ab, b, ldb, stride_b, (int)nrhs, (int)batch, (int)n, (int)kd, (int)ldab, info,
                      (cudaStream_t)stream);
}

}  // extern "C"

// ----------------------------------------------------------------------------
// measurement utility: FP64 FMA-pipe peak (roofline denominator)
// ----------------------------------------------------------------------------
namespace bcg {
__global__ void __launch_bounds__(512) dfma_probe_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}
}  // namespace bcg

extern "C" int bcg_set_trace(void* device_buffer, size_t bytes) {
  unsigned long long* p = (unsigned long long*)device_buffer;
  unsigned long long cap = device_buffer ? bytes / sizeof(unsigned long long) : 0;
  if (int r = cuda_status(cudaMemcpyToSymbol(bcg::g_trace, &p, sizeof p), "cudaMemcpyToSymbol(trace)")) return r;
  return cuda_status(cudaMemcpyToSymbol(bcg::g_trace_cap, &cap, sizeof cap), "cudaMemcpyToSymbol(trace cap)");
}

extern "C" int bcg_probe_fp64_peak(double* tflops) {
  if (!tflops) return fail_arg(1, "tflops is NULL");
  double* d = nullptr;
  if (int r = cuda_status(cudaMalloc(&d, sizeof(double)), "cudaMalloc")) return r;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sm_count() * 4, tpb = 512, iters = 1024;
  bcg::dfma_probe_kernel<<<blocks, tpb>>>(d, 16);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    bcg::dfma_probe_kernel<<<blocks, tpb>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_status(e, "dfma_probe_kernel");
  *tflops = 2.0 * 64.0 * iters * (double)blocks * tpb / (best * 1e-3) / 1e12;
  return 0;
}

// ---- device residual --------------------------------------------
static int residual_blocks() { return sm_count() * 8; }

extern "C" size_t bcg_band_residual_workspace_size(void) {
  return (size_t)residual_blocks() * 2 * sizeof(double);
}

extern "C" int bcg_band_residual(int64_t n, int64_t kd, const double* a, int64_t lda, const double* l, int64_t ldl,
                                 double* result, void* workspace, size_t workspace_bytes, void* stream) {
  if (int r = check_geom(n, kd, lda)) return r;
  if (ldl < kd + 1 || ldl > INT_MAX / 2) return fail_arg(6, "ldl=%lld < kd+1", (long long)ldl);
  if (!a) return fail_arg(3, "a is NULL");
  if (!l) return fail_arg(5, "l is NULL");
  if (!result) return fail_arg(7, "result is NULL");
  const int blocks = residual_blocks();
  if (!workspace || workspace_bytes < (size_t)blocks * 2 * sizeof(double))
    return fail_arg(8, "workspace smaller than bcg_band_residual_workspace_size()");
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)workspace;
  bcg::band_residual_kernel<<<blocks, bcg::kResidThreads, 0, st>>>((int)n, (int)kd, a, (int)lda, l, (int)ldl, part);
  bcg::band_residual_finish<<<1, 32, 0, st>>>(part, blocks, result);
  return cuda_status(cudaGetLastError(), "band_residual_kernel launch");
}

// batched: kResidBatchBlocks blocks per matrix
static constexpr int kResidBatchBlocks = 4;

extern "C" size_t bcg_band_residual_batched_workspace_size(int64_t batch) {
  return batch < 0 ? 0 : (size_t)batch * kResidBatchBlocks * 2 * sizeof(double);
}

extern "C" int bcg_band_residual_batched(int64_t n, int64_t kd, const double* a, int64_t lda, int64_t stride_a,
                                         const double* l, int64_t ldl, int64_t stride_l, int64_t batch,
                                         double* result, void* workspace, size_t workspace_bytes, void* stream) {
  if (int r = check_geom(n, kd, lda)) return r;
  if (!a) return fail_arg(3, "a is NULL");
  if (stride_a < lda * n) return fail_arg(5, "stride_a < lda*n");
  if (!l) return fail_arg(6, "l is NULL");
  if (ldl < kd + 1 || ldl > INT_MAX / 2) return fail_arg(7, "ldl=%lld < kd+1", (long long)ldl);
  if (stride_l < ldl * n) return fail_arg(8, "stride_l < ldl*n");
  if (batch < 0 || batch > 65535) return fail_arg(9, "batch out of range [0, 65535]");
  if (!result) return fail_arg(10, "result is NULL");
  if (batch == 0) return 0;
  if (!workspace || workspace_bytes < bcg_band_residual_batched_workspace_size(batch))
    return fail_arg(11, "workspace smaller than bcg_band_residual_batched_workspace_size(batch)");
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)workspace;
  bcg::band_residual_kernel<<<dim3(kResidBatchBlocks, (unsigned)batch), bcg::kResidThreads, 0, st>>>(
      (int)n, (int)kd, a, (int)lda, l, (int)ldl, part, stride_a, stride_l);
  bcg::band_residual_finish<<<(unsigned)((batch + 127) / 128), 128, 0, st>>>(part, kResidBatchBlocks, result,
                                                                              (int)batch);
  return cuda_status(cudaGetLastError(), "band_residual_kernel launch (batched)");
}
