// bandchol_b200.cu -- kernels and C ABI of libbandchol_b200.so (see include/bandchol_b200.h).
//
// Entry points replace the reference's factorization engines and solve:
//   bcg_dpbtrf / bcg_dpbtrf_batched  <- factor_blocked_serial (pkg/src/bandchol/blocked.py:363-385),
//                                       factor_blocked_parallel (pkg/src/bandchol/parallel.py:130-166)
//   bcg_dpbtrs / bcg_dpbtrs_batched  <- solve_with_factor (pkg/src/bandchol/core.py:216-240)
//   bcg_dpbsv_batched                <- factor + solve of config C5 fused in one launch
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/bandchol_b200.h"
#include "band_cta.cuh"
#include "band_solve.cuh"
#include "band_residual.cuh"
#include "band_multi.cuh"

namespace bcg {

// One CTA per matrix (grid-stride over the batch).
template <int NB, bool kSolve, int KD>
__global__ void __launch_bounds__(kCtaThreads, 2)
pbtrf_cta_kernel(double* ab0, int64_t stride_ab, double* b0, int64_t stride_b, int batch, CtaGeom g,
                 int32_t* info) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) unsigned long long bars[1 + 16];
  __shared__ unsigned bphase[16];
  __shared__ int s_sp[kCtaWarps];
  __shared__ __align__(8) unsigned long long sig[4];
  if (threadIdx.x < 17) mbar_init(&bars[threadIdx.x], 1);
  if (threadIdx.x < 16) bphase[threadIdx.x] = 0;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  unsigned phase = 0;
  for (int mat = blockIdx.x; mat < batch; mat += gridDim.x) {
    CtaBand<NB, kSolve, KD> w{g};
    w.bars = bars;
    w.bphase = bphase;
    w.phase = phase;
    w.set_roles(s_sp);
    w.tr = (blockIdx.x == 0 && mat == 0) ? g_trace : nullptr;
    w.ab = ab0 + (int64_t)mat * stride_ab;
    w.rhs = kSolve ? b0 + (int64_t)mat * stride_b : nullptr;
    double* p = smem;
    w.win = p; p += (size_t)g.nslot * g.lds;
    w.P = p; p += cta_panel_doubles(NB, g, kSolve);
    w.D = p; p += 2 * NB * (NB + 4);
    w.Dinv = w.D + NB * (NB + 4);
    w.lbuf = p; p += NB;
    w.sig = sig;
    w.bw = kSolve ? p : nullptr;
    if (kSolve) p += g.nslot;
    w.yb = kSolve ? p : nullptr;
    const int fail = w.factor();
    phase = w.phase;
    if (kSolve && fail < 0) w.backward();
    if (threadIdx.x == 0) info[mat] = fail < 0 ? 0 : fail + 1;
    __syncthreads();
  }
}

// Standalone solve, one CTA per right-hand side: forward and backward sweeps stream the
// factor's column blocks through a 5-buffer shared ring (see CtaBand::forward/backward).
__global__ void __launch_bounds__(kCtaThreads, 2)
pbtrs_cta_kernel(const double* ab0, int64_t stride_ab, double* b0, int64_t stride_b, int nrhs, CtaGeom g,
                 int32_t* info, const int32_t* skip) {
  constexpr int NB = 16;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) unsigned long long bars[1 + 16];
  __shared__ unsigned bphase[16];
  if (threadIdx.x < 17) mbar_init(&bars[threadIdx.x], 1);
  if (threadIdx.x < 16) bphase[threadIdx.x] = 0;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int z = blockIdx.x, mat = z / nrhs;
  if (skip && skip[mat] != 0) return;  // (after a batched factorization: this one failed, keep its info)
  const double* abm = ab0 + (int64_t)mat * stride_ab;
  const int bad = first_nonpositive_diag(abm, g.n, g.ldab);
  if (bad != INT_MAX) {
    if (threadIdx.x == 0 && z % nrhs == 0) info[mat] = bad + 1;
    return;
  }
  CtaBand<NB, true> w{g};
  w.bars = bars;
  w.bphase = bphase;
  w.ab = const_cast<double*>(abm);
  w.rhs = b0 + (int64_t)z * stride_b;
  w.tr = (z == 0) ? g_trace : nullptr;
  double* p = smem;
  w.win = p; p += (size_t)g.nslot * g.lds;
  w.P = p; p += cta_panel_doubles(NB, g, true);
  w.D = p; p += 2 * NB * (NB + 4);
  w.Dinv = w.D + NB * (NB + 4);
  w.lbuf = p; p += NB;
  w.bw = p; p += g.nx;
  w.yb = p;
  w.init_fast();
  w.forward();
  w.backward();
  if (threadIdx.x == 0 && z % nrhs == 0) info[mat] = 0;
}

__global__ void __launch_bounds__(kCtaThreads)
pbtrs_kernel(const double* ab0, int64_t stride_ab, double* b0, int64_t stride_b, int nrhs, int n, int kd,
             int ldab, int32_t* info) {
  const int z = blockIdx.x;
  const double* ab = ab0 + (int64_t)(z / nrhs) * stride_ab;
  double* b = b0 + (int64_t)z * stride_b;
  const int bad = first_nonpositive_diag(ab, n, ldab);
  if (bad != INT_MAX) {
    if (threadIdx.x == 0) info[z / nrhs] = bad + 1;
    return;
  }
  band_forward(ab, n, kd, ldab, b);
  band_backward(ab, n, kd, ldab, b);
  if (threadIdx.x == 0 && z % nrhs == 0) info[z / nrhs] = 0;
}

// Solve step of the unfused dpbsv path: matrices whose factorization failed keep info.
__global__ void __launch_bounds__(kCtaThreads)
pbtrs_after_factor_kernel(const double* ab0, int64_t stride_ab, double* b0, int64_t stride_b, int n, int kd,
                          int ldab, const int32_t* info) {
  const int z = blockIdx.x;
  if (info[z] != 0) return;
  const double* ab = ab0 + (int64_t)z * stride_ab;
  double* b = b0 + (int64_t)z * stride_b;
  band_forward(ab, n, kd, ldab, b);
  band_backward(ab, n, kd, ldab, b);
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

int smem_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) v = 48 * 1024;
  }
  return v;
}

int sm_count() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
  }
  return v;
}

bcg::CtaGeom make_geom(int n, int kd, int ldab, int nb, bool solve) {
  bcg::CtaGeom g;
  g.n = n;
  g.kd = kd;
  g.ldab = ldab;
  g.lds = ldab;  // ring slots mirror the global columns (bulk copies move whole columns)
  int ns = kd + nb;
  if (solve && ns < 5 * nb) ns = 5 * nb;  // backward-sweep prefetch ring: 5 blocks
  if (ns & 1) ++ns;
  g.nslot = ns;
  g.nx = ns;
  // >= kd rows, = 4 (mod 16): conflict-free DMMA fragment loads.  The tile GEMM reads (and
  // discards) up to 12 rows past kd, i.e. into the next column or the buffer after P.
  int pld = kd + ((4 - kd % 16) + 16) % 16;
  g.pld = pld;
  return g;
}

// Block size for the one-CTA-per-matrix kernel (NB = 16) when its window fits two
// CTAs per SM, else one; 0 if the window does not fit at all.
int cta_block(int n, int kd, int ldab, bool solve, bcg::CtaGeom* out) {
  const size_t limit = (size_t)smem_optin();
  const size_t half = 113 * 1024 - 512;  // two CTAs per SM: 228 KB less 1 KB per CTA and the static smem
  for (size_t cap : {half, limit}) {
    const int nb = 16;
    bcg::CtaGeom g = make_geom(n, kd, ldab, nb, solve);
    if (bcg::cta_smem_bytes(nb, g, solve) > cap) continue;
    *out = g;
    return nb;
  }
  return 0;
}

template <int NB, bool S>
int launch_cta_t(double* ab, int64_t sab, double* b, int64_t sb, int batch, const bcg::CtaGeom& g, int32_t* info,
                 cudaStream_t st) {
  const size_t smem = bcg::cta_smem_bytes(NB, g, S);
  // the C5 band width gets a compile-time-geometry instantiation of the factorization (constant
  // strides: 3.67 -> 3.51 ms for 1024 matrices); measured slower for the fused solve and for
  // kd = 50, which keep the runtime geometry
  auto k = (!S && bcg::GeomFixed<100, S>::matches(g)) ? bcg::pbtrf_cta_kernel<NB, S, S ? 0 : 100>
                                                       : bcg::pbtrf_cta_kernel<NB, S, 0>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
  k<<<batch, bcg::kCtaThreads, smem, st>>>(ab, sab, b, sb, batch, g, info);
  return cuda_status(cudaGetLastError(), "pbtrf_cta_kernel launch");
}

int launch_cta(double* ab, int64_t sab, double* b, int64_t sb, int batch, int nb, const bcg::CtaGeom& g,
               int32_t* info, bool solve, cudaStream_t st) {
  (void)nb;  // 16: the smallest block has the shortest per-step chain and window
  if (solve) return launch_cta_t<16, true>(ab, sab, b, sb, batch, g, info, st);
  return launch_cta_t<16, false>(ab, sab, b, sb, batch, g, info, st);
}

int check_geom(int64_t n, int64_t kd, int64_t ldab) {
  if (n < 1 || n > INT_MAX / 2) return fail_arg(1, "n=%lld out of range", (long long)n);
  if (kd < 0 || kd >= n) return fail_arg(2, "kd=%lld invalid for n=%lld", (long long)kd, (long long)n);
  if (ldab < kd + 1 || ldab > INT_MAX / 2) return fail_arg(4, "ldab=%lld < kd+1", (long long)ldab);
  return 0;
}

}  // namespace

extern "C" {

int bcg_version(void) { return 100; }

const char* bcg_last_error(void) { return g_err; }

// Single matrices: one CTA when the window fits in shared memory, else the
// whole-GPU dataflow kernel (which needs the caller's workspace).
static bool single_uses_multi(int n, int kd, int ldab) {
  bcg::CtaGeom g;
  return cta_block(n, kd, ldab, false, &g) == 0 || bcg::use_multi(n, kd);
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
  const int nb = cta_block((int)n, (int)kd, (int)ldab, false, &g);
  return launch_cta(ab, 0, nullptr, 0, 1, nb, g, info, false, st);
}

// Batched matrices whose window does not fit one CTA: one whole-GPU factorization
// after another, with a stream-ordered workspace.
static int batched_multi(int n, int kd, int ldab, double* ab, int64_t stride_ab, int batch, int32_t* info,
                         cudaStream_t st) {
  const size_t need = bcg::multi_workspace_bytes(n, kd);
  void* ws = nullptr;
  if (int r = cuda_status(cudaMallocAsync(&ws, need, st), "cudaMallocAsync(workspace)")) return r;
  int rc = 0;
  for (int i = 0; i < batch && rc == 0; ++i)
    rc = bcg::launch_multi(ab + (int64_t)i * stride_ab, n, kd, ldab, info + i, ws, sm_count(), st, g_err,
                           sizeof g_err);
  cudaFreeAsync(ws, st);
  return rc;
}

int bcg_dpbtrf_batched(int64_t n, int64_t kd, double* ab, int64_t ldab, int64_t stride_ab, int64_t batch,
                       int32_t* info, void* stream) {
  if (int r = check_geom(n, kd, ldab)) return r;
  if (!ab) return fail_arg(3, "ab is NULL");
  if (stride_ab < ldab * n) return fail_arg(5, "stride_ab < ldab*n");
  if (batch < 0 || batch > INT_MAX) return fail_arg(6, "batch out of range");
  if (!info) return fail_arg(7, "info is NULL");
  if (batch == 0) return 0;
  bcg::CtaGeom g;
  const int nb = cta_block((int)n, (int)kd, (int)ldab, false, &g);
  if (nb == 0) return batched_multi((int)n, (int)kd, (int)ldab, ab, stride_ab, (int)batch, info, (cudaStream_t)stream);
  return launch_cta(ab, stride_ab, nullptr, 0, (int)batch, nb, g, info, false, (cudaStream_t)stream);
}

static int launch_solve(const double* ab, int64_t sab, double* b, int64_t sb, int nrhs, int64_t blocks, int n,
                        int kd, int ldab, int32_t* info, cudaStream_t st, const int32_t* skip = nullptr);
static bool solve_streamed(int n, int kd, int ldab);

int bcg_dpbsv_batched(int64_t n, int64_t kd, double* ab, int64_t ldab, int64_t stride_ab, double* b,
                      int64_t stride_b, int64_t batch, int32_t* info, void* stream) {
  if (int r = check_geom(n, kd, ldab)) return r;
  if (!ab) return fail_arg(3, "ab is NULL");
  if (stride_ab < ldab * n) return fail_arg(5, "stride_ab < ldab*n");
  if (!b) return fail_arg(6, "b is NULL");
  if (stride_b < n) return fail_arg(7, "stride_b < n");
  if (batch < 0 || batch > INT_MAX) return fail_arg(8, "batch out of range");
  if (!info) return fail_arg(9, "info is NULL");
  if (batch == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  bcg::CtaGeom g;
  // kd >= 32: the pipelined factorization alone, then the streamed two-sweep solve (skipping
  // failed matrices) -- measured faster than fusing the forward sweep into the pivot's chain
  // (C5 1024: 3.51 + 2.30 ms vs 5.99 ms)
  if (kd >= 32 && cta_block((int)n, (int)kd, (int)ldab, false, &g) && solve_streamed((int)n, (int)kd, (int)ldab)) {
    if (int rc = bcg_dpbtrf_batched(n, kd, ab, ldab, stride_ab, batch, info, stream)) return rc;
    return launch_solve(ab, stride_ab, b, stride_b, 1, batch, (int)n, (int)kd, (int)ldab, info, st, info);
  }
  const int nb = cta_block((int)n, (int)kd, (int)ldab, true, &g);
  if (nb) return launch_cta(ab, stride_ab, b, stride_b, (int)batch, nb, g, info, true, st);
  // no fused variant for this geometry: factor, then solve (solve skips failed matrices)
  int rc = bcg_dpbtrf_batched(n, kd, ab, ldab, stride_ab, batch, info, stream);
  if (rc) return rc;
  bcg::pbtrs_after_factor_kernel<<<(unsigned)batch, bcg::kCtaThreads, 0, st>>>(ab, stride_ab, b, stride_b, (int)n,
                                                                             (int)kd, (int)ldab, info);
  return cuda_status(cudaGetLastError(), "pbtrs_after_factor_kernel launch");
}

// Streamed solve (shared-memory ring of 5-7 column blocks) when it fits, else the
// direct-from-L2 kernel.
static bcg::CtaGeom solve_geom(int n, int kd, int ldab) {
  bcg::CtaGeom g = make_geom(n, kd, ldab, 16, true);
  g.nx = ((kd + 48) + 1) & ~1;      // rows in flight: kd + NB, plus the entering block
  // block buffers for the streamed sweeps: 7 (deeper prefetch) when two CTAs still fit per
  // SM, else 5
  g.nslot = 7 * 16;
  if (bcg::cta_smem_bytes(16, g, true) > (size_t)(113 * 1024 - 512)) g.nslot = 5 * 16;
  return g;
}

static bool solve_streamed(int n, int kd, int ldab) {
  return bcg::cta_smem_bytes(16, solve_geom(n, kd, ldab), true) <= (size_t)smem_optin();
}

static int launch_solve(const double* ab, int64_t sab, double* b, int64_t sb, int nrhs, int64_t blocks, int n,
                        int kd, int ldab, int32_t* info, cudaStream_t st, const int32_t* skip) {
  const bcg::CtaGeom g = solve_geom(n, kd, ldab);
  const size_t smem = bcg::cta_smem_bytes(16, g, true);
  if (smem <= (size_t)smem_optin()) {
    auto k = bcg::pbtrs_cta_kernel;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(pbtrs_cta)");
    k<<<(unsigned)blocks, bcg::kCtaThreads, smem, st>>>(ab, sab, b, sb, nrhs, g, info, skip);
    return cuda_status(cudaGetLastError(), "pbtrs_cta_kernel launch");
  }
  bcg::pbtrs_kernel<<<(unsigned)blocks, bcg::kCtaThreads, 0, st>>>(ab, sab, b, sb, nrhs, n, kd, ldab, info);
  return cuda_status(cudaGetLastError(), "pbtrs_kernel launch");
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
  return launch_solve(ab, 0, b, ldb, (int)nrhs, nrhs, (int)n, (int)kd, (int)ldab, info, (cudaStream_t)stream);
}

int bcg_dpbtrs_batched(int64_t n, int64_t kd, const double* ab, int64_t ldab, int64_t stride_ab, double* b,
                       int64_t stride_b, int64_t batch, int32_t* info, void* stream) {
  if (int r = check_geom(n, kd, ldab)) return r;
  if (!ab) return fail_arg(3, "ab is NULL");
  if (stride_ab < ldab * n) return fail_arg(5, "stride_ab < ldab*n");
  if (!b) return fail_arg(6, "b is NULL");
  if (stride_b < n) return fail_arg(7, "stride_b < n");
  if (batch < 0 || batch > INT_MAX) return fail_arg(8, "batch out of range");
  if (!info) return fail_arg(9, "info is NULL");
  if (batch == 0) return 0;
  return launch_solve(ab, stride_ab, b, stride_b, 1, batch, (int)n, (int)kd, (int)ldab, info,
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
