// band_multi.cuh -- one band matrix factored by the whole GPU: a persistent dataflow kernel.
//
// The reference runs the blocked algorithm as a task DAG on CPU threads
// (pkg/src/bandchol/taskgraph.py:84-155, parallel.py:65-127).  Here the DAG
// becomes in-kernel dataflow over NB x NB tiles of the band (tile (R, C) covers
// rows R*NB.., columns C*NB..; T = ceil(kd/NB) sub-diagonal tiles per column):
//
//   * CTA 0 is the PIVOT.  Step j: POTRF of tile (j,j) fused with the inverse of
//     its factor (Linv, published for the workers' TRSMs), then the critical
//     near-diagonal work of the next step: tile (j+1,j) gets its last update
//     (with L(j+1,j-1), L(j,j-1)), its TRSM (a GEMM with Linv), and tile (j+1,j+1)
//     its last two updates -- so the chain POTRF(j) -> POTRF(j+1) never leaves
//     the SM.  The pivot owns updates (m+1,m+1,m), (m+2,m+1,m), (m+2,m+2,m).
//   * CTAs 1.. are WORKERS pulling tasks in a fixed topological order from an
//     atomic ticket: per step j the TRSMs L(R,j) = A(R,j) Linv(j)^T for
//     R = j+2..j+T, then the tile updates A(R,S) -= L(R,j) L(S,j)^T (R-major).
//     A task spins (ld.acquire.gpu + nanosleep) on per-tile flags:
//       lrdy[R][d]  L(R, R-d) final and published,
//       tcnt[R][d]  number of worker updates applied to tile (R, R-d),
//       irdy[j]     Linv(j) published.
//     Tickets are handed out in dependency order and every CTA is co-resident
//     (cooperative launch), so every wait is on work already owned by a running
//     CTA: no deadlock.  A failing pivot sets `fail`, which every spin polls.
//
// Tile GEMMs use the FP64 tensor path (mma.sync m8n8k4 f64 -> DMMA.8x8x4);
// tiles are staged in shared memory column-major with a padded leading
// dimension (LD = NB + 4 doubles: conflict-free fragment loads).  Band data
// that other CTAs wrote is read with ld.global.cg (L2), never through L1.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace bcg {

constexpr int kMultiThreads = 256;

struct MultiGeom {
  int n, kd, ldab;
  int nblk;  // ceil(n / NB)
  int T;     // ceil(kd / NB)
  int Q;     // worker tasks per step
};

// ---- workspace ---------------------------------------------------------------------
// [ctrl: 8 ints][tcnt: nblk*(T+1)][lrdy: nblk*(T+1)][irdy: nblk] ... (256-aligned) [linvT: nblk*NB*NB doubles]
struct MultiWs {
  int* ctrl;   // [0] ticket, [1] fail (global column + 1)
  int* tcnt;
  int* lrdy;
  int* irdy;
  double* linv;
};

__host__ __device__ inline size_t multi_flag_bytes(int nblk, int T) {
  size_t ints = 8 + 2 * (size_t)nblk * (T + 1) + (size_t)nblk;
  return (ints * sizeof(int) + 255) / 256 * 256;
}

__host__ __device__ inline MultiWs multi_ws(void* base, int nblk, int T) {
  MultiWs w;
  int* p = (int*)base;
  w.ctrl = p;
  w.tcnt = p + 8;
  w.lrdy = w.tcnt + (size_t)nblk * (T + 1);
  w.irdy = w.lrdy + (size_t)nblk * (T + 1);
  w.linv = (double*)((char*)base + multi_flag_bytes(nblk, T));
  return w;
}

// ---- sync primitives ---------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile(const int* p) { return *(volatile const int*)p; }

// thread 0: spin until *flag >= target; false if the kernel is aborting.
__device__ __forceinline__ bool spin_ge(const int* flag, int target, const int* fail) {
  if (ld_acquire(flag) >= target) return true;
  unsigned ns = 32;
  for (;;) {
    __nanosleep(ns);
    if (ld_acquire(flag) >= target) return true;
    if (ld_volatile(fail)) return false;
    if (ns < 256) ns <<= 1;
  }
}

// all threads: publish after this CTA's global stores
__device__ __forceinline__ void cta_publish(int* flag, int value) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(flag, value);
  }
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NB>
struct MultiTile {
  static constexpr int LD = NB + 4;  // LD = 4 (mod 16) doubles: conflict-free DMMA fragments
  static constexpr int ELEMS = NB * LD;
};

// ---- tile <-> band storage -----------------------------------------------------------
// smem tile layout: element (r, c) at s[c*LD + r].  Out-of-band / upper / past-n -> 0.
template <int NB>
__device__ __forceinline__ void load_tile(double* s, const double* ab, const MultiGeom& g, int R, int C) {
  constexpr int LD = MultiTile<NB>::LD;
  for (int idx = threadIdx.x; idx < NB * NB; idx += kMultiThreads) {
    const int c = idx / NB, r = idx - c * NB;
    const int i = R * NB + r, j = C * NB + c;
    const bool ok = (i < g.n) && (i >= j) && (i - j <= g.kd);
    s[c * LD + r] = ok ? __ldcg(ab + (int64_t)j * g.ldab + (i - j)) : 0.0;
  }
}

template <int NB>
__device__ __forceinline__ void store_tile(const double* s, double* ab, const MultiGeom& g, int R, int C) {
  constexpr int LD = MultiTile<NB>::LD;
  for (int idx = threadIdx.x; idx < NB * NB; idx += kMultiThreads) {
    const int c = idx / NB, r = idx - c * NB;
    const int i = R * NB + r, j = C * NB + c;
    if ((i < g.n) && (i >= j) && (i - j <= g.kd)) __stcg(ab + (int64_t)j * g.ldab + (i - j), s[c * LD + r]);
  }
}

// Linv^T stored densely: linvT[k*NB + n] = Linv(n, k); smem B layout s[k*LD + n] = Linv(n, k).
template <int NB>
__device__ __forceinline__ void load_linv(double* s, const double* linvT) {
  constexpr int LD = MultiTile<NB>::LD;
  for (int idx = threadIdx.x; idx < NB * NB; idx += kMultiThreads) {
    const int k = idx / NB, nn = idx - k * NB;
    s[k * LD + nn] = __ldcg(linvT + idx);
  }
}

template <int NB>
__device__ __forceinline__ void store_linv(const double* s, double* linvT) {
  constexpr int LD = MultiTile<NB>::LD;
  for (int idx = threadIdx.x; idx < NB * NB; idx += kMultiThreads) {
    const int k = idx / NB, nn = idx - k * NB;
    __stcg(linvT + idx, s[k * LD + nn]);
  }
}

// ---- tile GEMM on the FP64 tensor path -------------------------------------------------
// kSub: C -= A B^T   (C read from sC)      else: C = A B^T
// A(m,k) = sA[k*LD + m], B(n,k) = sB[k*LD + n], C(m,n) = sC[n*LD + m].  sC must not alias sA/sB.
template <int NB, bool kSub>
__device__ __forceinline__ void tile_gemm(double* sC, const double* sA, const double* sB) {
  constexpr int LD = MultiTile<NB>::LD;
  constexpr int MT = NB / 8;
  constexpr int WM = (NB == 64) ? 2 : 4;  // warps along m
  constexpr int WN = 8 / WM;
  constexpr int TM = MT / WM, TN = MT / WN;
  static_assert(TM >= 1 && TN >= 1, "tile too small for 8 warps");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp % WM, wn = warp / WM;
  const int gr = lane >> 2, gc = lane & 3;
  double acc[TM][TN][2];
#pragma unroll
  for (int tm = 0; tm < TM; ++tm)
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) {
      const int m = (wm * TM + tm) * 8 + gr, nn = (wn * TN + tn) * 8 + 2 * gc;
      acc[tm][tn][0] = kSub ? sC[nn * LD + m] : 0.0;
      acc[tm][tn][1] = kSub ? sC[(nn + 1) * LD + m] : 0.0;
    }
#pragma unroll 4
  for (int k0 = 0; k0 < NB; k0 += 4) {
    double a[TM], b[TN];
#pragma unroll
    for (int tm = 0; tm < TM; ++tm) {
      const double v = sA[(k0 + gc) * LD + (wm * TM + tm) * 8 + gr];
      a[tm] = kSub ? -v : v;
    }
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) b[tn] = sB[(k0 + gc) * LD + (wn * TN + tn) * 8 + gr];
#pragma unroll
    for (int tm = 0; tm < TM; ++tm)
#pragma unroll
      for (int tn = 0; tn < TN; ++tn) dmma_8x8x4(acc[tm][tn][0], acc[tm][tn][1], a[tm], b[tn]);
  }
  __syncthreads();  // sC may be read by other warps' fragment loads above (kSub) -- finish before writing
#pragma unroll
  for (int tm = 0; tm < TM; ++tm)
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) {
      const int m = (wm * TM + tm) * 8 + gr, nn = (wn * TN + tn) * 8 + 2 * gc;
      sC[nn * LD + m] = acc[tm][tn][0];
      sC[(nn + 1) * LD + m] = acc[tm][tn][1];
    }
  __syncthreads();
}

// ---- pivot: Cholesky of the diagonal tile fused with the inverse of its factor -------
// D(r,c) = sD[c*LD + r] (lower, zero upper) -> L; sX <- L^{-1} (X(i,q) = sX[q*LD + i]).
// Right-looking, one barrier per column: step c reads column c of D / row c of X
// unscaled and updates only later columns / rows; the scaling of column c is
// done lazily in the same step after the barrier, touching data no later step reads
// before the next barrier.  Returns the failing local column or -1.
template <int NB>
__device__ int potrf_inv_tile(double* sD, double* sX, int nvalid) {
  constexpr int LD = MultiTile<NB>::LD;
  constexpr int G = kMultiThreads / NB;  // thread groups per row
  const int r = threadIdx.x % NB, grp = threadIdx.x / NB;
  for (int idx = threadIdx.x; idx < NB * NB; idx += kMultiThreads) {
    const int q = idx / NB, i = idx - q * NB;
    sX[q * LD + i] = (i == q) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int c = 0; c < nvalid; ++c) {
    const double p = sD[c * LD + c];
    if (!(p > 0.0)) return c;  // uniform: every thread read the same value
    const double pinv = 1.0 / p;
    const double rs = rsqrt(p);
    if (r > c) {
      const double ur = sD[c * LD + r] * pinv;
      for (int c2 = c + 1 + grp; c2 <= r; c2 += G) sD[c2 * LD + r] = fma(-ur, sD[c * LD + c2], sD[c2 * LD + r]);
      for (int q = grp; q <= c; q += G) sX[q * LD + r] = fma(-ur, sX[q * LD + c], sX[q * LD + r]);
    }
    __syncthreads();
    // lazy scaling of column c of D and row c of X (read again only after the next barrier)
    if (grp == 0 && r >= c) sD[c * LD + r] = (r == c) ? p * rs : sD[c * LD + r] * rs;
    if (grp == 1 % G && r <= c) sX[r * LD + c] *= rs;
  }
  __syncthreads();
  return -1;
}

// ---- the kernel ------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(kMultiThreads, 1)
band_multi_kernel(double* __restrict__ ab, MultiGeom g, MultiWs ws, int32_t* info) {
  extern __shared__ __align__(16) double smem[];
  constexpr int E = MultiTile<NB>::ELEMS;
  __shared__ int s_task;
  __shared__ int s_ok;
  const int T = g.T, nblk = g.nblk;
  auto TC = [&](int R, int d) -> int* { return ws.tcnt + (size_t)R * (T + 1) + d; };
  auto LR = [&](int R, int d) -> int* { return ws.lrdy + (size_t)R * (T + 1) + d; };

  if (blockIdx.x == 0) {
    // ------------------------------ pivot ---------------------------------------
    double* buf[6];
#pragma unroll
    for (int b = 0; b < 6; ++b) buf[b] = smem + b * E;
    double* sD = buf[0];   // current diagonal tile (fully updated)
    double* sX = buf[1];   // Linv of the current diagonal
    double* sLp = buf[2];  // L(j, j-1) from the previous step
    double* f0 = buf[3];
    double* f1 = buf[4];
    double* f2 = buf[5];
    unsigned long long* tr = g_trace;
    load_tile<NB>(sD, ab, g, 0, 0);
    __syncthreads();
    int fail_col = -1;
    for (int j = 0; j < nblk; ++j) {
      const int nvalid = min(NB, g.n - j * NB);
      if (threadIdx.x == 0) trace_stamp_to(tr, j, 0);
      const int f = potrf_inv_tile<NB>(sD, sX, nvalid);
      if (threadIdx.x == 0) trace_stamp_to(tr, j, 1);
      if (f >= 0) {
        fail_col = j * NB + f;
        if (threadIdx.x == 0) atomicExch(ws.ctrl + 1, fail_col + 1);
        break;
      }
      store_tile<NB>(sD, ab, g, j, j);
      store_linv<NB>(sX, ws.linv + (size_t)j * NB * NB);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        st_release(LR(j, 0), 1);
        st_release(ws.irdy + j, 1);
      }
      if (threadIdx.x == 0) trace_stamp_to(tr, j, 2);
      if (j + 1 >= nblk) break;
      // --- critical near-diagonal work for step j+1 ---
      double* sW = f0;   // L(j+1, j-1), then L(j+1, j)
      double* sP = f1;   // A(j+1, j)
      double* sD2 = f2;  // A(j+1, j+1)
      const int lo = max(0, j + 1 - T);
      const int need = max(0, j - 1 - lo);  // worker updates m in [lo, j-2]
      const bool has_w = (j >= 1) && (T >= 2);
      if (threadIdx.x == 0) {
        bool ok = spin_ge(TC(j + 1, 1), need, ws.ctrl + 1) && spin_ge(TC(j + 1, 0), need, ws.ctrl + 1);
        if (ok && has_w) ok = spin_ge(LR(j + 1, 2), 1, ws.ctrl + 1);
        s_ok = ok;
      }
      __syncthreads();
      if (!s_ok) break;
      if (threadIdx.x == 0) trace_stamp_to(tr, j, 3);
      load_tile<NB>(sP, ab, g, j + 1, j);
      load_tile<NB>(sD2, ab, g, j + 1, j + 1);
      if (has_w) load_tile<NB>(sW, ab, g, j + 1, j - 1);
      __syncthreads();
      if (threadIdx.x == 0) trace_stamp_to(tr, j, 4);
      if (has_w) {
        tile_gemm<NB, true>(sP, sW, sLp);   // A(j+1,j)   -= L(j+1,j-1) L(j,j-1)^T
        tile_gemm<NB, true>(sD2, sW, sW);   // A(j+1,j+1) -= L(j+1,j-1) L(j+1,j-1)^T
      }
      tile_gemm<NB, false>(sW, sP, sX);     // L(j+1,j) = A(j+1,j) Linv(j)^T
      tile_gemm<NB, true>(sD2, sW, sW);     // A(j+1,j+1) -= L(j+1,j) L(j+1,j)^T
      if (threadIdx.x == 0) trace_stamp_to(tr, j, 5);
      store_tile<NB>(sW, ab, g, j + 1, j);
      cta_publish(LR(j + 1, 1), 1);
      if (threadIdx.x == 0) trace_stamp_to(tr, j, 6);
      // rotate: D <- D2, Lp <- W; free = old D, old Lp, P
      double* oldD = sD;
      double* oldLp = sLp;
      sD = sD2;
      sLp = sW;
      f0 = oldD;
      f1 = oldLp;
      f2 = sP;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const int fl = ld_volatile(ws.ctrl + 1);
      info[0] = fail_col >= 0 ? fail_col + 1 : (fl ? fl : 0);
    }
    return;
  }

  // -------------------------------- workers -------------------------------------------
  double* sA = smem;
  double* sB = smem + E;
  double* sC = smem + 2 * E;
  const int Q = g.Q;
  const long long total = (long long)nblk * Q;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(ws.ctrl, 1);
    __syncthreads();
    const long long t = s_task;
    if (t >= total) break;
    const int j = (int)(t / Q), q = (int)(t - (long long)j * Q);
    if (q < T - 1) {
      // TRSM: L(R, j) = A(R, j) Linv(j)^T
      const int R = j + 2 + q;
      if (R >= nblk) { __syncthreads(); continue; }
      if (threadIdx.x == 0)
        s_ok = spin_ge(ws.irdy + j, 1, ws.ctrl + 1) && spin_ge(TC(R, R - j), j - max(0, R - T), ws.ctrl + 1);
      __syncthreads();
      if (!s_ok) break;
      load_tile<NB>(sA, ab, g, R, j);
      load_linv<NB>(sB, ws.linv + (size_t)j * NB * NB);
      __syncthreads();
      tile_gemm<NB, false>(sC, sA, sB);
      store_tile<NB>(sC, ab, g, R, j);
      cta_publish(LR(R, R - j), 1);
    } else {
      const int u = q - (T - 1);
      int a = (int)((sqrtf(8.0f * (float)u + 1.0f) - 1.0f) * 0.5f);
      while (a * (a + 1) / 2 > u) --a;
      while ((a + 1) * (a + 2) / 2 <= u) ++a;
      const int b = u - a * (a + 1) / 2;
      const int R = j + 1 + a, S = R - b;
      const bool pivot_owned = (R == j + 1) || (R == j + 2 && S >= j + 1);
      if (R >= nblk || pivot_owned) { __syncthreads(); continue; }
      const int done = j - max(0, R - T);
      if (threadIdx.x == 0)
        s_ok = spin_ge(LR(R, R - j), 1, ws.ctrl + 1) && spin_ge(LR(S, S - j), 1, ws.ctrl + 1) &&
               spin_ge(TC(R, R - S), done, ws.ctrl + 1);
      __syncthreads();
      if (!s_ok) break;
      load_tile<NB>(sA, ab, g, R, j);
      load_tile<NB>(sB, ab, g, S, j);
      load_tile<NB>(sC, ab, g, R, S);
      __syncthreads();
      tile_gemm<NB, true>(sC, sA, sB);
      store_tile<NB>(sC, ab, g, R, S);
      cta_publish(TC(R, R - S), done + 1);
    }
  }
}

// ---- host side -------------------------------------------------------------------------
inline int multi_nb(int kd) { return kd >= 1000 ? 64 : 32; }

inline bool use_multi(int n, int kd) { (void)n; return kd >= 160; }

inline MultiGeom multi_geom(int n, int kd, int ldab) {
  MultiGeom g;
  const int nb = multi_nb(kd);
  g.n = n;
  g.kd = kd;
  g.ldab = ldab;
  g.nblk = (n + nb - 1) / nb;
  g.T = (kd + nb - 1) / nb;
  g.Q = (g.T - 1) + g.T * (g.T + 1) / 2;
  return g;
}

inline size_t multi_workspace_bytes(int n, int kd) {
  MultiGeom g = multi_geom(n, kd, kd + 1);
  const int nb = multi_nb(kd);
  return multi_flag_bytes(g.nblk, g.T) + (size_t)g.nblk * nb * nb * sizeof(double);
}

template <int NB>
inline int launch_multi_t(double* ab, const MultiGeom& g, int32_t* info, void* workspace, int sms, cudaStream_t st,
                          char* err, size_t errlen) {
  const size_t smem = 6 * (size_t)MultiTile<NB>::ELEMS * sizeof(double);
  auto k = band_multi_kernel<NB>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    snprintf(err, errlen, "cudaFuncSetAttribute(band_multi): %s", cudaGetErrorString(e));
    return (int)e;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kMultiThreads, smem);
  if (per_sm < 1) {
    snprintf(err, errlen, "band_multi kernel does not fit on an SM");
    return (int)cudaErrorInvalidConfiguration;
  }
  e = cudaMemsetAsync(workspace, 0, multi_flag_bytes(g.nblk, g.T), st);
  if (e != cudaSuccess) {
    snprintf(err, errlen, "cudaMemsetAsync(workspace): %s", cudaGetErrorString(e));
    return (int)e;
  }
  MultiWs ws = multi_ws(workspace, g.nblk, g.T);
  if (per_sm > 2) per_sm = 2;
  int grid = sms * per_sm;
  MultiGeom gg = g;
  void* args[] = {(void*)&ab, (void*)&gg, (void*)&ws, (void*)&info};
  e = cudaLaunchCooperativeKernel((void*)k, dim3(grid), dim3(kMultiThreads), args, smem, st);
  if (e != cudaSuccess) {
    snprintf(err, errlen, "cudaLaunchCooperativeKernel(band_multi): %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

inline int launch_multi(double* ab, int n, int kd, int ldab, int32_t* info, void* workspace, int sms,
                        cudaStream_t st, char* err, size_t errlen) {
  MultiGeom g = multi_geom(n, kd, ldab);
  if (multi_nb(kd) == 64) return launch_multi_t<64>(ab, g, info, workspace, sms, st, err, errlen);
  return launch_multi_t<32>(ab, g, info, workspace, sms, st, err, errlen);
}

}  // namespace bcg
