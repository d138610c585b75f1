// band_multi.cuh -- one band matrix factored by the whole GPU: a persistent dataflow kernel.
//
// The reference runs the blocked algorithm as a task DAG on CPU threads
// (pkg/src/bandchol/taskgraph.py:84-155, parallel.py:65-127).  Here the DAG
// becomes in-kernel dataflow over NB x NB tiles of the band (tile (R, C) covers
// rows R*NB.., columns C*NB..; T = ceil(kd/NB) sub-diagonal tiles per column):
//
//   * CTA 0 is the PIVOT: the whole near-diagonal chain stays in its shared memory.  Step j,
//     stage A: warp 0 factors tile (j,j) (warp-level redundant-chain POTRF), warp 1 forms
//     L(j,j)^-1 in lock step, the others fetch A(j+1,j), A(j+1,j+1) and L(j+1,j-2) and apply
//     the lookback products (with L(j+1,j-1), the pivot's own TRSM of the step before, and
//     L(j,j-1), L(j,j-2)); stage B: L(j+1,j) and L(j+2,j) as products with L(j,j)^-1, SYRK of
//     (j+1,j+1), and straight into the next POTRF; write-backs and flag releases run behind,
//     asynchronously.  One CTA barrier per step.  The pivot owns the TRSMs of rows j+1, j+2
//     and the updates (m+1,m+1,m), (m+2,m+1,m), (m+2,m+2,m), (m+3,m+2,m).
//   * CTAs 1.. are WORKERS pulling tasks in a fixed topological order from an atomic
//     ticket.  Per super-step s: (A) step s-1's updates of tile column s+1, (B) the ROW OWNER
//     of the row entering the band -- one group runs the row's whole chain TRSM L(R,m) ->
//     update of (R,m+1) -> TRSM L(R,m+1) ... for m = R-T .. R-3, the tile staying in shared
//     memory between links -- (C) step s-1's other tile updates A(R,S) -= L(R,m) L(S,m)^T.
//     A task spins (ld.acquire.gpu + nanosleep) on per-tile flags:
//       lrdy[R][d]  L(R, R-d) final and published,
//       tcnt[R][d]  number of worker updates applied to tile (R, R-d).
//     Tickets are handed out in dependency order and every CTA is co-resident
//     (cooperative launch), so every wait is on work already owned by a running
//     CTA: no deadlock (a row owner holds its group for up to T steps, so row owners are
//     used only when the grid has >= 2T+16 groups).  A failing pivot sets `fail`, which
//     every spin polls.
//
// Tile GEMMs use the FP64 tensor path (mma.sync m8n8k4 f64 -> DMMA.8x8x4);
// tiles are staged in shared memory column-major with a padded leading
// dimension (LD = NB + 4 doubles: conflict-free fragment loads).  Band data
// that other CTAs wrote is read with ld.global.cg (L2), never through L1, and
// every thread issues all of its tile loads before the first shared store, so a
// tile costs one L2 round trip.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "band_cta.cuh"

namespace bcg {

constexpr int kMultiThreads = 256;
#ifndef BCG_WIDE_GROUPS
#define BCG_WIDE_GROUPS 4  // worker groups per CTA for wide bands (kd >= 1000)
#define BCG_WIDE_PERSM 2
#endif
#ifndef BCG_WORKER_SPIN_NS
#define BCG_WORKER_SPIN_NS 64
#endif
constexpr unsigned kWorkerSpinNs = BCG_WORKER_SPIN_NS;  // longest back-off of a worker's flag spin
#ifndef BCG_MULTI_PREFETCH
#define BCG_MULTI_PREFETCH true  // fetch a worker's next ticket while its current update task runs
#endif

struct MultiGeom {
  int n, kd, ldab;
  int nblk;  // ceil(n / NB)
  int T;     // ceil(kd / NB)
  int Q;     // worker tasks per step
  int owner; // row-owner scheduling of the row tasks (needs spare worker groups: host decides)
};

// ---- workspace ---------------------------------------------------------------------
// [ctrl: 8 ints][tcnt: nblk*(T+1)][lrdy: nblk*(T+1)] (zeroed per launch) [inv: nblk*NB*NB doubles]
struct MultiWs {
  int* ctrl;  // [0] ticket, [1] fail (global column + 1), [2] pivot's SM id + 1
  int* tcnt;
  int* lrdy;
  double* inv;  // inv[j][k*NB + c] = (L(j,j)^-1)(c, k): the row tasks' TRSM is a product with it
};

__host__ __device__ inline size_t multi_flag_bytes(int nblk, int T) {
  size_t ints = 8 + 2 * (size_t)nblk * (T + 1);
  return (ints * sizeof(int) + 255) / 256 * 256;
}

__host__ __device__ inline MultiWs multi_ws(void* base, int nblk, int T) {
  MultiWs w;
  int* p = (int*)base;
  w.ctrl = p;
  w.tcnt = p + 8;
  w.lrdy = w.tcnt + (size_t)nblk * (T + 1);
  w.inv = (double*)((char*)base + multi_flag_bytes(nblk, T));
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

// one thread: spin until *flag >= target; false if the kernel is aborting.
__device__ __forceinline__ bool spin_ge(const int* flag, int target, const int* fail, unsigned max_ns) {
  if (ld_acquire(flag) >= target) return true;
  unsigned ns = 16;
  for (;;) {
    __nanosleep(ns);
    if (ld_acquire(flag) >= target) return true;
    if (ld_volatile(fail)) return false;
    if (ns < max_ns) ns <<= 1;
  }
}

// all threads: publish after this CTA's global stores.  The barrier orders every
// thread's stores before thread 0's release, and a release is cumulative over what its
// thread has synchronised with, so no separate fence is needed (the consumer pairs it
// with ld.acquire + a barrier).
__device__ __forceinline__ void cta_publish(int* flag, int value) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(flag, value);
}

__device__ __forceinline__ void named_sync(int id, int cnt) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}

// cross-SM event stamps (trace build): %globaltimer ns into trace row nblk + step
__device__ __forceinline__ void xstamp(int nblk, int step, int ph) {
#ifdef BCG_TRACE
  if (g_trace && step >= 0 && step < nblk) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long idx = 1 + (unsigned long long)(nblk + step) * kTracePhases + ph;
    if (idx < g_trace_cap - 8) g_trace[idx] = t;
  }
#endif
}

template <int NB>
struct MultiTile {
  static constexpr int LD = NB + 4;  // LD = 4 (mod 16) doubles: conflict-free DMMA fragments
  static constexpr int ELEMS = NB * LD;
};

// ---- tile <-> band storage -----------------------------------------------------------
// smem tile layout: element (r, c) at s[c*LD + r].  Out-of-band / upper / past-n -> 0.
// Threads t in [0, NT) take part; every thread issues its loads before its stores.
// Tiles wholly inside the band (1 <= R - C, (R - C) NB + NB - 1 <= kd, all rows < n) take a
// path without per-element index arithmetic or masks: thread t keeps row t % NB and walks
// the columns with a constant pointer stride (the instruction stream of the generic path --
// ~15 instructions per element -- was most of a worker task's time).
__device__ __forceinline__ bool tile_interior(const MultiGeom& g, int NB, int R, int C) {
  const int d = R - C;
  return d >= 1 && d * NB + NB - 1 <= g.kd && R * NB + NB <= g.n;
}
// A diagonal tile may be LOADED without masks as well: its entries above the diagonal then
// come from the preceding columns' storage (in bounds for R >= 1), and every consumer treats
// the upper triangle as don't-care (POTRF, the SYRK-type products; write-backs are masked).
__device__ __forceinline__ bool tile_loadable_unmasked(const MultiGeom& g, int NB, int R, int C) {
  return tile_interior(g, NB, R, C) || (R == C && R >= 1 && NB - 1 <= g.kd && R * NB + NB <= g.n);
}

template <int NB, int NT>
__device__ __forceinline__ void load_tile(double* s, const double* ab, const MultiGeom& g, int R, int C, int t) {
  constexpr int LD = MultiTile<NB>::LD;
  constexpr int E = (NB * NB + NT - 1) / NT;
  double v[E];
  if (NT % NB == 0 && tile_interior(g, NB, R, C)) {
    constexpr int CS = NT / NB;  // columns per sweep of the threads
    const int r = t % NB, c0 = t / NB;
    const double* p = ab + (int64_t)(C * NB + c0) * g.ldab + ((R - C) * NB + r - c0);
    const int64_t step = (int64_t)CS * (g.ldab - 1);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = __ldcg(p + e * step);
    double* q = s + c0 * LD + r;
#pragma unroll
    for (int e = 0; e < E; ++e) q[e * CS * LD] = v[e];
    return;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int idx = t + e * NT;
    const int c = idx / NB, r = idx - c * NB;
    const int i = R * NB + r, j = C * NB + c;
    const bool ok = (idx < NB * NB) && (i < g.n) && (i >= j) && (i - j <= g.kd);
    v[e] = ok ? __ldcg(ab + (int64_t)j * g.ldab + (i - j)) : 0.0;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int idx = t + e * NT;
    const int c = idx / NB, r = idx - c * NB;
    if (idx < NB * NB) s[c * LD + r] = v[e];
  }
}

// one tile whose upper triangle is don't-care: unmasked whenever the addresses are in bounds
template <int NB, int NT>
__device__ __forceinline__ void load_tile_unmasked_ok(double* s, const double* ab, const MultiGeom& g, int R, int C,
                                                      int t) {
  constexpr int LD = MultiTile<NB>::LD;
  if (tile_loadable_unmasked(g, NB, R, C)) {
    constexpr int CS = NT / NB, E = NB * NB / NT;
    const int r = t % NB, c0 = t / NB;
    const double* p = ab + (int64_t)(C * NB + c0) * g.ldab + ((R - C) * NB + r - c0);
    const int64_t step = (int64_t)CS * (g.ldab - 1);
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = __ldcg(p + e * step);
    double* q = s + c0 * LD + r;
#pragma unroll
    for (int e = 0; e < E; ++e) q[e * CS * LD] = v[e];
  } else {
    load_tile<NB, NT>(s, ab, g, R, C, t);
  }
}

// tiles (R, C0) -> s0, (R, C1) -> s1 and, with K3, (R, C2) -> s2 in ONE L2 round trip
template <int NB, int NT, bool K3>
__device__ __forceinline__ void load_tiles3(double* s0, double* s1, double* s2, const double* ab, const MultiGeom& g,
                                            int R, int C0, int C1, int C2, int t) {
  constexpr int LD = MultiTile<NB>::LD;
  constexpr int E = NB * NB / NT;
  static_assert(NB * NB % NT == 0 && NT % NB == 0, "whole columns per sweep");
  constexpr int K = K3 ? 3 : 2;
  constexpr int CS = NT / NB;
  const int r = t % NB, c0 = t / NB;
  double v[K][E];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int C = k == 0 ? C0 : (k == 1 ? C1 : C2);
    if (tile_loadable_unmasked(g, NB, R, C)) {
      const double* p = ab + (int64_t)(C * NB + c0) * g.ldab + ((R - C) * NB + r - c0);
      const int64_t step = (int64_t)CS * (g.ldab - 1);
#pragma unroll
      for (int e = 0; e < E; ++e) v[k][e] = __ldcg(p + e * step);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int c = c0 + e * CS;
        const int i = R * NB + r, j = C * NB + c;
        const bool ok = (i < g.n) && (i >= j) && (i - j <= g.kd);
        v[k][e] = ok ? __ldcg(ab + (int64_t)j * g.ldab + (i - j)) : 0.0;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double* q = (k == 0 ? s0 : (k == 1 ? s1 : s2)) + c0 * LD + r;
#pragma unroll
    for (int e = 0; e < E; ++e) q[e * CS * LD] = v[k][e];
  }
}

template <int NB, int NT = kMultiThreads>
__device__ __forceinline__ void store_tile(const double* s, double* ab, const MultiGeom& g, int R, int C,
                                           int t = threadIdx.x) {
  constexpr int LD = MultiTile<NB>::LD;
  if (NT % NB == 0 && tile_interior(g, NB, R, C)) {
    constexpr int CS = NT / NB, E = NB * NB / NT;
    const int r = t % NB, c0 = t / NB;
    double* p = ab + (int64_t)(C * NB + c0) * g.ldab + ((R - C) * NB + r - c0);
    const int64_t step = (int64_t)CS * (g.ldab - 1);
    const double* q = s + c0 * LD + r;
#pragma unroll
    for (int e = 0; e < E; ++e) __stcg(p + e * step, q[e * CS * LD]);
    return;
  }
  for (int idx = t; idx < NB * NB; idx += NT) {
    const int c = idx / NB, r = idx - c * NB;
    const int i = R * NB + r, j = C * NB + c;
    if ((i < g.n) && (i >= j) && (i - j <= g.kd)) __stcg(ab + (int64_t)j * g.ldab + (i - j), s[c * LD + r]);
  }
}

// ---- tile GEMM on the FP64 tensor path -------------------------------------------------
// kSub: C -= A B^T (C read from sC)      else: C = A B^T.  NW warps (warp index wg within
// the group, synchronised by named barrier bar_id over bar_cnt threads), M = N = K = NB.
// A(m,k) = sA[k*LD + m], B(n,k) = sB[k*LD + n], C(m,n) = sC[n*LD + m].  sC must not alias sA/sB.
// kBTri: B(n,k) = 0 for k > n (the transposed inverse of a lower-triangular block): k-steps
// past an 8-column block's last column are skipped.
__device__ __forceinline__ void dmma884p(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
template <int NB, bool kSub, int NW = 8, bool kBTri = false>
__device__ __forceinline__ void tile_gemm(double* sC, const double* sA, const double* sB, int wg = threadIdx.x >> 5,
                                          int bar_id = 0, int bar_cnt = kMultiThreads, const double* sA2 = nullptr,
                                          const double* sB2 = nullptr) {
  constexpr int LD = MultiTile<NB>::LD;
  constexpr int MT = NB / 8;
  constexpr int WM = (NB == 64) ? 2 : (NW < 4 ? NW : 4);  // warps along m
  constexpr int WN = NW / WM;
  constexpr int TM = MT / WM, TN = MT / WN;
  static_assert(TM >= 1 && TN >= 1, "tile too small for the warps");
  const int warp = wg, lane = threadIdx.x & 31;
  const int wm = warp % WM, wn = warp / WM;
  const int gr = lane >> 2, gc = lane & 3;
  double acc[TM][TN][2];
  // B columns / C column pairs in the kperm order (band_cta.cuh): with LD = 4 (mod 16) doubles
  // the C fragment loads and stores of a half-warp then hit 16 distinct bank pairs (the
  // identity order is 2-way conflicted: 25 % of the kernel's shared-memory wavefronts on C4)
  const int pb = kperm(gr), pc0 = kperm(2 * gc), pc1 = kperm(2 * gc + 1);
#pragma unroll
  for (int tm = 0; tm < TM; ++tm)
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) {
      const int m = (wm * TM + tm) * 8 + gr, n0 = (wn * TN + tn) * 8;
      acc[tm][tn][0] = kSub ? sC[(n0 + pc0) * LD + m] : 0.0;
      acc[tm][tn][1] = kSub ? sC[(n0 + pc1) * LD + m] : 0.0;
    }
#pragma unroll
  for (int k0 = 0; k0 < NB; k0 += 4) {
    double a[TM], b[TN];
#pragma unroll
    for (int tm = 0; tm < TM; ++tm) {
      const double v = sA[(k0 + gc) * LD + (wm * TM + tm) * 8 + gr];
      a[tm] = kSub ? -v : v;
    }
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) b[tn] = sB[(k0 + gc) * LD + (wn * TN + tn) * 8 + pb];
#pragma unroll
    for (int tm = 0; tm < TM; ++tm)
#pragma unroll
      for (int tn = 0; tn < TN; ++tn) {
        if (kBTri && WN == 1 && k0 > tn * 8 + 7) continue;  // (WN == 1: the block index is static)
        dmma884p(acc[tm][tn][0], acc[tm][tn][1], a[tm], b[tn]);
      }
  }
  // optional second product into the same accumulators (C -= A B^T + A2 B2^T: one pass over C)
  if (sA2) {
#pragma unroll
    for (int k0 = 0; k0 < NB; k0 += 4) {
      double a[TM], b[TN];
#pragma unroll
      for (int tm = 0; tm < TM; ++tm) {
        const double v = sA2[(k0 + gc) * LD + (wm * TM + tm) * 8 + gr];
        a[tm] = kSub ? -v : v;
      }
#pragma unroll
      for (int tn = 0; tn < TN; ++tn) b[tn] = sB2[(k0 + gc) * LD + (wn * TN + tn) * 8 + pb];
#pragma unroll
      for (int tm = 0; tm < TM; ++tm)
#pragma unroll
        for (int tn = 0; tn < TN; ++tn) dmma884p(acc[tm][tn][0], acc[tm][tn][1], a[tm], b[tn]);
    }
  }
  named_sync(bar_id, bar_cnt);  // sC may be read by other warps' fragment loads above (kSub)
#pragma unroll
  for (int tm = 0; tm < TM; ++tm)
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) {
      const int m = (wm * TM + tm) * 8 + gr, n0 = (wn * TN + tn) * 8;
      sC[(n0 + pc0) * LD + m] = acc[tm][tn][0];
      sC[(n0 + pc1) * LD + m] = acc[tm][tn][1];
    }
  named_sync(bar_id, bar_cnt);
}

// C -= A A^T on the LOWER 8x8 blocks of a 32x32 tile only (10 of 16: the upper triangle of a
// diagonal tile is don't-care everywhere), four warps, blocks dealt 3/3/2/2.  Same fragment
// conventions and kperm column order as tile_gemm.
template <int NB>
__device__ __forceinline__ void tile_syrk_lower4(double* sC, const double* sA, int w4, int bar_id, int bar_cnt) {
  static_assert(NB == 32, "block lists below are for a 4x4 grid of 8x8 blocks");
  constexpr int LD = MultiTile<NB>::LD;
  // (tm, tn) per warp, packed 4 bits each; count in cnt
  const unsigned tmv = w4 == 0 ? 0x033u : w4 == 1 ? 0x133u : w4 == 2 ? 0x22u : 0x12u;
  const unsigned tnv = w4 == 0 ? 0x010u : w4 == 1 ? 0x032u : w4 == 2 ? 0x10u : 0x12u;
  const int cnt = w4 < 2 ? 3 : 2;
  const int lane = threadIdx.x & 31, gr = lane >> 2, gc = lane & 3;
  const int pb = kperm(gr), pc0 = kperm(2 * gc), pc1 = kperm(2 * gc + 1);
  double acc[3][2];
  int mo[3], no[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    mo[b] = 8 * (int)((tmv >> (4 * b)) & 15u);
    no[b] = 8 * (int)((tnv >> (4 * b)) & 15u);
    acc[b][0] = b < cnt ? sC[(no[b] + pc0) * LD + mo[b] + gr] : 0.0;
    acc[b][1] = b < cnt ? sC[(no[b] + pc1) * LD + mo[b] + gr] : 0.0;
  }
#pragma unroll
  for (int k0 = 0; k0 < NB; k0 += 4) {
    const double* col = sA + (k0 + gc) * LD;
#pragma unroll
    for (int b = 0; b < 3; ++b)
      if (b < cnt) dmma884p(acc[b][0], acc[b][1], -col[mo[b] + gr], col[no[b] + pb]);
  }
  named_sync(bar_id, bar_cnt);
#pragma unroll
  for (int b = 0; b < 3; ++b)
    if (b < cnt) {
      sC[(no[b] + pc0) * LD + mo[b] + gr] = acc[b][0];
      sC[(no[b] + pc1) * LD + mo[b] + gr] = acc[b][1];
    }
  named_sync(bar_id, bar_cnt);
}

// ---- warp-level Cholesky of a 32x32 block in a smem tile (the pivot chain) ------------
// s(r, c) = s[c*ld + r], lower part valid; ld*8 bytes must keep columns 16-byte aligned.
// Same scheme as CtaBand::potrf_diag: every lane computes the pivot sequence (branch-free
// Newton rsqrt, the next column's operands broadcast a column early), lane r owns row r.
// Column c of L is written straight into its tile column, which then serves as the
// broadcast buffer of the rank-1 update (one __syncwarp per column); entries above the
// diagonal become don't-care.  Rows past nvalid are identity rows.  Failure: after a bad
// pivot every later pivot is NaN, so the failing column is the first lane whose L(r, r)
// is not > 0.  Returns it or -1 (uniform).
//
// For the inverse warp (warp_inverse32) trailing this one column group by column group:
// sdinv[c] = 1 / L(c, c), and colbar[c / 4] (one mbarrier per four columns, one arrival,
// one phase per call) is completed once columns 4(c/4)..4(c/4)+3 and their sdinv are written.
__device__ __forceinline__ int warp_potrf32(double* s, int ld, int nvalid, double* sdinv,
                                            unsigned long long* colbar) {
  const int r = threadIdx.x & 31;
  double row[32];
  if (nvalid == 32) {
#pragma unroll
    for (int c = 0; c < 32; ++c) row[c] = s[c * ld + r];
  } else {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const double v = s[c * ld + r];
      row[c] = (r < nvalid) ? v : ((c == r) ? 1.0 : 0.0);
    }
  }
  double p = __shfl_sync(kFull, row[0], 0);
  double alpha = __shfl_sync(kFull, row[0], 1);
  double beta = __shfl_sync(kFull, row[1], 1);
  double rs = rsqrt_nr(p);
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const double lrc = row[c] * rs;  // L(r, c) for r >= c (lane c: p * rs bit for bit)
    const double l1 = alpha * rs;
    const double pn = fma(-l1, l1, beta);
    const double rsn = rsqrt_nr(pn);
    if (c + 1 < 32) row[c + 1 < 32 ? c + 1 : 0] = fma(-lrc, l1, row[c + 1 < 32 ? c + 1 : 0]);
    double alpha_n = 0.0, beta_n = 0.0;
    if (c + 2 < 32) {
      const double bn = fma(-lrc, lrc, row[c + 2 < 32 ? c + 2 : 0]);
      alpha_n = shfl_early(row[c + 1 < 32 ? c + 1 : 0], c + 2);
      beta_n = shfl_early(bn, c + 2);
    }
    row[c] = lrc;
    double* sc = s + c * ld;
    sc[r] = lrc;
    if (r == 0) sdinv[c] = rs;
    __syncwarp();
    if ((c & 3) == 3 && r == 0) mbar_arrive(colbar + (c >> 2));  // (release: cumulative over the warp barrier)
#pragma unroll
    for (int h = 0; h < 16; ++h) {
      if (2 * h + 1 >= c + 2) {
        const double2 l2 = reinterpret_cast<const double2*>(sc)[h];
        if (2 * h >= c + 2) row[2 * h] = fma(-lrc, l2.x, row[2 * h]);
        row[2 * h + 1] = fma(-lrc, l2.y, row[2 * h + 1]);
      }
    }
    p = pn;
    rs = rsn;
    alpha = alpha_n;
    beta = beta_n;
  }
  const double dgl = (r < nvalid) ? s[r * ld + r] : 1.0;
  const unsigned bad = __ballot_sync(kFull, !(dgl > 0.0));
  __syncwarp();
  return bad ? __ffs(bad) - 1 : -1;
}

// ---- L^-1 of the 32x32 block, one warp, in lock step behind warp_potrf32 ------------------
// Lane k applies the POTRF's column operations to e_k: y[c] = (y[c] - sum_{c'<c} y[c'] L(c,c')) / L(c,c),
// i.e. y = e_k^T L^-T, so y[c] = (L^-1)(c, k).  Stored as sInv[k*LD + c]: the B operand of
// X = A L^-T = A (L^-1)^T in tile_gemm's convention (B(n, k) = sB[k*LD + n]).  Column c of L
// and sdinv[c] are read from the tile the POTRF warp is writing, four columns behind it.
__device__ __forceinline__ void warp_inverse32(const double* s, int ld, const double* sdinv, double* sInv,
                                               unsigned long long* colbar, unsigned parity) {
  const int k = threadIdx.x & 31;
  double v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = (c == k) ? 1.0 : 0.0;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if ((c & 3) == 0) mbar_wait(colbar + (c >> 2), parity);
    const double y = v[c] * sdinv[c];
    sInv[k * ld + c] = y;
    const double* sc = s + c * ld;
#pragma unroll
    for (int h = 0; h < 16; ++h) {
      if (2 * h + 1 >= c + 1) {
        const double2 l2 = reinterpret_cast<const double2*>(sc)[h];
        if (2 * h >= c + 1) v[2 * h] = fma(-y, l2.x, v[2 * h]);
        v[2 * h + 1] = fma(-y, l2.y, v[2 * h + 1]);
      }
    }
  }
}

// dense NB x NB block (ld NB) in global memory <-> smem tile; every load before the first store
template <int NB, int NT>
__device__ __forceinline__ void load_dense(double* s, const double* src, int t) {
  constexpr int LD = MultiTile<NB>::LD;
  constexpr int E = NB * NB / NT;
  double v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcg(src + t + e * NT);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int idx = t + e * NT;
    s[(idx / NB) * LD + (idx % NB)] = v[e];
  }
}
template <int NB, int NT>
__device__ __forceinline__ void store_dense(const double* s, double* dst, int t) {
  constexpr int LD = MultiTile<NB>::LD;
  for (int idx = t; idx < NB * NB; idx += NT) __stcg(dst + idx, s[(idx / NB) * LD + (idx % NB)]);
}

// ---- TRSM of a tile by substitution: X <- X L^-T (L lower NB x NB), row per thread ------
// Thread r (< NB) owns row r; sdinv[c] = 1 / L(c,c) must be ready.
template <int NB>
__device__ __forceinline__ void trsm_rows(double* sX, const double* __restrict__ sL, const double* __restrict__ sdinv,
                                          int r) {
  constexpr int LD = MultiTile<NB>::LD;
  double x[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) x[c] = sX[c * LD + r];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    x[c] *= sdinv[c];
#pragma unroll
    for (int c2 = c + 1; c2 < NB; ++c2) x[c2] = fma(-x[c], sL[c * LD + c2], x[c2]);
  }
#pragma unroll
  for (int c = 0; c < NB; ++c) sX[c * LD + r] = x[c];
}

// ---- the kernel ------------------------------------------------------------------------
template <int NB, int kPerSM, int kGroups>
__global__ void __launch_bounds__(kMultiThreads, kPerSM)
band_multi_kernel(double* __restrict__ ab, MultiGeom g, MultiWs ws, int32_t* info) {
  static_assert(NB == 32, "the pivot chain is a 32-lane warp POTRF");
  extern __shared__ __align__(16) double smem[];
  constexpr int E = MultiTile<NB>::ELEMS;
  constexpr int LD = MultiTile<NB>::LD;
  __shared__ int s_ok;
  __shared__ int s_fail;
  __shared__ double sdinv[NB];
  const int T = g.T, nblk = g.nblk;
  const int warp = warp_uniform(threadIdx.x >> 5);  // provably warp-uniform branches
  auto TC = [&](int R, int d) -> int* { return ws.tcnt + (size_t)R * (T + 1) + d; };
  auto LR = [&](int R, int d) -> int* { return ws.lrdy + (size_t)R * (T + 1) + d; };

  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) st_release(ws.ctrl + 2, (int)smid + 1);
    // ------------------------------ pivot ---------------------------------------
    // Warp roles (warp w sits on SM sub-partition w & 3):
    //   0      POTRF of (j,j)                       -- the chain, alone on SMSP 0 in stage A
    //   1      L(j,j)^-1 in lock step behind it
    //   2,3    flags + loads of A(j+1,j), L(j+1,j-2)
    //   2,3,6,7  the lookback products (DMMA on SMSPs 2-3 only)
    //   4,5    service, no FP64: write-backs and flag releases of the previous stage B, the
    //          late flag + load of the diagonal tile A(j+1,j+1) (warp 5)
    // Stage B (after the POTRF): warps 0-3 run the TRSM as a product with L(j,j)^-1 and the
    // SYRK of (j+1,j+1) and go on to the next POTRF; warps 6-7 form L(j+2,j); warps 4-5 write
    // back and publish L(j,j)^-1, L(j,j), L(j+1,j), L(j+2,j) behind them.
    __shared__ __align__(8) unsigned long long colbar[8];
    __shared__ int s_okx, s_okd;
    double* sD = smem;             // current diagonal tile (fully updated)
    double* sLp = smem + E;        // L(j, j-1) from the previous step
    double* sInv2 = smem + 2 * E;  // L(j,j)^-1 by step parity (sInv[k*LD + c] = Linv(c, k)): the
                                   // service warps may still be storing the previous one
    double* sW = smem + 4 * E;     // L(j+1, j-1): the previous step's own TRSM of row j+1
    double* sP = smem + 5 * E;     // A(j+1, j)
    double* sD2 = smem + 6 * E;    // A(j+1, j+1)
    double* sX = smem + 7 * E;     // L(j+1, j)
    double* sA2 = smem + 8 * E;    // A(j+2, j)
    double* sX2 = smem + 9 * E;    // L(j+2, j)
    double* sW2 = smem + 10 * E;   // L(j, j-2): the TRSM of row j two steps ago
    double* sV = smem + 11 * E;    // L(j+1, j-2) (the row owner's, from global memory)
    unsigned long long* tr = g_trace;
    load_tile<NB, kMultiThreads>(sD, ab, g, 0, 0, threadIdx.x);
    if (threadIdx.x == 0) {
      s_fail = -1;
      s_ok = 1;
      s_okx = 1;
      s_okd = 1;
      for (int i = 0; i < 8; ++i) mbar_init(colbar + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    int fail_col = -1;
    // Per step ONE CTA-wide barrier (between the stages).  Warps 0-3 run the chain -- POTRF,
    // L^-1, TRSM product, SYRK -- and go straight into the next POTRF; warps 4-7 (service)
    // follow asynchronously: write-backs and releases of step j overlap POTRF(j+1).
    for (int j = 0; j < nblk; ++j) {
      const int nvalid = min(NB, g.n - j * NB);
      double* sInv = sInv2 + (j & 1) * E;
      const bool next = j + 1 < nblk;
      const bool has_w = next && (j >= 1) && (T >= 2);
      const bool has_x2 = (j + 2 < nblk) && (T >= 2);  // row j+2's TRSM is the pivot's too
      const bool has_v = next && (j >= 2) && (T >= 3);  // A(j+1,j) -= L(j+1,j-2) L(j,j-2)^T is the pivot's
      if (threadIdx.x == 0) { trace_stamp_to(tr, j, 0); xstamp(nblk, j, 7); }
      // ---- stage A ----
      if (warp == 0) {
        const int f = warp_potrf32(sD, LD, nvalid, sdinv, colbar);
        if (threadIdx.x == 0) {
          s_fail = f;
          trace_stamp_to(tr, j, 1);
        }
      } else if (warp == 1) {
        warp_inverse32(sD, LD, sdinv, sInv, colbar, (unsigned)(j & 1));
      } else if (next && warp != 4 && warp != 5) {
        // warps 2, 3: the next step's tiles; warps 6, 7 arrive when L(j+1, j-1) (their TRSM of
        // the previous step) is done; then one lookback product each pair
        if (warp == 2 || warp == 3) {
          const int t = threadIdx.x - 64;
          const int lo = max(0, j + 1 - T);
          const int need = max(0, j - 1 - lo);  // worker updates m in [lo, j-2]
          // A(j+1,j): the workers' updates end at step j-3 -- the one of step j-2 needs
          // L(j,j-2), this CTA's own TRSM of the step before last, so it is applied here and
          // not behind a release -> worker -> release round trip
          const int need1 = has_v ? max(0, j - 2 - lo) : need;
          // A(j+1,j) and L(j+1,j-2): their flags are a step old.  The diagonal tile A(j+1,j+1)
          // is fetched by warp 5 (below): its last worker update is released ~2 K cycles into
          // this step, and only the last lookback product needs it.
          if (warp == 2) {
            bool ok = true;
            if (t == 0) ok = spin_ge(TC(j + 1, 1), need1, ws.ctrl + 1, 64);
            if (t == 1 && has_v) ok = spin_ge(LR(j + 1, 3), 1, ws.ctrl + 1, 64);
            ok = __all_sync(kFull, ok);
            if (t == 0) {
              trace_stamp_to(tr, j, 6);
              s_ok = ok;
            }
          }
          named_sync(6, 64);
          if (warp_uniform(s_ok)) {
            if (has_v) load_tiles3<NB, 64, false>(sP, sV, nullptr, ab, g, j + 1, j, j - 2, 0, t);
            else load_tile<NB, 64>(sP, ab, g, j + 1, j, t);
          }
          if (t == 0) trace_stamp_to(tr, j, 7);  // (tiles loaded)
        }
        named_sync(5, 128);  // warps 2, 3, 6, 7: the tiles are in shared memory (sW is the pivot's own)
        if (has_w && warp_uniform(s_ok)) {
          // A(j+1,j) -= L(j+1,j-1) L(j,j-1)^T + L(j+1,j-2) L(j,j-2)^T, one pass over the tile, on
          // four warps (two per SM sub-partition 2 / 3: the FP64 pipes of sub-partitions 0 / 1
          // stay with the POTRF and inverse chains)
          const int w4 = warp < 4 ? warp - 2 : warp - 4;
          tile_gemm<NB, true, 4>(sP, sW, sLp, w4, 5, 128, has_v ? sV : nullptr, sW2);
          // then the diagonal tile, once warp 5 has it: A(j+1,j+1) -= L(j+1,j-1) L(j+1,j-1)^T
          named_sync(10, 160);
          if (warp_uniform(s_okd)) tile_syrk_lower4<NB>(sD2, sW, w4, 5, 128);
        } else {
          named_sync(10, 160);
        }
      } else if (next && warp == 5) {
        // (after this warp's write-back of L(j,j-1), above)
        const int t = threadIdx.x - 160;
        const int need = max(0, j - 1 - max(0, j + 1 - T));  // worker updates m in [lo, j-2]
        if (t == 0) {
          trace_stamp_to(tr, j, 5);  // (warp 5 free for the diagonal tile)
          s_okd = spin_ge(TC(j + 1, 0), need, ws.ctrl + 1, 64);
          trace_stamp_to(tr, j, 4);  // (its flag seen)
        }
        __syncwarp();
        if (warp_uniform(s_okd)) load_tile_unmasked_ok<NB, 32>(sD2, ab, g, j + 1, j + 1, t);
        if (t == 0) trace_stamp_to(tr, j, 3);  // (diagonal tile loaded)
        named_sync(10, 160);
      }
      __syncthreads();
      if (threadIdx.x == 0) trace_stamp_to(tr, j, 2);
      const int fl = warp_uniform(s_fail);
      const int okn = warp_uniform(s_ok) && warp_uniform(s_okx) && warp_uniform(s_okd);
      if (fl >= 0) {
        fail_col = j * NB + fl;
        if (threadIdx.x == 0) atomicExch(ws.ctrl + 1, fail_col + 1);
        break;
      }
      if (next && !okn) break;  // aborting
      // ---- stage B ----
      if (warp == 4) {
        // the inverse first: every row's TRSM waits for it (L(j,j) itself is only output)
        const int t = threadIdx.x - 128;
        store_dense<NB, 32>(sInv, ws.inv + (size_t)j * NB * NB, t);
        __syncwarp();
        if (t == 0) { st_release(LR(j, 0), 1); xstamp(nblk, j + 1, 6); }
        store_tile<NB, 32>(sD, ab, g, j, j, t);
        if (has_x2) {
          named_sync(8, 96);  // warps 6, 7: L(j+2, j) is in sX2 (they go straight on to the lookback)
          if (warp_uniform(s_okx)) {
            store_tile<NB, 32>(sX2, ab, g, j + 2, j, t);
            __syncwarp();
            if (t == 0) st_release(LR(j + 2, 2), 1);
          }
        }
      } else if (warp == 5) {
        if (next) {
          const int t = threadIdx.x - 160;
          named_sync(4, 160);  // the TRSM product is in sX
          store_tile<NB, 32>(sX, ab, g, j + 1, j, t);
          __syncwarp();
          if (t == 0) st_release(LR(j + 1, 1), 1);
        }
      } else if (warp >= 6) {
        // L(j+2,j) = A(j+2,j) L(j,j)^-T as soon as the row owner's last task has published
        // A(j+2,j) -- not tied to the stage barrier (the next POTRF and the release of
        // L(j,j)^-1 do not wait for it): the next step's lookback products read it from shared
        // memory (these warps join that step's barrier of warps 2-7 when it is done), the
        // workers' updates of column j+1 from global memory
        if (has_x2) {
          const int t = threadIdx.x - 192;
          if (t == 0) s_okx = spin_ge(TC(j + 2, 2), max(0, j - max(0, j + 2 - T)), ws.ctrl + 1, 64);
          named_sync(7, 64);
          if (warp_uniform(s_okx)) {
            load_tile<NB, 64>(sA2, ab, g, j + 2, j, t);
            named_sync(7, 64);
            tile_gemm<NB, false, 2, true>(sX2, sA2, sInv, warp - 6, 7, 64);
          }
          asm volatile("bar.arrive 8, 96;" ::: "memory");  // warp 4 writes it back and publishes it
        }
      } else if (next) {
        tile_gemm<NB, false, 4, true>(sX, sP, sInv, warp, 2, 128);  // L(j+1,j) = A(j+1,j) L(j,j)^-T
        asm volatile("bar.arrive 4, 160;" ::: "memory");
        tile_syrk_lower4<NB>(sD2, sX, warp, 2, 128);  // A(j+1,j+1) -= L(j+1,j) L(j+1,j)^T (lower blocks)
      }
      if (!next) break;
      // rotate (every thread for itself, no barrier).  Buffers that lagging warps may still
      // use: old sD (warp 4's write-back, done before the next stage barrier) becomes sA2,
      // loaded after that barrier; sX and sX2 (write-backs) become sLp and sW, read-only; old
      // sA2 (warps 6-7's TRSM input) becomes sX2, their own; old sLp / sW / sP are free since
      // this step's stage barrier / TRSM and become sP / sD2 / sX.
      {
        double* const oD = sD; double* const oLp = sLp; double* const oW = sW; double* const oW2 = sW2;
        double* const oP = sP; double* const oA2 = sA2;
        sD = sD2; sLp = sX; sW = sX2; sW2 = oW;
        sP = oLp; sD2 = oW2; sX = oP; sA2 = oD; sX2 = oA2;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int fl = ld_volatile(ws.ctrl + 1);
      info[0] = fail_col >= 0 ? fail_col + 1 : (fl ? fl : 0);
    }
    return;
  }

  // -------------------------------- workers -------------------------------------------
  // The pivot's SM is left to the pivot: its chain is the critical path, and worker
  // tiles on the same SM would compete for its issue slots and pipes.  (Cooperative
  // launch: block 0 is resident, so its id appears.)
  {
    __shared__ int s_piv;
    if (threadIdx.x == 0) {
      int v;
      while ((v = ld_acquire(ws.ctrl + 2)) == 0) __nanosleep(64);
      s_piv = v - 1;
    }
    __syncthreads();
    if (s_piv == (int)smid) return;
  }
  // kGroups independent warp groups per CTA (2 for wide bands), each with its own three
  // tiles, its own named barrier and its own tickets: while one group waits on a flag or
  // an L2 round trip the other computes.  The next ticket is fetched while the current
  // task runs (a held, not-yet-started ticket cannot deadlock: the smallest unfinished
  // ticket is always a group's current task, and its dependencies are all smaller).
  constexpr int GT = kMultiThreads / kGroups, GW = GT / 32;
  constexpr bool kPrefetchTicket = BCG_MULTI_PREFETCH;
  const int grp = warp / GW, gt = threadIdx.x - grp * GT, wg = warp - grp * GW;
  const int bar = 1 + grp;
  __shared__ int s_task2[kGroups], s_ok2[kGroups];
  double* sA = smem + grp * 3 * E;
  double* sB = sA + E;
  double* sC = sA + 2 * E;
  const int Q = g.Q;
  const long long total = (long long)(nblk + 1) * Q;  // super-step nblk: the last rest updates
  int held = -1;  // (thread 0 of the group) a ticket fetched early, not yet started
  auto gsync = [&]() { named_sync(bar, GT); };
  // cumulative release after the group barrier, by the last warp's lane 0: the release waits
  // until the group's stores are performed (~1 K cycles), and thread 0 spends that time
  // fetching the next ticket and reading its flags
  auto gpublish = [&](int* flag, int value) {
    gsync();
    if (gt == GT - 32) st_release(flag, value);
  };
  // one thread: wait for up to three flags (issued together, then spun on one by one)
  auto wait3 = [&](const int* f0, int v0, const int* f1, int v1, const int* f2, int v2) -> bool {
    const int a0 = ld_acquire(f0), a1 = f1 ? ld_acquire(f1) : v1, a2 = f2 ? ld_acquire(f2) : v2;
    if (a0 < v0 && !spin_ge(f0, v0, ws.ctrl + 1, kWorkerSpinNs)) return false;
    if (a1 < v1 && !spin_ge(f1, v1, ws.ctrl + 1, kWorkerSpinNs)) return false;
    if (a2 < v2 && !spin_ge(f2, v2, ws.ctrl + 1, kWorkerSpinNs)) return false;
    return true;
  };
#ifdef BCG_TRACE
  unsigned long long acc_ph[6] = {0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
  auto ph = [&](int k) {
    const long long now = clock64();
    acc_ph[k] += (unsigned long long)(now - tprev);
    tprev = now;
  };
#else
  auto ph = [&](int) {};
#endif
  for (;;) {
    if (gt == 0) {
      s_task2[grp] = held >= 0 ? held : atomicAdd(ws.ctrl, 1);
      held = -1;
    }
    gsync();
    const long long t = warp_uniform(s_task2[grp]);
    if (t >= total) break;
    ph(0);
    // Ticket order, super-step s (Q tickets):
    //   A  the updates of step s-1 to the tile column s+1 (rows s+2..),
    //   B  the row tasks of step s: TRSM L(R,s) = A(R,s) L(s,s)^-T, then -- with L(R,s)
    //      still in shared memory -- the update of (R, s+1), which the row's TRSM of step
    //      s+1 waits for: one task per row per step on the critical row chain,
    //   C  the remaining updates of step s-1 (columns s+2..).
    // A topological order (B needs A of its super-step and B of the previous one; C needs
    // the TRSMs of step s-1), and the critical row tasks never queue behind C.
    const int sstep = (int)(t / Q), q = (int)(t - (long long)sstep * Q);
    const int nA = T - 1, nB = T - 1;
    if (q >= nA && q < nA + nB) {
      // One row task: TRSM L(R,m) = A(R,m) L(m,m)^-T as a product with the published inverse,
      // then -- L(R,m) still in sC -- the row's update of tile (R, m+1), the input of its next
      // TRSM.  resident: A(R,m) is already in sA, complete (left there by the previous task of
      // the same owner); keep: leave the updated (R, m+1) in sA instead of publishing it.
      auto row_task = [&](int m, int R, bool resident, bool keep) -> bool {
        if (gt == 0)
          s_ok2[grp] = resident ? wait3(LR(m, 0), 1, nullptr, 0, nullptr, 0)
                                : wait3(LR(m, 0), 1, TC(R, R - m), m - max(0, R - T), nullptr, 0);
        gsync();
        if (!warp_uniform(s_ok2[grp])) return false;
        ph(1);
#ifdef BCG_TRACE
        const long long rt0 = clock64();
        if (gt == 0 && m == R - 3) xstamp(nblk, R - 2, 0);
#endif
        if (!resident) load_tile<NB, GT>(sA, ab, g, R, m, gt);
        load_dense<NB, GT>(sB, ws.inv + (size_t)m * NB * NB, gt);
        gsync();
        ph(2);
        tile_gemm<NB, false, GW, (GW <= 4)>(sC, sA, sB, wg, bar, GT);
        store_tile<NB, GT>(sC, ab, g, R, m, gt);
        ph(3);
        gpublish(LR(R, R - m), 1);
        ph(4);
        if (gt == 0 && m == R - 3) xstamp(nblk, R - 2, 1);
        const int S = m + 1;
        if (R >= m + 3 && S < nblk) {  // ((m+2, m+1) is the pivot's)
          const int done = m - max(0, R - T);
          if (gt == 0) s_ok2[grp] = wait3(LR(S, 1), 1, TC(R, R - S), done, nullptr, 0);
          gsync();
          if (!warp_uniform(s_ok2[grp])) return false;
          ph(1);
          if (gt == 0 && m == R - 3) xstamp(nblk, R - 2, 2);
          load_tile<NB, GT>(sB, ab, g, S, m, gt);
          load_tile<NB, GT>(sA, ab, g, R, S, gt);
          gsync();
          ph(2);
          tile_gemm<NB, true, GW>(sA, sC, sB, wg, bar, GT);
          if (!keep) {
            store_tile<NB, GT>(sA, ab, g, R, S, gt);
            ph(3);
            gpublish(TC(R, R - S), done + 1);
            ph(4);
            if (gt == 0 && m == R - 3) xstamp(nblk, R - 2, 3);
          }
        }
#ifdef BCG_TRACE
        if (gt == 0 && g_trace && g_trace_cap > 8) {  // row-task latency: sum and count
          atomicAdd(g_trace + g_trace_cap - 8 + 5, (unsigned long long)(clock64() - rt0));
          atomicAdd(g_trace + g_trace_cap - 8 + 6, 1ull);
        }
#endif
        return true;
      };
      const int R = sstep + 2 + (q - nA);
      // (row s + 2 is the pivot's: it forms L(s+2, s) itself during its next step)
      if (R >= nblk || sstep >= nblk || R == sstep + 2) { gsync(); continue; }
      if (g.owner) {
        // ROW OWNER: the ticket of the super-step in which row R enters the band (m0) runs the
        // row's whole chain of tasks m0 .. R-3 on one worker group, the tile between two of them
        // staying in shared memory: the store -> release -> acquire -> load round trip through
        // L2 (and the group switch) leaves the row chain TRSM(m) -> update -> TRSM(m+1).  The
        // last task (m = R-3) publishes tile (R, R-2) for the pivot's own TRSM.  An owner holds
        // its group for <= T steps; g.owner is set only when the grid has spare groups.
        const int m0 = max(0, R - T);
        if (sstep != m0) { gsync(); continue; }
        bool ok = true, resident = false;
        for (int m = m0; m <= R - 3 && ok; ++m) {
          const bool keep = m < R - 3;
          ok = row_task(m, R, resident, keep);
          resident = keep;
        }
        if (!ok) break;
      } else {
        if (!row_task(sstep, R, false, false)) break;
      }
    } else {
      // updates of step s-1: part A (b = a-1: column s+1) or part C (b <= a-2)
      const int j = sstep - 1;
      int a, b;
      if (q < nA) {
        a = q + 1;
        b = a - 1;
      } else {
        const int v = q - nA - nB;
        int w = (int)((1.0f + sqrtf(8.0f * (float)v + 1.0f)) * 0.5f);
        while (w * (w - 1) / 2 > v) --w;
        while ((w + 1) * w / 2 <= v) ++w;
        a = w + 1;
        b = v - w * (w - 1) / 2;
      }
      const int R = j + 1 + a, S = R - b;
      if (j < 0 || j >= nblk) { gsync(); continue; }
      // pivot's: rows j+1, j+2 near the diagonal, and (j+3, j+2) (needs the pivot's own L(j+2, j))
      const bool pivot_owned = (R == j + 1) || (R == j + 2 && S >= j + 1) || (R == j + 3 && S == j + 2 && T >= 3);
      if (R >= nblk || pivot_owned) { gsync(); continue; }
      const int done = j - max(0, R - T);
      if (gt == 0)
        s_ok2[grp] = wait3(LR(R, R - j), 1, LR(S, S - j), 1, TC(R, R - S), done);
      gsync();
      if (!warp_uniform(s_ok2[grp])) break;
      ph(1);
      // the next ticket while this task's tiles travel (update tasks only: a row owner keeps
      // its group for many steps and must not sit on an unstarted ticket).  A held ticket
      // cannot deadlock: this task's dependencies are all on smaller tickets.
      if (kPrefetchTicket && gt == 0) held = atomicAdd(ws.ctrl, 1);
      load_tile<NB, GT>(sA, ab, g, R, j, gt);
      load_tile<NB, GT>(sB, ab, g, S, j, gt);
      load_tile<NB, GT>(sC, ab, g, R, S, gt);
      gsync();
      ph(2);
      tile_gemm<NB, true, GW>(sC, sA, sB, wg, bar, GT);
      store_tile<NB, GT>(sC, ab, g, R, S, gt);
      ph(3);
      gpublish(TC(R, R - S), done + 1);
      ph(4);
    }
  }
#ifdef BCG_TRACE
  // worker phase totals (cycles, summed over groups): ticket, deps, loads, compute, publish
  if (gt == 0 && g_trace && g_trace_cap > 8)
    for (int k = 0; k < 5; ++k) atomicAdd(g_trace + g_trace_cap - 8 + k, acc_ph[k]);
#endif
}

// ---- host side -------------------------------------------------------------------------
constexpr int kMultiNB = 32;

inline bool use_multi(int n, int kd) { (void)n; return kd >= 160; }

inline MultiGeom multi_geom(int n, int kd, int ldab) {
  MultiGeom g;
  g.n = n;
  g.kd = kd;
  g.ldab = ldab;
  g.nblk = (n + kMultiNB - 1) / kMultiNB;
  g.T = (kd + kMultiNB - 1) / kMultiNB;
  g.Q = (g.T - 1) + g.T * (g.T - 1) / 2;  // per super-step: T-1 row tasks + the step's other updates
  g.owner = 0;
  return g;
}

inline size_t multi_workspace_bytes(int n, int kd) {
  MultiGeom g = multi_geom(n, kd, kd + 1);
  return multi_flag_bytes(g.nblk, g.T) + (size_t)g.nblk * kMultiNB * kMultiNB * sizeof(double);
}

// Occupancy: wide bands (many worker tasks per step) run 3 CTAs per SM for latency
// hiding; narrower bands keep 2 so the pivot CTA gets the registers of its chain.
template <int kPerSM, int kGroups>
inline int launch_multi_t(double* ab, int n, int kd, int ldab, int32_t* info, void* workspace, int sms,
                          cudaStream_t st, char* err, size_t errlen) {
  constexpr int NB = kMultiNB;
  MultiGeom g = multi_geom(n, kd, ldab);
  // pivot: 12 tiles; workers: 3 per group
  const size_t smem = (size_t)(3 * kGroups > 12 ? 3 * kGroups : 12) * MultiTile<NB>::ELEMS * sizeof(double);
  auto k = band_multi_kernel<NB, kPerSM, kGroups>;
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
  if (per_sm > kPerSM) per_sm = kPerSM;
  e = cudaMemsetAsync(workspace, 0, multi_flag_bytes(g.nblk, g.T), st);
  if (e != cudaSuccess) {
    snprintf(err, errlen, "cudaMemsetAsync(workspace): %s", cudaGetErrorString(e));
    return (int)e;
  }
  MultiWs ws = multi_ws(workspace, g.nblk, g.T);
  int grid = sms * per_sm;
  // row owners hold up to T groups at a time: only with at least twice as many (plus slack)
  g.owner = ((long long)(sms - 1) * per_sm * kGroups >= 2LL * g.T + 16) ? 1 : 0;
  if (const char* e = getenv("BCG_MULTI_NO_OWNER")) {  // (tests: the one-ticket-per-link fallback)
    if (e[0] == '1') g.owner = 0;
  }
  void* args[] = {(void*)&ab, (void*)&g, (void*)&ws, (void*)&info};
  e = cudaLaunchCooperativeKernel((void*)k, dim3(grid), dim3(kMultiThreads), args, smem, st);
  if (e != cudaSuccess) {
    snprintf(err, errlen, "cudaLaunchCooperativeKernel(band_multi): %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

inline int launch_multi(double* ab, int n, int kd, int ldab, int32_t* info, void* workspace, int sms,
                        cudaStream_t st, char* err, size_t errlen) {
  if (kd >= 1000) return launch_multi_t<BCG_WIDE_PERSM, BCG_WIDE_GROUPS>(ab, n, kd, ldab, info, workspace, sms, st, err, errlen);
  return launch_multi_t<1, 1>(ab, n, kd, ldab, info, workspace, sms, st, err, errlen);
}

}  // namespace bcg
