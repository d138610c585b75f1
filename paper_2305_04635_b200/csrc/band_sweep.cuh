// band_sweep.cuh -- streamed band solve L L^T X = B for R right-hand sides per CTA
// (the reference's solve_with_factor, pkg/src/bandchol/core.py:216-240, generalised to
// several right-hand sides that share one pass over L).
//
// One CTA per (matrix, group of <= R right-hand sides).  The factor streams through a
// ring of nbuf shared-memory buffers of 16 columns (bulk async copies, one mbarrier pair
// per buffer) twice: forward in column order, backward in reverse.  Block b = rows and
// columns 16b..16b+15, Linv_b = L_bb^-1, N_b = L_{b,b-1}, N'_b = L_{b+1,b}:
//   forward   y_b = t_b - H_b y_{b-1},   H_b = Linv_b N_b,
//             t_b = Linv_b (b_b + acc_b - L_{b,b-2} y_{b-2}),
//             acc_i -= sum_{c in block b} L(i, c) y_c   for rows i >= 16b+48 (far update)
//   backward  x_b = t_b - G_b^T x_{b+1},   G_b = N'_b Linv_b,
//             t_b = Linv_b^T (y_b - f_b - L_{b+2,b}^T x_{b+2}),
//             f_b  = sum_{rows i >= 16b+48} L(i, block b)^T x_i   (far dot products)
// so the serial path (the chain) is ONE 16x16 product per block; everything else is
// computed ahead of it by other warps.  Warp roles, mbarrier dataflow only (no CTA-wide
// barrier inside the sweeps):
//   warp 0     chain: y_b / x_b
//   warps 1-3  prep (blocks round robin): one triangular substitution per block with 32
//              right-hand sides -- lanes 0-15 give Linv_b, lanes 16-31 H_b (forward) or
//              G_b (backward), the same instructions -- then t_b once its inputs are
//              complete (forward: after y_{b-2} and the far update by y_{b-3}; backward:
//              after x_{b+2} and the far dot products of block b)
//   warps 4-6  far: the far update / far dot products on the FP64 tensor path (DMMA), no
//              barrier among them
//   warp 7     producer: waits for a free buffer, loads the block's right-hand-side rows
//              (forward: b, backward: y) with cp.async and issues the bulk copy of its
//              16 columns
// A step s numbers the blocks of both sweeps (forward b = s, backward b = 2*nblk-1-s);
// every ring index and mbarrier parity is a function of s.
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "band_cta.cuh"
#include "band_solve.cuh"

namespace bcg {

constexpr int kSweepWarps = 8;
constexpr int kSweepThreads = 32 * kSweepWarps;
constexpr int kSweepPrepWarps = 3;
constexpr int kSweepFarWarps = 3;
// prep ring slots and backward far partials per column: the FMA path (R <= 2) runs prep
// further ahead and splits a column over 6 row chunks; the DMMA path (R >= 8) keeps 4 slots
// and one partial per far warp, so that two R = 8 CTAs fit on an SM
__host__ __device__ constexpr int sweep_np(int R) { return R <= 2 ? 6 : 4; }
__host__ __device__ constexpr int sweep_parts(int R) { return R <= 2 ? 6 : 3; }
constexpr int kSweepNPMax = 6;
constexpr int kSweepNY = 4;      // chain-output / t ring slots (a power of two)
constexpr int kLinvLd = 18;      // row stride of a prep matrix (16-byte aligned rows)
constexpr int kPrepSlot = 2 * 16 * kLinvLd;  // [0] Linv (for t), [1] H / G (for the chain)
constexpr int kFarBar = 2;       // named barrier of the far warps

struct SweepGeom {
  int n, kd, ldab;
  int nblk;   // ceil(n / 16)
  int nbuf;   // L buffers in the ring (4..8)
  int nx;     // rows of the accumulator / solution ring (multiple of 16, >= kd + 16)
};

// Shared-memory footprint in doubles (before the mbarriers, which are static).
__host__ __device__ inline size_t sweep_smem_doubles(const SweepGeom& g, int R) {
  return (size_t)g.nbuf * 16 * g.ldab          // L ring
         + (size_t)g.nbuf * 16 * R              // right-hand-side rows per buffer
         + (size_t)sweep_np(R) * kPrepSlot      // prep ring
         + (size_t)kSweepNY * 16 * R            // chain outputs
         + (size_t)kSweepNY * 16 * R            // t
         + (size_t)4 * sweep_parts(R) * 16 * R  // backward far partials (a ring of 4 steps)
         + (size_t)kSweepPrepWarps * 16 * R     // the prep warps' staged vectors
         + (size_t)g.nx * R;                    // accumulator / solution ring
}

// C (16 x R) += A (16 x 16, row r at a[r * lda + k]) * B (16 x R, b[k * R + n]) on the FP64
// tensor path (R = 8 or 16: one or two 8-wide n-tiles; mma.sync m8n8k4 f64).  Lane (gr, gc)
// ends holding C[8 mt + gr][8 nt + 2 gc + e] in acc[mt][nt][e].
template <int R>
__device__ __forceinline__ void dmma_16x16xR(const double* a, int lda, const double* b, double (&acc)[2][R / 8][2]) {
  const int lane = threadIdx.x & 31, gr = lane >> 2, gc = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    double af[2], bf[R / 8];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) af[mt] = a[(8 * mt + gr) * lda + 4 * ks + gc];
#pragma unroll
    for (int nt = 0; nt < R / 8; ++nt) bf[nt] = b[(4 * ks + gc) * R + 8 * nt + gr];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < R / 8; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
  }
}

// a phase-tracked position in a ring of `size` slots: slot and parity advance together
struct RingPos {
  int slot = 0;
  unsigned par = 0;
  __device__ __forceinline__ void next(int size) {
    if (++slot == size) { slot = 0; par ^= 1u; }
  }
};

// prep, forward step: L_bb X = [I | N_b] by column-oriented forward substitution (columns of
// L_bb are broadcast loads; the reciprocal pivots are computed up front).  Lane j < 16
// solves for e_j (column j of Linv_b), lane 16 + j for N_b(:, j) (column j of H_b), rows
// past the matrix are identity.  out[i*kLinvLd + j] = X(i, j) of the lane's half.
// kWhole (a full block, kd >= 31): every operand is in the band, so each load is
// base + constant offset and no entry needs a mask -- the instruction stream this warp
// issues is the cost, so the interior blocks take this path.
template <bool kWhole>
__device__ __forceinline__ void prep_forward(const double* blk, const double* prevb, bool has_prev, int nb, int kd,
                                             int ldab, int j, bool second, double* out) {
  // bit i of ej = (e_j)_i, made opaque: with `i == j` (or a visible 1 << j) the compiler turns
  // the initialisation into a dynamically indexed store and moves t[] to local memory
  unsigned ej;
  asm("mov.b32 %0, %1;" : "=r"(ej) : "r"(1u << j));
  const int st = ldab - 1;  // AB storage: (r, c) -> (r + 1, c + 1) is ldab doubles on, (r, c+1) st
  double dk[16], t[16];
  if (kWhole) {
    const double* nj = prevb + j * st + 16;  // N_b(i, j) = nj[i]
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) dk[kk] = blk[kk * ldab];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double nv = nj[i];
      t[i] = second ? nv : (((ej >> i) & 1u) ? 1.0 : 0.0);
    }
  } else {
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const double d = blk[(kk < nb ? kk : 0) * ldab];  // (unconditional load + select: no branch)
      dk[kk] = kk < nb ? d : 1.0;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int o = 16 + i - j;
      const bool in = has_prev && i < nb && o <= kd;
      const double nv0 = prevb[j * ldab + (in ? o : 0)];
      const double nv = in ? nv0 : 0.0;
      t[i] = second ? nv : (((ej >> i) & 1u) ? 1.0 : 0.0);
    }
  }
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) dk[kk] = rcp_nr(dk[kk]);
  // fixed 16 x 16 iteration space (conditions fold at compile time after unrolling); in the
  // masked path unconditional in-bounds loads + select (a conditional load is a branch)
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    t[kk] *= dk[kk];
    const double* col = blk + kk * ldab;  // column kk: L(i, kk) = col[i - kk]
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i <= kk) continue;
      if (kWhole) {
        t[i] = fma(-col[i - kk], t[kk], t[i]);
      } else {
        const bool in = i < nb && i - kk <= kd;
        const double lv = col[in ? i - kk : 0];
        t[i] = fma(in ? -lv : 0.0, t[kk], t[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) out[i * kLinvLd + j] = t[i];
}

// prep, backward step: X^T L_bb = [I | N'_b]^T row by row, z_kk = r_kk / L(kk,kk) and
// r_m -= z_kk L(kk, m) from the last column.  Lane j < 16: row j of Linv_b, lane 16 + j:
// row j of G_b = N'_b Linv_b (N'_b(j, k) = L(c0+16+j, c0+k), `rows` rows below the block).
// out[k*kLinvLd + j] = X(j, k): the chain and t read row i as [i*kLinvLd + k] = X(k, i).
// kWhole: a full block with a full block below it and kd >= 31 (no masks).
template <bool kWhole>
__device__ __forceinline__ void prep_backward(const double* blk, int rows, int nb, int kd, int ldab, int j,
                                              bool second, double* out) {
  unsigned ej;  // (opaque, as in prep_forward)
  asm("mov.b32 %0, %1;" : "=r"(ej) : "r"(1u << j));
  const int st = ldab - 1;
  double dk[16], t[16];
  if (kWhole) {
    const double* nj = blk + 16 + j;  // N'_b(j, k) = L(c0+16+j, c0+k) = nj[k * st]
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) dk[kk] = blk[kk * ldab];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double nv = nj[k * st];
      t[k] = second ? nv : (((ej >> k) & 1u) ? 1.0 : 0.0);
    }
  } else {
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const double d = blk[(kk < nb ? kk : 0) * ldab];
      dk[kk] = kk < nb ? d : 1.0;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int o = 16 + j - k;
      const bool in = j < rows && k < nb && o <= kd;
      const double nv0 = blk[k * ldab + (in ? o : 0)];
      const double nv = in ? nv0 : 0.0;
      t[k] = second ? nv : (((ej >> k) & 1u) ? 1.0 : 0.0);
    }
  }
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) dk[kk] = rcp_nr(dk[kk]);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int kk = 15 - q;
    t[kk] *= dk[kk];
    const double* row = blk + kk;  // row kk: L(kk, m) = row[m * st]
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      if (m >= kk) continue;
      if (kWhole) {
        t[m] = fma(-row[m * st], t[kk], t[m]);
      } else {
        const bool in = kk < nb && kk - m <= kd;
        const double lv = blk[m * ldab + (in ? kk - m : 0)];
        t[m] = fma(in ? -lv : 0.0, t[kk], t[m]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) out[k * kLinvLd + j] = t[k];
}

template <int R>
__global__ void __launch_bounds__(kSweepThreads, R <= 8 ? 2 : 1)
pbtrs_sweep_kernel(const double* __restrict__ ab0, int64_t stride_ab, double* b0, int64_t ldb, int64_t stride_b,
                   int nrhs, int groups, SweepGeom g, int32_t* info, const int32_t* skip, int check_diag,
                   const double* y0, int64_t stride_y) {
  extern __shared__ __align__(16) double smem[];
  constexpr int kSweepNP = sweep_np(R);
  __shared__ __align__(8) unsigned long long full[8], empty[8], pfull[kSweepNPMax], pempty[kSweepNPMax];
  __shared__ __align__(8) unsigned long long ydone[kSweepNY], fardone[kSweepNY], tdone[kSweepNY], fwd_done;

  const int mat = blockIdx.x / groups, grp = blockIdx.x - mat * groups;
  if (skip && skip[mat] != 0) return;  // (after a batched factorization: this one failed, keep its info)
  const double* ab = ab0 + (int64_t)mat * stride_ab;
  const int r0 = grp * R;
  const int rv = min(R, nrhs - r0);  // valid right-hand sides of this group
  double* bm = b0 + (int64_t)mat * stride_b + (int64_t)r0 * ldb;
  // y0: the forward sweep already ran (fused into the factorization, y of this matrix at
  // y0 + mat * stride_y): only the nblk backward steps run, reading y from there
  const double* ym = y0 ? y0 + (int64_t)mat * stride_y + (int64_t)r0 * ldb : bm;
  if (check_diag) {
    // the reference checks every diagonal entry before any arithmetic (core.py:227-230)
    const int bad = first_nonpositive_diag(ab, g.n, g.ldab);
    if (bad != INT_MAX) {
      if (threadIdx.x == 0 && grp == 0) info[mat] = bad + 1;
      return;
    }
  }
  const int n = g.n, kd = g.kd, ldab = g.ldab, nblk = g.nblk, nbuf = g.nbuf, nx = g.nx;
  const int warp = warp_uniform(threadIdx.x >> 5), lane = threadIdx.x & 31;

  double* Lring = smem;
  double* rbuf = Lring + (size_t)nbuf * 16 * ldab;   // [nbuf][16 rows][R]
  double* prep = rbuf + (size_t)nbuf * 16 * R;        // [NP][2][16][kLinvLd]
  double* ych = prep + kSweepNP * kPrepSlot;          // [NY][16][R]
  double* tbuf = ych + kSweepNY * 16 * R;             // [NY][16][R]
  double* fpart = tbuf + kSweepNY * 16 * R;           // [4][kFarParts][16][R]
  double* cstage = fpart + 4 * sweep_parts(R) * 16 * R;  // [kSweepPrepWarps][16][R]
  double* ring = cstage + kSweepPrepWarps * 16 * R;   // [nx][R]

  if (threadIdx.x < 8) {
    mbar_init(&full[threadIdx.x], 1 + 32);  // the bulk copy's expect_tx + 32 producer lanes' cp.async
    mbar_init(&empty[threadIdx.x], kSweepFarWarps + 3);  // every far warp, three prep arrivals
  }
  if (threadIdx.x < kSweepNP) {
    mbar_init(&pfull[threadIdx.x], 1);
    mbar_init(&pempty[threadIdx.x], 1);
  }
  if (threadIdx.x < kSweepNY) {
    mbar_init(&ydone[threadIdx.x], 1);
    mbar_init(&fardone[threadIdx.x], kSweepFarWarps);
    mbar_init(&tdone[threadIdx.x], 1);
  }
  if (threadIdx.x == 0) mbar_init(&fwd_done, 1);
  for (int i = threadIdx.x; i < nx * R; i += kSweepThreads) ring[i] = 0.0;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  const int nf = y0 ? 0 : nblk;  // forward steps
  const int nsteps = nf + nblk;
#ifdef BCG_TRACE
  // phase stamps of CTA 0 (SM cycles), per step s: chain 0 start, 1 waits done, 2 end;
  // far 3 waits done, 4 done; prep 5 substitution done, 6 t's waits done, 7 t published.
  // [0] = steps (written once): no global read per stamp.
  // (not in backward-only mode: the fused factorization before it owns the trace buffer)
  unsigned long long* const tr = (blockIdx.x == 0 && !y0) ? g_trace : nullptr;
  const unsigned long long tcap = g_trace_cap;  // (read once: no global load inside a phase)
  auto stamp = [&](int step, int ph) {
    if (tr && (threadIdx.x & 31) == 0) {
      const unsigned long long idx = 1 + (unsigned long long)step * kTracePhases + ph;
      if (idx < tcap) tr[idx] = gtime();
    }
  };
  if (tr && threadIdx.x == 0) tr[0] = nsteps;
#else
  auto stamp = [](int, int) {};
#endif
  auto block_of = [&](int s) { return s < nf ? s : nf + nblk - 1 - s; };
  auto Lbuf = [&](int s) { return Lring + (size_t)(s % nbuf) * 16 * ldab; };
  auto full_wait = [&](int s) { mbar_wait(&full[s % nbuf], (unsigned)(s / nbuf) & 1u); };
  constexpr int RL = R == 1 ? 1 : R / 2;
  constexpr bool kScalar = R <= 2;  // far work on the FMA pipe (else DMMA)
  constexpr int kFarParts = sweep_parts(R);  // backward partials per column
  static_assert(kFarParts == (kScalar ? 2 * kSweepFarWarps : kSweepFarWarps), "partials per column");
  const int i = lane & 15, h = lane >> 4;
  const bool store = R > 1 || h == 0;  // R == 1: both halves compute, only h == 0 stores
  auto rhs_of = [&](int rr) { return R == 1 ? 0 : h + 2 * rr; };
  // prep's t staging (R >= 8: contiguous runs, lane half h takes rhs [RL h, RL h + RL))
  auto stage_of = [&](int rr) { return R >= 8 ? RL * h + rr : rhs_of(rr); };

  if (warp == kSweepWarps - 1) {
    // ---------------------------------- producer ----------------------------------
    const bool bulk_ok = !(((uintptr_t)ab) & 15);
    for (int s = 0; s < nsteps; ++s) {
      const int k = s % nbuf;
      if (s >= nbuf) mbar_wait(&empty[k], (unsigned)(s / nbuf - 1) & 1u);
      if (s == nf && nf > 0) mbar_wait(&fwd_done, 0);  // y is complete in global memory
      const int b = block_of(s), c0 = 16 * b, cols = min(16, n - c0);
      // right-hand-side rows of the block (forward: b, backward: y): 8-byte cp.async (zero fill
      // past n / past the group's right-hand sides).  full[k] completes after 32 lane
      // arrivals that trigger once each lane's cp.asyncs landed, plus the bulk copy's bytes.
      double* rb = rbuf + (size_t)k * 16 * R;
      for (int e = lane; e < 16 * R; e += 32) {
        const int ii = e / R, r = e - ii * R;
        const bool ok = ii < cols && r < rv;
        cp_async8_zfill(rb + e, ok ? ym + (int64_t)r * ldb + c0 + ii : ym, ok);
      }
      double* dst = Lbuf(s);
      const double* src = ab + (int64_t)c0 * ldab;
      const int total = cols * ldab;
      const int nb2 = bulk_ok ? (total & ~1) : 0;  // bulk part: a 16-byte multiple
      for (int e = nb2 + lane; e < total; e += 32) cp_async8_zfill(dst + e, src + e, true);
      cp_async_mbar_arrive(&full[k]);
      if (lane == 0) {
        mbar_expect_tx(&full[k], (unsigned)nb2 * 8u);
        if (nb2) bulk_g2s(dst, src, (unsigned)nb2 * 8u, &full[k]);
      }
    }
    return;
  }

  if (warp >= 1 && warp <= kSweepPrepWarps) {
    // ------------------------------------ prep ------------------------------------
    // Step s (s = w, w + 3, ...):
    //  1. one triangular substitution with 32 right-hand sides.  Forward: L_bb X = [I | N_b];
    //     lane j < 16 gets column j of Linv_b, lane 16 + j column j of H_b (N_b comes from
    //     the previous block's buffer).  Backward: X^T L_bb = [I | N'_b]^T row by row; lane j
    //     gets row j of Linv_b, lane 16 + j row j of G_b.  Stored so that row i of each
    //     operand is [i*kLinvLd + k] for its reader: forward Linv(i, k) and H(i, k), backward
    //     Linv(k, i) and G(k, i).
    //  2. t_b, once its inputs are complete: forward (after the far update by y_{b-2})
    //     t_b = Linv_b (b_b + acc_b), zeroing the accumulators; backward (after the far dot
    //     products of the step) t_b = Linv_b^T (y_b - f_b), the chunk partials summed in a
    //     fixed order.  Published to tbuf, then tdone.
    // Buffer releases: three per step (see the end of the step).
    const int j = lane & 15;
    const bool second = lane >= 16;
    double* cv = cstage + (warp - 1) * 16 * R;
    for (int s = warp - 1; s < nsteps; s += kSweepPrepWarps) {
      const int p = s % kSweepNP;
      if (s >= kSweepNP) mbar_wait(&pempty[p], (unsigned)(s / kSweepNP - 1) & 1u);
      const bool fwd = s < nf;
      full_wait(s);
      if (fwd && s >= 1) full_wait(s - 1);
      if (fwd && s >= 2) full_wait(s - 2);
      
      const int b = block_of(s), c0 = 16 * b, nb = min(16, n - c0);
      const double* blk = Lbuf(s);
      double* slot = prep + p * kPrepSlot;
      double* out = slot + (second ? 16 * kLinvLd : 0);
      if (fwd) {
        // right-hand side: e_j, or N_b(:, j) = L(c0 + i, c0 - 16 + j) from the previous buffer
        const double* pb = Lbuf(s == 0 ? 0 : s - 1);
        if (kd >= 31 && nb == 16 && s >= 1) prep_forward<true>(blk, pb, true, nb, kd, ldab, j, second, out);
        else prep_forward<false>(blk, pb, s >= 1, nb, kd, ldab, j, second, out);
      } else {
        // right-hand side (as a row): e_j, or N'_b(j, :) = L(c0 + 16 + j, c0 + k)
        const int rows = min(16, n - c0 - 16);
        if (kd >= 31 && nb == 16 && rows == 16) prep_backward<true>(blk, rows, nb, kd, ldab, j, second, out);
        else prep_backward<false>(blk, rows, nb, kd, ldab, j, second, out);
      }
      __syncwarp();
      stamp(s, 5);
      if (lane == 0) mbar_arrive(&pfull[p]);  // (H_b / G_b for the chain)
      // ---- t_b ----
      // u2 = the second-nearest block's term, which the far warps leave to this warp so the
      // far work has a step more of slack: forward N2_b y_{b-2}, N2_b = L_{b,b-2} (previous-
      // but-one buffer, offsets 32..47); backward N2'_b^T x_{b+2}, N2'_b = L_{b+2,b} (this
      // buffer, offsets 32..47).  Everything that does not depend on the awaited inputs
      // (indices, the operand rows) is loaded before the waits: only the products and the
      // staging round trip sit between the inputs and tdone.
      const int own = s % nbuf;
      const int q = s % kSweepNY;
      const double* rb = rbuf + (size_t)own * 16 * R;
      double* acc = ring + (size_t)((c0 + i) % nx) * R;
      double* tq = tbuf + q * 16 * R;
      double mr[16];  // row i of Linv_b (forward) / Linv_b^T (backward)
      {
        const double* m = slot + i * kLinvLd;
#pragma unroll
        for (int kk = 0; kk < 16; kk += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(m + kk);
          mr[kk] = t2.x;
          mr[kk + 1] = t2.y;
        }
      }
      double u2[RL];
#pragma unroll
      for (int rr = 0; rr < RL; ++rr) u2[rr] = 0.0;
      const bool has2 = fwd ? b >= 2 : b + 2 < nblk;
      if (has2) {
        double l[16];
        if (fwd) {
          const double* nb2 = Lbuf(s - 2) + 32 + i;  // L(c0+i, c0-32+c) = nb2[c * (ldab-1)]
          const bool rowin = i < nb;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const bool in = rowin && 32 + i - c <= kd;
            const double lv = nb2[in ? c * (ldab - 1) : 0];
            l[c] = in ? lv : 0.0;
          }
        } else {
          const double* nb2 = blk + i * (ldab - 1) + 32;  // L(c0+32+k, c0+i) = nb2[k]
          const int rows2 = min(16, n - c0 - 32);
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const bool in = k < rows2 && i < nb && 32 + k - i <= kd;
            const double lv = nb2[in ? k : 0];
            l[k] = in ? lv : 0.0;
          }
        }
        mbar_wait(&ydone[(s - 2) % kSweepNY], (unsigned)((s - 2) / kSweepNY) & 1u);
        const double* v2 = ych + ((s - 2) % kSweepNY) * 16 * R;
#pragma unroll
        for (int rr = 0; rr < RL; ++rr) {
          double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) a4[kk & 3] = fma(l[kk], v2[kk * R + stage_of(rr)], a4[kk & 3]);
          u2[rr] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        }
      }
      if (fwd) {
        // every far update of block b's rows (by y_{<= b-3}) landed
        if (b >= 3) mbar_wait(&fardone[(s - 3) % kSweepNY], (unsigned)((s - 3) / kSweepNY) & 1u);
        stamp(s, 6);
        if (store) {
#pragma unroll
          for (int rr = 0; rr < RL; ++rr) {
            const int r = stage_of(rr);
            cv[i * R + r] = (rb[i * R + r] + acc[r]) - u2[rr];
            acc[r] = 0.0;  // the slot's next row starts from zero
          }
        }
      } else {
        mbar_wait(&fardone[q], (unsigned)(s / kSweepNY) & 1u);
        stamp(s, 6);
        const double* fp = fpart + (size_t)((s & 3) * kFarParts * 16) * R;
        if (store) {
#pragma unroll
          for (int rr = 0; rr < RL; ++rr) {
            const int r = stage_of(rr);
            double f = 0.0;
#pragma unroll
            for (int w = 0; w < kFarParts; ++w) f += fp[(size_t)(w * 16 + i) * R + r];
            cv[i * R + r] = (rb[i * R + r] - f) - u2[rr];
          }
        }
      }
      __syncwarp();
      if constexpr (R >= 8) {
        // t = Linv_b cv (16 x R) on the tensor path
        const int gr = lane >> 2, gc = lane & 3;
        double acc[2][R / 8][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < R / 8; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        dmma_16x16xR<R>(slot, kLinvLd, cv, acc);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < R / 8; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) tq[(8 * mt + gr) * R + 8 * nt + 2 * gc + e] = acc[mt][nt][e];
      } else {
#pragma unroll
      for (int rr = 0; rr < RL; ++rr) {
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        if (R == 1) {
#pragma unroll
          for (int kk = 0; kk < 16; kk += 2) {
            const double2 c2 = *reinterpret_cast<const double2*>(cv + kk);
            a4[kk & 3] = fma(mr[kk], c2.x, a4[kk & 3]);
            a4[(kk + 1) & 3] = fma(mr[kk + 1], c2.y, a4[(kk + 1) & 3]);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) a4[kk & 3] = fma(mr[kk], cv[kk * R + rhs_of(rr)], a4[kk & 3]);
        }
        if (store) tq[i * R + rhs_of(rr)] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      }
      }
      __syncwarp();
      stamp(s, 7);
      if (lane == 0) {
        mbar_arrive(&tdone[q]);
        // buffer releases, 3 per step by prep: forward step s reads buffers s (L_bb, rb),
        // s-1 (N_b) and s-2 (N2_b); the last forward step stands in for the steps that do
        // not exist; a backward step reads only its own buffer
        if (fwd) {
          mbar_arrive(&empty[own]);
          if (s >= 1) mbar_arrive(&empty[(s - 1) % nbuf]);
          if (s >= 2) mbar_arrive(&empty[(s - 2) % nbuf]);
          if (s == nf - 1) {
            mbar_arrive(&empty[own]);
            mbar_arrive(&empty[own]);
            if (s >= 1) mbar_arrive(&empty[(s - 1) % nbuf]);
          }
        } else {
          mbar_arrive(&empty[own]);
          mbar_arrive(&empty[own]);
          mbar_arrive(&empty[own]);
        }
      }
    }
    return;
  }

  if (warp > kSweepPrepWarps) {
    // ------------------------------------ far -------------------------------------
    // R <= 2 (kScalar): thread-per-row / thread-per-(column, chunk) FMA loops -- forward: row
    // r always by thread r mod 96 (no race between steps); backward: 6 row chunks per column,
    // partials to fpart[s & 3][chunk].  R >= 4: the far work is a skinny GEMM on the FP64
    // tensor path (mma.sync m8n8k4 f64, SASS DMMA), where the right-hand sides fill the
    // n-dimension: A = the block's 16 columns of L below block b+1 (rows c0+48 .. c0+15+kd),
    // the right-hand sides the N = 8 columns of B (R <= 8; two n-tiles for R = 16), zeros
    // elsewhere.  Fragments: A lane (gr, gc) = A[gr][gc], B lane (gr, gc) = B[gc][gr], C lane
    // (gr, gc) = C[gr][2gc], C[gr][2gc+1].
    //   forward   acc[rows] -= L(rows, block b) y_b: 8-row m-tiles on absolute row indices,
    //             tile T owned by far warp T mod 3, row 8T+gr by lane gr: a row is always
    //             updated by the same thread, so successive steps never race (no barrier)
    //   backward  f_b = L(rows, block b)^T x: 4-row k-steps dealt round robin to the far
    //             warps, each warp's 16 x R partial to fpart[s & 3][warp]; prep adds the three
    //             partials in a fixed order
    // Each warp arrives on fardone and on the buffer's empty barrier when its part is done.
    const int fw = warp - (1 + kSweepPrepWarps);  // 0 .. kSweepFarWarps-1
    const int ft = threadIdx.x - 32 * (1 + kSweepPrepWarps);
    const int gr = lane >> 2, gc = lane & 3;
    constexpr int NT = R > 8 ? 2 : 1;  // n-tiles of 8 right-hand sides
    constexpr int kFarThreads = 32 * kSweepFarWarps, kFarChunks = kFarThreads / 16;
    RingPos kb;  // this step's L buffer and its full-phase parity (no divisions in the loop)
    for (int s = 0; s < nsteps; ++s, kb.next(nbuf)) {
      const int b = block_of(s), c0 = 16 * b;
      const double* blk = Lring + (size_t)kb.slot * 16 * ldab;
      if (s < nf) {
        mbar_wait(&ydone[s % kSweepNY], (unsigned)(s / kSweepNY) & 1u);
        mbar_wait(&full[kb.slot], kb.par);
        if (fw == 0 && lane == 0) stamp(s, 3);
        if constexpr (kScalar) {
        const double* y = ych + (s % kSweepNY) * 16 * R;
        const int lo = c0 + 48, hi = min(n - 1, c0 + 15 + kd);
        if (lo <= hi) {
          int r = lo + ((ft - lo) % kFarThreads + kFarThreads) % kFarThreads;
          int sl = r % nx;  // ring slot of row r, advanced without divisions
          for (; r <= hi; r += kFarThreads) {
            const int o = r - c0;  // row offset within the block's columns
            double l[16];          // the row's 16 entries first: one shared-memory latency
            if (o <= kd) {         // every column of the block reaches row r
#pragma unroll
              for (int c = 0; c < 16; ++c) l[c] = blk[c * ldab + o - c];
            } else {
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                const bool in = o - c <= kd;
                const double lv = blk[c * ldab + (in ? o - c : 0)];
                l[c] = in ? lv : 0.0;
              }
            }
            double* dst = ring + (size_t)sl * R;
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
              for (int c = 0; c < 16; ++c) a4[c & 3] = fma(l[c], y[c * R + rr], a4[c & 3]);
              dst[rr] -= (a4[0] + a4[1]) + (a4[2] + a4[3]);
            }
            sl += kFarThreads;
            while (sl >= nx) sl -= nx;
          }
        }
        } else {
        const double* y = ych + (s % kSweepNY) * 16 * R;
        const int lo = c0 + 48, hi = min(n - 1, c0 + 15 + kd);
        if (lo <= hi) {
          // B fragments (y_b, k = 4 ks + gc, n = gr) for the four k-steps
          double bf[4][NT];
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int rh = 8 * nt + gr;
              bf[ks][nt] = rh < R ? y[(4 * ks + gc) * R + (rh < R ? rh : 0)] : 0.0;
            }
          const int t_lo = lo >> 3, t_hi = hi >> 3;
          int t = t_lo + ((fw - t_lo) % kSweepFarWarps + kSweepFarWarps) % kSweepFarWarps;
          for (; t <= t_hi; t += kSweepFarWarps) {
            const int row = 8 * t + gr;                 // this lane's A row
            const bool rin = row >= lo && row <= hi;
            double acc[NT][2];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const int k = 4 * ks + gc, o = row - c0 - k;  // L(row, c0 + k)
              const bool in = rin && o <= kd;
              const double av = blk[k * ldab + (in ? o : 0)];
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) dmma884(acc[nt][0], acc[nt][1], in ? av : 0.0, bf[ks][nt]);
            }
            // C[gr][2gc + e] (row 8t + gr, rhs 8 nt + 2 gc + e) -> the accumulator ring
            const int crow = 8 * t + gr;
            if (crow >= lo && crow <= hi) {
              double* dst = ring + (size_t)(crow % nx) * R;
#pragma unroll
              for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const int rh = 8 * nt + 2 * gc + e;
                  if (rh < R) dst[rh] -= acc[nt][e];
                }
            }
          }
        }
        }
      } else {
        if (b + 3 <= nblk - 1) mbar_wait(&ydone[(s - 3) % kSweepNY], (unsigned)((s - 3) / kSweepNY) & 1u);
        mbar_wait(&full[kb.slot], kb.par);
        if (fw == 0 && lane == 0) stamp(s, 3);
        if constexpr (kScalar) {
        constexpr int Q = kFarChunks;
        // thread (column ft / 6, chunk ft % 6) takes rows c0+48+chunk, +6, ... (loads first,
        // four at a time); consecutive lanes read consecutive rows of one column (contiguous
        // shared-memory addresses); its partial goes to fpart[s & 3][chunk][column]
        const int c = ft / Q, qc = ft - (ft / Q) * Q;
        const int hi = c0 + c < n ? min(n - 1, c0 + c + kd) : c0;  // (no rows for columns past n)
        double acc[R][2];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[rr][0] = acc[rr][1] = 0.0;
        const double* colp = blk + c * ldab - (c0 + c);  // colp[row] = L(row, c0 + c)
        int r = c0 + 48 + qc;
        int sl = r % nx;
        for (; r + 3 * Q <= hi; r += 4 * Q) {
          double l4[4], x4[4][R];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            int su = sl + Q * u;
            su = su >= nx ? su - nx : su;
            l4[u] = colp[r + Q * u];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) x4[u][rr] = ring[(size_t)su * R + rr];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int rr = 0; rr < R; ++rr) acc[rr][u & 1] = fma(l4[u], x4[u][rr], acc[rr][u & 1]);
          sl += 4 * Q;
          sl = sl >= nx ? sl - nx : sl;
        }
        for (; r <= hi; r += Q) {
#pragma unroll
          for (int rr = 0; rr < R; ++rr) acc[rr][0] = fma(colp[r], ring[(size_t)sl * R + rr], acc[rr][0]);
          sl += Q;
          sl = sl >= nx ? sl - nx : sl;
        }
        double* fp = fpart + (size_t)(((s & 3) * kFarParts + qc) * 16 + c) * R;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) fp[rr] = acc[rr][0] + acc[rr][1];
        } else {
        const int lo = c0 + 48, hi = min(n - 1, c0 + 15 + kd);
        double acc[2][NT][2];  // m-tiles (columns 0-7, 8-15) x n-tiles
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        const int nks = hi >= lo ? (hi - lo + 4) >> 2 : 0;
        for (int ks = fw; ks < nks; ks += kSweepFarWarps) {
          const int row = lo + 4 * ks + gc;  // k index of this lane's A / B entries
          const bool rin = row <= hi;
          const double* xr = ring + (size_t)((rin ? row : lo) % nx) * R;
          double bv[NT];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int rh = 8 * nt + gr;
            const double xv = xr[rh < R ? rh : 0];
            bv[nt] = (rin && rh < R) ? xv : 0.0;
          }
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const int c = 8 * mt + gr, o = row - c0 - c;  // A[c][k] = L(row, c0 + c)
            const bool in = rin && o <= kd && c0 + c < n;
            const double av = blk[c * ldab + (in ? o : 0)];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], in ? av : 0.0, bv[nt]);
          }
        }
        // this warp's partial: column 8 mt + gr, rhs 8 nt + 2 gc + e
        double* fp = fpart + (size_t)(((s & 3) * kFarParts + fw) * 16) * R;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int rh = 8 * nt + 2 * gc + e;
              if (rh < R) fp[(8 * mt + gr) * R + rh] = acc[mt][nt][e];
            }
        }
      }
      __syncwarp();
      if (fw == 0 && lane == 0) stamp(s, 4);
      if (lane == 0) {
        mbar_arrive(&fardone[s % kSweepNY]);
        mbar_arrive(&empty[kb.slot]);
      }
    }
    return;
  }

  // ------------------------------------- chain ------------------------------------
  // lane (i = lane & 15, h = lane >> 4): row i of the block, right-hand sides h, h+2, ...
  // Per block: wait for the prep slot (H_b / G_b^T row i, loaded while t_b is awaited) and
  // for t_b, then out = t_b - M row i . (the previous block's output).
  RingPos pp, qq;              // prep slot and t / output slot of this step
  int xs = nf ? 0 : (16 * nblk) % nx;  // ring slot of row 16*b (backward: the solution ring)
  for (int s = 0; s < nsteps; ++s) {
    const bool fwd = s < nf;
    const int b = block_of(s), c0 = 16 * b, nb = min(16, n - c0);
    if (!fwd) xs = xs == 0 ? nx - 16 : xs - 16;
    stamp(s, 0);
    mbar_wait(&pfull[pp.slot], pp.par);
    double mr[16];  // row i of H_b (forward) / of G_b^T (backward)
    {
      const double* m = prep + pp.slot * kPrepSlot + 16 * kLinvLd + i * kLinvLd;
#pragma unroll
      for (int kk = 0; kk < 16; kk += 2) {
        const double2 t2 = *reinterpret_cast<const double2*>(m + kk);
        mr[kk] = t2.x;
        mr[kk + 1] = t2.y;
      }
    }
    const bool has_prev = fwd ? b >= 1 : b + 1 < nblk;
    const double* prevo = ych + ((s - 1) & (kSweepNY - 1)) * 16 * R;
    if constexpr (R >= 8) {
      // right-hand sides fill the n-dimension of a DMMA product: C = M . (previous output),
      // then out = t_b - C; lane (gr, gc) owns rows gr, 8+gr and right-hand sides 2gc, 2gc+1
      // (+8 for R = 16)
      constexpr int NT = R / 8;
      const int gr = lane >> 2, gc = lane & 3;
      double acc[2][NT][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
      if (has_prev) dmma_16x16xR<R>(prep + pp.slot * kPrepSlot + 16 * kLinvLd, kLinvLd, prevo, acc);
      mbar_wait(&tdone[qq.slot], qq.par);
      stamp(s, 1);
      const double* tq = tbuf + qq.slot * 16 * R;
      double* yo = ych + qq.slot * 16 * R;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = 8 * mt + gr, rh = 8 * nt + 2 * gc + e;
            const double o = row < nb ? tq[row * R + rh] - acc[mt][nt][e] : 0.0;
            acc[mt][nt][e] = o;
            yo[row * R + rh] = o;
            if (!fwd) ring[(size_t)(xs + row) * R + rh] = o;  // for the far dot products
          }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&ydone[qq.slot]);
        mbar_arrive(&pempty[pp.slot]);
      }
      double* brow = bm + c0;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = 8 * mt + gr, rh = 8 * nt + 2 * gc + e;
            if (row < nb && rh < rv) brow[(int64_t)rh * ldb + row] = acc[mt][nt][e];
          }
    } else {
    // the product with the previous block's output needs nothing of this step but M: it runs
      // before t_b is awaited, so only t_b - dot is left on the serial path
      double dot[RL];
  #pragma unroll
      for (int rr = 0; rr < RL; ++rr) {
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        if (has_prev) {
          if (R == 1) {
  #pragma unroll
            for (int kk = 0; kk < 16; kk += 2) {
              const double2 p2 = *reinterpret_cast<const double2*>(prevo + kk);
              a4[kk & 3] = fma(mr[kk], p2.x, a4[kk & 3]);
              a4[(kk + 1) & 3] = fma(mr[kk + 1], p2.y, a4[(kk + 1) & 3]);
            }
          } else {
  #pragma unroll
            for (int kk = 0; kk < 16; ++kk) a4[kk & 3] = fma(mr[kk], prevo[kk * R + rhs_of(rr)], a4[kk & 3]);
          }
        }
        dot[rr] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      }
      mbar_wait(&tdone[qq.slot], qq.par);
      stamp(s, 1);
      const double* tq = tbuf + qq.slot * 16 * R;
      double o[RL];
  #pragma unroll
      for (int rr = 0; rr < RL; ++rr) o[rr] = i < nb ? tq[i * R + rhs_of(rr)] - dot[rr] : 0.0;
      double* yo = ych + qq.slot * 16 * R;
      if (store) {
  #pragma unroll
        for (int rr = 0; rr < RL; ++rr) {
          yo[i * R + rhs_of(rr)] = o[rr];
          if (!fwd) ring[(size_t)(xs + i) * R + rhs_of(rr)] = o[rr];  // for the far dot products
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&ydone[qq.slot]);
        mbar_arrive(&pempty[pp.slot]);
      }
      if (store) {  // to global memory after the signals (nothing in this CTA waits on it soon)
        double* brow = bm + c0;
  #pragma unroll
        for (int rr = 0; rr < RL; ++rr)
          if (i < nb && rhs_of(rr) < rv) brow[(int64_t)rhs_of(rr) * ldb + i] = o[rr];
      }
    }
    stamp(s, 2);
    if (s == nf - 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&fwd_done);  // release: the y stores above -> the producer's loads
    }
    pp.next(kSweepNP);
    qq.next(kSweepNY);
    if (fwd) {
      xs += 16;
      if (xs == nx) xs = 0;
    }
  }
  if (threadIdx.x == 0 && grp == 0) info[mat] = 0;
}

}  // namespace bcg
