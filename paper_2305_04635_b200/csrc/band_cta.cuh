// band_cta.cuh -- one thread block factors (and optionally solves) one band matrix.
//
// Right-looking blocked band Cholesky (the reference's sliding window of
// blocked.py:1-7, :297-315, re-derived for one CTA): step k owns columns
// [j0, j0+nb), j0 = k*NB.
//   1. POTRF of the nb x nb diagonal block      (blocked.py:259-269 factor_diag)
//   2. TRSM of the m x nb panel below it, m = min(kd, n-j0-nb); the out-of-band
//      triangle (blocked.py:136-167 WorkArray) is treated as exact zeros in
//      registers instead of being staged       (blocked.py:271-276 solve_panel)
//   3. SYRK/GEMM of the m x m trailing triangle with the panel
//                                               (blocked.py:278-284 update_*)
// The active window (kd+NB columns of kd+1 entries) lives in shared memory as a
// ring of column slots; each column is loaded from HBM once (cp.async, one step
// ahead of its first use) and written back once, right after its panel step.
// When the window does not fit in shared memory the same code runs in place on
// the band in global memory (kWinSmem = false).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bcg {

constexpr int kCtaThreads = 256;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

struct CtaGeom {
  int n, kd, ldab;   // matrix geometry
  int lds, nslot;    // shared window: nslot column slots of lds doubles (kWinSmem)
  int pld;           // leading dimension of the dense panel buffer P (>= kd rounded to 4)
};

// Shared-memory footprint (bytes) of one CTA for block size NB.
// With the window in global memory the panel buffer P lives in global scratch too.
__host__ __device__ inline size_t cta_smem_bytes(int nb_block, const CtaGeom& g, bool win_smem, bool solve) {
  size_t d = (size_t)nb_block * nb_block + nb_block;
  if (win_smem) d += (size_t)g.nslot * g.lds + (size_t)nb_block * g.pld;
  if (solve) d += (size_t)g.nslot;  // ring of right-hand-side entries
  return d * sizeof(double) + 16;
}

template <int NB, bool kWinSmem, bool kSolve>
struct CtaBand {
  const CtaGeom g;
  double* __restrict__ ab;  // this matrix in global memory
  double* __restrict__ rhs; // this matrix's right-hand side (kSolve)
  double* win;              // shared ring (kWinSmem)
  double* P;                // NB x pld dense panel, P[c*pld + r] = L(j0+nb+r, j0+c)
  double* D;                // NB x NB dense L11, row-major
  double* Dinv;             // NB reciprocals of diag(L11)
  double* bw;               // ring of rhs entries, bw[i % nslot] (kSolve)

  __device__ __forceinline__ double* colp(int j) const {
    if (kWinSmem) return win + (j % g.nslot) * g.lds;
    return ab + (int64_t)j * g.ldab;
  }
  __device__ __forceinline__ int col_len(int j) const {  // in-band entries of column j
    return min(g.kd, g.n - 1 - j) + 1;
  }

  // cp.async columns [jlo, jhi) (and their rhs entries) into the ring.
  __device__ void load_cols(int jlo, int jhi) {
    if (!kWinSmem && !kSolve) return;
    const int tid = threadIdx.x;
    const int per = g.kd + 1;
    if (kWinSmem) {
      const int total = (jhi - jlo) * per;
      for (int idx = tid; idx < total; idx += kCtaThreads) {
        const int c = idx / per, o = idx - c * per;
        const int j = jlo + c;
        if (o < col_len(j)) cp_async8(colp(j) + o, ab + (int64_t)j * g.ldab + o);
      }
    }
    if (kSolve) {
      for (int j = jlo + tid; j < jhi; j += kCtaThreads) cp_async8(bw + (j % g.nslot), rhs + j);
    }
    cp_async_commit();
  }

  // Panel columns [j0, j0+nb) back to HBM (final L).
  __device__ void store_cols(int j0, int nb) {
    if (!kWinSmem) return;
    const int per = g.kd + 1;
    const int total = nb * per;
    for (int idx = threadIdx.x; idx < total; idx += kCtaThreads) {
      const int c = idx / per, o = idx - c * per;
      const int j = j0 + c;
      if (o < col_len(j)) ab[(int64_t)j * g.ldab + o] = colp(j)[o];
    }
  }

  // Warp 0: Cholesky of the nb x nb diagonal block.  Lane r holds row r.
  // Returns the local failing column or -1 (uniform across the warp).
  __device__ int potrf_diag(int j0, int nb) {
    const int r = threadIdx.x & 31;
    double row[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) row[c] = (r < nb && c <= r && r - c <= g.kd) ? colp(j0 + c)[r - c] : 0.0;
    double myinv = 0.0;
    int fail = -1;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < nb) {
        const double dcc = __shfl_sync(kFull, row[c], c);
        if (!(dcc > 0.0)) { fail = c; break; }
        const double d = sqrt(dcc);
        const double inv = 1.0 / d;
        if (r == c) { row[c] = d; myinv = inv; }
        else if (r > c) row[c] *= inv;
#pragma unroll
        for (int c2 = c + 1; c2 < NB; ++c2) {
          const double l2 = __shfl_sync(kFull, row[c], c2);
          if (r >= c2) row[c2] = fma(-row[c], l2, row[c2]);
        }
      }
    }
    if (fail < 0) {
      if (r < nb) {
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c <= r && r - c <= g.kd) colp(j0 + c)[r - c] = row[c];
      }
      if (r < NB) {
#pragma unroll
        for (int c = 0; c < NB; ++c) D[r * NB + c] = (r < nb && c <= r) ? row[c] : 0.0;
        Dinv[r] = r < nb ? myinv : 0.0;
      }
    }
    return fail;
  }

  // Forward sweep for the panel rows: solve L11 y = bw[j0..j0+nb) (warp 0 after
  // potrf_diag; reads D/Dinv it just wrote, so only needs __syncwarp).
  __device__ void forward_diag(int j0, int nb) {
    const int r = threadIdx.x & 31;
    double s = (r < nb) ? bw[(j0 + r) % g.nslot] : 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < nb) {
        const double yc = __shfl_sync(kFull, s, c) * Dinv[c];
        if (r == c) s = yc;
        else if (r > c && r < nb) s = fma(-D[r * NB + c], yc, s);
      }
    }
    if (r < nb) {
      bw[(j0 + r) % g.nslot] = s;
      rhs[j0 + r] = s;
    }
  }

  // Panel TRSM: row r of P solves x L11^T = a_r.  Threads [first_thread, ...).
  __device__ void trsm_panel(int j0, int nb, int m, int first_thread) {
    for (int r = (int)threadIdx.x - first_thread; r < m; r += kCtaThreads - first_thread) {
      if (r < 0) break;
      double x[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const int off = nb + r - c;
        x[c] = (c < nb && off <= g.kd) ? colp(j0 + c)[off] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        x[c] *= Dinv[c];
#pragma unroll
        for (int c2 = c + 1; c2 < NB; ++c2) x[c2] = fma(-x[c], D[c2 * NB + c], x[c2]);
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const int off = nb + r - c;
        if (c < nb && off <= g.kd) colp(j0 + c)[off] = x[c];
        P[c * g.pld + r] = x[c];
      }
    }
  }

  // Trailing update: lower triangle of the m x m window -= P P^T, 4x4 register tiles;
  // plus the forward-sweep update of the trailing rhs entries.
  __device__ void update_trailing(int j0, int nb, int m) {
    const int base = j0 + nb;
    const int T = (m + 3) >> 2;
    const int ntile = T * (T + 1) / 2;
    for (int t = threadIdx.x; t < ntile; t += kCtaThreads) {
      int ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
      while (ti * (ti + 1) / 2 > t) --ti;
      while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
      const int tj = t - ti * (ti + 1) / 2;
      const int i0 = ti * 4, q0 = tj * 4;
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
#pragma unroll 4
      for (int c = 0; c < nb; ++c) {
        const double* pc = P + c * g.pld;
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { a[u] = pc[i0 + u]; b[u] = pc[q0 + u]; }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int q = q0 + v;
        if (q >= m) continue;
        double* cp = colp(base + q);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u;
          if (i < m && i >= q) cp[i - q] -= acc[u][v];
        }
      }
    }
    if (kSolve) {
      for (int i = threadIdx.x; i < m; i += kCtaThreads) {
        double s = 0.0;
        for (int c = 0; c < nb; ++c) s = fma(P[c * g.pld + i], bw[(j0 + c) % g.nslot], s);
        bw[(base + i) % g.nslot] -= s;
      }
    }
  }

  // Whole factorization (+ forward sweep when kSolve).  Returns -1 or failing column.
  __device__ int factor() {
    const int n = g.n, kd = g.kd;
    __shared__ int s_fail;
    load_cols(0, min(n, kd + NB));
    cp_async_wait_all();
    __syncthreads();
    for (int j0 = 0; j0 < n; j0 += NB) {
      const int nb = min(NB, n - j0);
      const int m = min(kd, n - j0 - nb);
      if (kd < NB) {  // the previous step's prefetch overlaps this panel
        cp_async_wait_all();
        __syncthreads();
      }
      if (threadIdx.x < 32) {
        const int f = potrf_diag(j0, nb);
        if (threadIdx.x == 0) s_fail = f;
        __syncwarp();
        if (kSolve && f < 0) forward_diag(j0, nb);
      }
      __syncthreads();
      if (s_fail >= 0) {
        const int col = j0 + s_fail;
        cp_async_wait_all();
        __syncthreads();
        return col;
      }
      trsm_panel(j0, nb, m, kSolve ? 32 : 0);
      cp_async_wait_all();
      __syncthreads();
      store_cols(j0, nb);
      update_trailing(j0, nb, m);
      __syncthreads();
      const int jlo = j0 + NB + kd;
      if (jlo < n) load_cols(jlo, min(n, jlo + NB));
    }
    cp_async_wait_all();
    __syncthreads();
    return -1;
  }

  // Backward sweep L^T x = y (y in rhs from the fused forward sweep), reading L
  // columns from global memory; the ring `win` is reused as a prefetch buffer
  // when it lives in shared memory.
  __device__ void backward() {
    const int n = g.n, kd = g.kd;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kWarps = kCtaThreads / 32;
    // bw ring now holds x entries, indexed by row % nslot.
    const int last0 = ((n - 1) / NB) * NB;
    for (int c0 = last0; c0 >= 0; c0 -= NB) {
      const int nb = min(NB, n - c0);
      // s_j = y_j - sum_{i >= c0+nb, i <= j+kd} L(i,j) x_i for the nb columns
      for (int c = warp; c < nb; c += kWarps) {
        const int j = c0 + c;
        const double* colj = ab + (int64_t)j * g.ldab;
        const int len = col_len(j);  // offsets 0..len-1
        double s = 0.0;
        for (int o = nb - c + lane; o < len; o += 32) s = fma(colj[o], bw[(j + o) % g.nslot], s);
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) s += __shfl_xor_sync(kFull, s, sh);
        if (lane == 0) P[c] = rhs[j] - s;
        // diagonal block column j, rows c0..c0+nb-1 for the triangular solve
        if (lane < NB) D[lane * NB + c] = (lane >= c && lane < nb && lane - c < len) ? colj[lane - c] : 0.0;
      }
      __syncthreads();
      if (warp == 0) {
        // upper-triangular solve L11^T x = s, lane r holds s_r
        double s = lane < nb ? P[lane] : 0.0;
        const double dinv = lane < nb ? 1.0 / D[lane * NB + lane] : 0.0;
#pragma unroll
        for (int c = NB - 1; c >= 0; --c) {
          if (c < nb) {
            const double xc = __shfl_sync(kFull, s * dinv, c);
            if (lane == c) s = xc;
            else if (lane < c) s = fma(-D[c * NB + lane], xc, s);
          }
        }
        if (lane < nb) {
          bw[(c0 + lane) % g.nslot] = s;
          rhs[c0 + lane] = s;
        }
      }
      __syncthreads();
    }
  }
};

}  // namespace bcg
