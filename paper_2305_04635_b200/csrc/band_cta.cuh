// band_cta.cuh -- one thread block factors (and optionally solves) one band matrix.
//
// Right-looking blocked band Cholesky (the reference's sliding window of
// blocked.py:1-7, :297-315, re-derived for one CTA).  Step k owns columns
// [j0, j0+nb), j0 = k*NB:
//   1. POTRF of the nb x nb diagonal block        (blocked.py:259-269 factor_diag)
//   2. TRSM of the m x nb panel below it, m = min(kd, n-j0-nb); the out-of-band
//      triangle (blocked.py:136-167 WorkArray) is exact zeros in registers
//                                                  (blocked.py:271-276 solve_panel)
//   3. SYRK/GEMM of the m x m trailing triangle    (blocked.py:278-284 update_*)
//
// B200 mapping:
//   * The active window (kd+NB columns x (kd+1) entries) lives in shared memory as
//     a ring of column slots; every column is loaded from HBM once (cp.async, a
//     step ahead of first use) and written back once, right after its panel step.
//   * POTRF runs in warp 0 with the pivot chain computed REDUNDANTLY in every
//     lane (p_{c+1} = A'(c+1,c+1) - (A'(c+1,c) rsqrt(p_c))^2 from two values
//     broadcast one step ahead), so one column costs rsqrt + mul + fma on the
//     critical path instead of rsqrt + shuffle + mul + fma.  The forward sweep of
//     the solve rides along in the same loop.
//   * Lookahead: the update of step k is split; the part that touches the next
//     panel's columns runs first, then warp 0 factors the next diagonal block
//     while warps 1-7 finish the rest of step k's update.
//   * The trailing update runs on the FP64 tensor path (mma.sync m8n8k4 f64 ->
//     DMMA), 16x16 warp tiles, operands from a dense panel copy P whose leading
//     dimension is 4 (mod 16) doubles (conflict-free fragment loads).
//   * Backward sweep (fused solve): L is streamed back through the same ring with a
//     cp.async pipeline several blocks deep.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bcg {

constexpr int kCtaThreads = 256;
constexpr int kCtaWarps = kCtaThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct CtaGeom {
  int n, kd, ldab;  // matrix geometry
  int lds, nslot;   // shared window: nslot column slots of lds doubles
  int pld;          // leading dimension of the dense panel P (>= kd rounded up to 16, = 4 mod 16)
};

// Shared-memory footprint (bytes) of one CTA for block size NB.
__host__ __device__ inline size_t cta_smem_bytes(int nb_block, const CtaGeom& g, bool solve) {
  size_t d = (size_t)g.nslot * g.lds + (size_t)nb_block * g.pld + (size_t)nb_block * nb_block + nb_block + 32;
  if (solve) d += (size_t)g.nslot;  // ring of right-hand-side entries
  return d * sizeof(double) + 64;
}

template <int NB, bool kSolve>
struct CtaBand {
  static_assert(NB == 16 || NB == 32, "block size");
  const CtaGeom g;
  double* __restrict__ ab;   // this matrix in global memory
  double* __restrict__ rhs;  // its right-hand side (kSolve)
  double* win;               // shared ring of column slots
  double* P;                 // NB x pld dense panel, P[c*pld + r] = L(j0+nb+r, j0+c)
  double* D;                 // NB x NB dense L11, row-major
  double* Dinv;              // NB reciprocals of diag(L11)
  double* lbuf;              // 32 doubles: column broadcast inside the POTRF warp
  double* bw;                // ring of rhs / solution entries, slot(i) like columns

  // ---- ring addressing: slot(j) = j mod nslot without a division on hot paths ----
  __device__ __forceinline__ int slot_from(int s0, int j0, int j) const {
    int s = s0 + (j - j0);
    return s >= g.nslot ? s - g.nslot : s;  // valid for j0 <= j < j0 + nslot
  }
  __device__ __forceinline__ int col_len(int j) const { return min(g.kd, g.n - 1 - j) + 1; }

  // cp.async columns [jlo, jhi) (and their rhs entries) into the ring.
  __device__ void load_cols(int jlo, int jhi) {
    const int per = g.kd + 1;
    const int total = (jhi - jlo) * per;
    for (int idx = threadIdx.x; idx < total; idx += kCtaThreads) {
      const int c = idx / per, o = idx - c * per;
      const int j = jlo + c;
      if (o < col_len(j)) cp_async8(win + (j % g.nslot) * g.lds + o, ab + (int64_t)j * g.ldab + o);
    }
    if (kSolve)
      for (int j = jlo + threadIdx.x; j < jhi; j += kCtaThreads) cp_async8(bw + (j % g.nslot), rhs + j);
    cp_async_commit();
  }

  // Panel columns [j0, j0+nb) back to HBM (final L).
  __device__ void store_cols(int s0, int j0, int nb) {
    const int per = g.kd + 1;
    const int total = nb * per;
    for (int idx = threadIdx.x; idx < total; idx += kCtaThreads) {
      const int c = idx / per, o = idx - c * per;
      const int j = j0 + c;
      if (o < col_len(j)) ab[(int64_t)j * g.ldab + o] = win[slot_from(s0, j0, j) * g.lds + o];
    }
  }

  // Warp 0: Cholesky of the nb x nb diagonal block at column j0 (+ forward sweep).
  // Lane r holds row r.  Returns the local failing column or -1 (uniform).
  __device__ int potrf_diag(int s0, int j0, int nb) {
    const int r = threadIdx.x & 31;
    double row[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c)
      row[c] = (r < nb && c <= r && r - c <= g.kd) ? win[slot_from(s0, j0, j0 + c) * g.lds + (r - c)] : 0.0;
    double s = 0.0;
    if (kSolve && r < nb) s = bw[slot_from(s0, j0, j0 + r)];
    // chain state, identical in every lane
    double p = __shfl_sync(kFull, row[0], 0);
    double alpha = __shfl_sync(kFull, row[0], 1);  // A'(1,0)
    double beta = __shfl_sync(kFull, row[1], 1);   // A'(1,1)
    double myinv = 0.0;
    int fail = -1;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < nb) {
        if (!(p > 0.0)) { fail = c; break; }
        const double rs = rsqrt(p);
        const double lrc = row[c] * rs;     // L(r, c) for r > c
        const double l1 = alpha * rs;       // L(c+1, c), known to every lane
        const double pn = fma(-l1, l1, beta);
        if (r == c) { row[c] = p * rs; myinv = rs; }
        else if (r > c) row[c] = lrc;
        if (kSolve) {
          const double yc = __shfl_sync(kFull, s, c) * rs;
          if (r == c) s = yc;
          else if (r > c) s = fma(-lrc, yc, s);
        }
        lbuf[r] = (r > c) ? lrc : 0.0;
        __syncwarp();
        if (r > c) {
#pragma unroll
          for (int c2 = c + 1; c2 < NB; ++c2) {
            const double lc2 = (c2 == c + 1) ? l1 : ((c2 == r) ? lrc : lbuf[c2]);
            if (r >= c2) row[c2] = fma(-lrc, lc2, row[c2]);
          }
        }
        __syncwarp();
        if (c + 2 < NB) {
          alpha = __shfl_sync(kFull, row[c + 1 < NB ? c + 1 : 0], c + 2);
          beta = __shfl_sync(kFull, row[c + 2 < NB ? c + 2 : 0], c + 2);
        }
        p = pn;
      }
    }
    if (fail < 0) {
      if (r < nb) {
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c <= r && r - c <= g.kd) win[slot_from(s0, j0, j0 + c) * g.lds + (r - c)] = row[c];
        if (kSolve) {
          bw[slot_from(s0, j0, j0 + r)] = s;
          rhs[j0 + r] = s;
        }
      }
      if (r < NB) {
#pragma unroll
        for (int c = 0; c < NB; ++c) D[r * NB + c] = (r < nb && c <= r) ? row[c] : 0.0;
        Dinv[r] = r < nb ? myinv : 0.0;
      }
    }
    return fail;
  }

  // Panel TRSM: row r of P solves x L11^T = a_r (all threads).
  __device__ void trsm_panel(int s0, int j0, int nb, int m) {
    for (int r = threadIdx.x; r < m; r += kCtaThreads) {
      double x[NB];
      int sl[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const int off = nb + r - c;
        sl[c] = slot_from(s0, j0, j0 + (c < nb ? c : 0)) * g.lds + off;
        x[c] = (c < nb && off <= g.kd) ? win[sl[c]] : 0.0;
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
        if (c < nb && off <= g.kd) win[sl[c]] = x[c];
        P[c * g.pld + r] = x[c];
      }
    }
  }

  // Trailing update of 16x16 tiles (ti >= tj) with tile column tj in [tj_lo, tj_hi),
  // by warps [w_lo, kCtaWarps).  C(i,j) -= sum_c P(i,c) P(j,c), i,j < m, lower only.
  __device__ void update_tiles(int s0, int j0, int nb, int m, int tj_lo, int tj_hi, int w_lo) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < w_lo) return;
    const int gr = lane >> 2, gc = lane & 3;
    const int base = j0 + nb;
    const int T = (m + 15) >> 4;
    tj_hi = min(tj_hi, T);
    if (tj_lo >= tj_hi) return;
    // tiles of columns [tj_lo, tj_hi): column tj holds T - tj tiles
    const int first = tj_lo * T - tj_lo * (tj_lo - 1) / 2;
    const int last = tj_hi * T - tj_hi * (tj_hi - 1) / 2;
    const int nw = kCtaWarps - w_lo;
    for (int t = first + (warp - w_lo); t < last; t += nw) {
      int tj = tj_lo;
      while (tj + 1 < tj_hi && (tj + 1) * T - (tj + 1) * tj / 2 <= t) ++tj;
      const int ti = tj + (t - (tj * T - tj * (tj - 1) / 2));
      const int i0 = ti * 16, q0 = tj * 16;
      double acc[2][2][2];
      int ofs[2][2][2];
      bool ok[2][2][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = i0 + u * 8 + gr, q = q0 + v * 8 + 2 * gc + e;
            ok[u][v][e] = (i < m) && (q <= i);
            ofs[u][v][e] = slot_from(s0, j0, base + (q < m ? q : 0)) * g.lds + (i - q);
            acc[u][v][e] = ok[u][v][e] ? win[ofs[u][v][e]] : 0.0;
          }
#pragma unroll
      for (int k0 = 0; k0 < NB; k0 += 4) {
        const double* pk = P + (k0 + gc) * g.pld;
        double a[2], b[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) a[u] = -pk[i0 + u * 8 + gr];
#pragma unroll
        for (int v = 0; v < 2; ++v) b[v] = pk[q0 + v * 8 + gr];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) dmma884(acc[u][v][0], acc[u][v][1], a[u], b[v]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (ok[u][v][e]) win[ofs[u][v][e]] = acc[u][v][e];
    }
  }

  // Forward-sweep update of the trailing rhs entries: b_i -= sum_c P(i,c) y_c.
  __device__ void update_rhs(int s0, int j0, int nb, int m) {
    const int base = j0 + nb;
    for (int i = threadIdx.x; i < m; i += kCtaThreads) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c < nb) s = fma(P[c * g.pld + i], bw[slot_from(s0, j0, j0 + c)], s);
      bw[slot_from(s0, j0, base + i)] -= s;
    }
  }

  // Whole factorization (+ forward sweep when kSolve).  Returns -1 or failing column.
  __device__ int factor() {
    const int n = g.n, kd = g.kd;
    __shared__ int s_fail;
    const int warp = threadIdx.x >> 5;
    // zero the panel buffer once (rows past m are read, never used, by the tile GEMM)
    for (int idx = threadIdx.x; idx < NB * g.pld; idx += kCtaThreads) P[idx] = 0.0;
    load_cols(0, min(n, kd + NB));
    cp_async_wait_all();
    __syncthreads();
    if (warp == 0) {
      const int f = potrf_diag(0, 0, min(NB, n));
      if (threadIdx.x == 0) s_fail = f;
    }
    __syncthreads();
    if (s_fail >= 0) return s_fail;
    int j0 = 0, s0 = 0;
    for (;;) {
      const int nb = min(NB, n - j0);
      const int m = min(kd, n - j0 - nb);
      trsm_panel(s0, j0, nb, m);
      cp_async_wait_all();  // columns prefetched by the previous step
      __syncthreads();
      store_cols(s0, j0, nb);
      // part 1: tile columns touching the next panel, then the rhs
      update_tiles(s0, j0, nb, m, 0, NB / 16, 0);
      if (kSolve) update_rhs(s0, j0, nb, m);
      __syncthreads();
      const int jlo = j0 + NB + kd;
      if (jlo < n) load_cols(jlo, min(n, jlo + NB));
      const int j1 = j0 + nb;
      if (j1 >= n) break;
      int s1 = s0 + nb;
      if (s1 >= g.nslot) s1 -= g.nslot;
      if (kd < NB) {  // the prefetch just issued overlaps the next panel
        cp_async_wait_all();
        __syncthreads();
      }
      // warp 0: next diagonal block; warps 1..7: rest of this step's update
      if (warp == 0) {
        const int f = potrf_diag(s1, j1, min(NB, n - j1));
        if (threadIdx.x == 0) s_fail = f;
      } else {
        update_tiles(s0, j0, nb, m, NB / 16, 1 << 20, 1);
      }
      __syncthreads();
      if (s_fail >= 0) {
        cp_async_wait_all();
        __syncthreads();
        return j1 + s_fail;
      }
      j0 = j1;
      s0 = s1;
    }
    cp_async_wait_all();
    __syncthreads();
    return -1;
  }

  // Backward sweep L^T x = y (y in rhs / bw after the fused forward sweep).  The L
  // columns stream back from global memory into the (now free) ring in blocks of NB,
  // kDepth blocks in flight.
  __device__ void backward() {
    const int n = g.n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kDepth = 4;
    const int nbuf = g.nslot / NB;  // >= kDepth + 1 (host guarantees nslot >= (kDepth+1)*NB)
    const int nblk = (n + NB - 1) / NB;
    auto buf_of = [&](int b) -> double* { return win + (size_t)(b % nbuf) * NB * g.lds; };
    auto issue = [&](int b) {
      if (b >= 0) {
        const int c0 = b * NB;
        const int cols = min(NB, n - c0);
        const int per = g.kd + 1;
        double* dst = buf_of(b);
        for (int idx = threadIdx.x; idx < cols * per; idx += kCtaThreads) {
          const int c = idx / per, o = idx - c * per;
          if (o < col_len(c0 + c)) cp_async8(dst + c * g.lds + o, ab + (int64_t)(c0 + c) * g.ldab + o);
        }
      }
      cp_async_commit();  // always commit (possibly empty) so group counting stays uniform
    };
    for (int d = 0; d < kDepth; ++d) issue(nblk - 1 - d);
    for (int b = nblk - 1; b >= 0; --b) {
      cp_async_wait_group<kDepth - 1>();
      __syncthreads();
      const int c0 = b * NB;
      const int nb = min(NB, n - c0);
      const double* blk = buf_of(b);
      const int sx = (c0 + nb) % g.nslot;  // slot of row c0+nb in the x ring
      for (int c = warp; c < nb; c += kCtaWarps) {
        const int j = c0 + c;
        const int len = col_len(j);
        const double* colj = blk + c * g.lds;
        double s = 0.0;
        for (int o = nb - c + lane; o < len; o += 32) {
          int sl = sx + (j + o - (c0 + nb));
          if (sl >= g.nslot) sl -= g.nslot;
          s = fma(colj[o], bw[sl], s);
        }
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) s += __shfl_xor_sync(kFull, s, sh);
        if (lane == 0) Dinv[c] = rhs[j] - s;  // Dinv reused as the block's right-hand side
      }
      __syncthreads();
      if (warp == 0) {
        double v = lane < nb ? Dinv[lane] : 0.0;
        const double dinv = lane < nb ? 1.0 / blk[lane * g.lds] : 0.0;
#pragma unroll
        for (int c = NB - 1; c >= 0; --c) {
          if (c < nb) {
            const double xc = __shfl_sync(kFull, v * dinv, c);
            if (lane == c) v = xc;
            else if (lane < c && lane < nb) v = fma(-blk[lane * g.lds + (c - lane)], xc, v);
          }
        }
        if (lane < nb) {
          bw[(c0 + lane) % g.nslot] = v;
          rhs[c0 + lane] = v;
        }
      }
      __syncthreads();
      issue(b - kDepth);
    }
    cp_async_wait_all();
    __syncthreads();
  }
};

}  // namespace bcg
