// band_solve.cuh -- standalone band solve L L^T x = b (reference solve_with_factor,
// pkg/src/bandchol/core.py:216-240), one thread block per right-hand side.
//
// Forward sweep, blocks of NB=32 rows:  y_i = (b_i - sum_l L(i,l) y_l) / L(i,i).
//   The bulk of each row's dot product (columns left of the block) is spread
//   over the 8 warps with lanes on consecutive rows, so every load instruction
//   reads one contiguous 256-byte run of the band (the skewed view
//   A(i,l) = ab[l*(ldab-1) + i], blocked.py:122); warp 0 then solves the 32x32
//   diagonal block with shuffles.
// Backward sweep over columns: x_j = (y_j - sum_r L(r,j) x_r) / L(j,j); a
//   column of L is contiguous, so each warp reduces whole columns.
// The diagonal is checked first, exactly like core.py:227-230: if any
// diagonal entry is <= 0 nothing is written and info = first bad column + 1.
#pragma once
#include "band_cta.cuh"

namespace bcg {

constexpr int kSolveNB = 32;

__device__ int first_nonpositive_diag(const double* __restrict__ ab, int n, int ldab) {
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = INT_MAX;
  __syncthreads();
  int mine = INT_MAX;
  // no early exit: the loads of a thread are independent and overlap (one latency, not n/T)
#pragma unroll 8
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    if (ab[(int64_t)j * ldab] <= 0.0 && mine == INT_MAX) mine = j;
  if (mine != INT_MAX) atomicMin(&s_bad, mine);
  __syncthreads();
  const int r = s_bad;
  __syncthreads();
  return r;
}

__device__ void band_forward(const double* __restrict__ ab, int n, int kd, int ldab, double* b) {
  constexpr int NB = kSolveNB;
  __shared__ double red[kCtaThreads / 32][NB];
  const int lane = threadIdx.x & 31, warp = warp_uniform(threadIdx.x >> 5);
  for (int r0 = 0; r0 < n; r0 += NB) {
    const int nb = min(NB, n - r0);
    const int i = r0 + lane;
    double s = 0.0;
    const int lbeg = max(0, r0 - kd);
    if (lane < nb) {
      // four independent chains so the L2/HBM loads of a row overlap
      constexpr int W = kCtaThreads / 32;
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int l = max(lbeg, i - kd) + warp;  // columns in band for row i
      for (; l + 3 * W < r0; l += 4 * W) {
        const double a0 = ab[(int64_t)l * ldab + (i - l)], a1 = ab[(int64_t)(l + W) * ldab + (i - l - W)];
        const double a2 = ab[(int64_t)(l + 2 * W) * ldab + (i - l - 2 * W)];
        const double a3 = ab[(int64_t)(l + 3 * W) * ldab + (i - l - 3 * W)];
        s = fma(a0, b[l], s);
        s1 = fma(a1, b[l + W], s1);
        s2 = fma(a2, b[l + 2 * W], s2);
        s3 = fma(a3, b[l + 3 * W], s3);
      }
      for (; l < r0; l += W) s = fma(ab[(int64_t)l * ldab + (i - l)], b[l], s);
      s += (s1 + s2) + s3;
    }
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kCtaThreads / 32; ++w) t += red[w][lane];
      double row[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c)
        row[c] = (lane < nb && c <= lane && lane - c <= kd) ? ab[(int64_t)(r0 + c) * ldab + (lane - c)] : 0.0;
      double v = lane < nb ? b[i] - t : 0.0;
      const double dinv = lane < nb ? rcp_nr(ab[(int64_t)i * ldab]) : 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        if (c < nb) {
          const double yc = __shfl_sync(kFull, v * dinv, c);
          if (lane == c) v = yc;
          else if (lane > c) v = fma(-row[c], yc, v);
        }
      }
      if (lane < nb) b[i] = v;
    }
    __syncthreads();
  }
}

__device__ void band_backward(const double* __restrict__ ab, int n, int kd, int ldab, double* b) {
  constexpr int NB = kSolveNB;
  constexpr int kWarps = kCtaThreads / 32;
  __shared__ double sv[NB];
  __shared__ double dblk[NB][NB + 1];
  const int lane = threadIdx.x & 31, warp = warp_uniform(threadIdx.x >> 5);
  const int last0 = ((n - 1) / NB) * NB;
  for (int c0 = last0; c0 >= 0; c0 -= NB) {
    const int nb = min(NB, n - c0);
    for (int c = warp; c < nb; c += kWarps) {
      const int j = c0 + c;
      const double* colj = ab + (int64_t)j * ldab;
      const int len = min(kd, n - 1 - j) + 1;
      double s = 0.0, s1 = 0.0;
      int o = nb - c + lane;
      for (; o + 32 < len; o += 64) {
        const double a0 = colj[o], a1 = colj[o + 32];
        s = fma(a0, b[j + o], s);
        s1 = fma(a1, b[j + o + 32], s1);
      }
      if (o < len) s = fma(colj[o], b[j + o], s);
      s += s1;
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1) s += __shfl_xor_sync(kFull, s, sh);
      if (lane == 0) sv[c] = b[j] - s;
      dblk[lane][c] = (lane >= c && lane < nb && lane - c < len) ? colj[lane - c] : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      double v = lane < nb ? sv[lane] : 0.0;
      const double dinv = lane < nb ? rcp_nr(dblk[lane][lane]) : 0.0;
#pragma unroll
      for (int c = NB - 1; c >= 0; --c) {
        if (c < nb) {
          const double xc = __shfl_sync(kFull, v * dinv, c);
          if (lane == c) v = xc;
          else if (lane < c) v = fma(-dblk[c][lane], xc, v);
        }
      }
      if (lane < nb) b[c0 + lane] = v;
    }
    __syncthreads();
  }
}

// Solve for wide bands (the streamed ring does not fit): one CTA per right-hand side,
// blockIdx.x = matrix * nrhs + rhs; column r of matrix m at b0 + m*stride_b + r*ldb.
// Matrices with skip[m] != 0 (failed factorization) are left untouched.
__global__ void __launch_bounds__(kCtaThreads)
pbtrs_kernel(const double* ab0, int64_t stride_ab, double* b0, int64_t ldb, int64_t stride_b, int nrhs, int n, int kd,
             int ldab, int32_t* info, const int32_t* skip) {
  const int z = blockIdx.x, mat = z / nrhs, r = z - mat * nrhs;
  if (skip && skip[mat] != 0) return;
  const double* ab = ab0 + (int64_t)mat * stride_ab;
  double* b = b0 + (int64_t)mat * stride_b + (int64_t)r * ldb;
  if (!skip) {
    const int bad = first_nonpositive_diag(ab, n, ldab);
    if (bad != INT_MAX) {
      if (threadIdx.x == 0 && r == 0) info[mat] = bad + 1;
      return;
    }
  }
  band_forward(ab, n, kd, ldab, b);
  band_backward(ab, n, kd, ldab, b);
  if (threadIdx.x == 0 && r == 0) info[mat] = 0;
}

}  // namespace bcg
