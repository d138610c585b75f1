// band_residual.cuh -- device-side backward error ||A - L L^T||_F / ||A||_F over the band,
// the GPU restatement of the reference's residual_norm (pkg/src/bandchol/core.py:186-213)
// for fast validation of the large configs.
//
// Entry (d, j) of the band (row j+d, column j, d = 0..kd, j+d < n):
//   recon(d, j) = sum_{s=0}^{min(kd-d, j)} L(j+d, j-s) L(j, j-s)       (core.py:203-205)
//   num += w_d (A(d,j) - recon(d,j))^2,  den += w_d A(d,j)^2,  w_0 = 1, w_d = 2  (:207-210)
// One thread per band entry, lanes along d so the L(j+d, j-s) loads of a warp are one
// contiguous run of column j-s; L(j, j-s) is a broadcast.  Deterministic: a fixed grid,
// per-block tree reductions into a caller workspace, then one block sums the partials in
// block order (no atomics).
#pragma once
#include "band_cta.cuh"

namespace bcg {

constexpr int kResidThreads = 256;

__device__ __forceinline__ void block_sum2(double& a, double& b) {
  __shared__ double sa[kResidThreads / 32], sb[kResidThreads / 32];
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {
    a += __shfl_xor_sync(kFull, a, sh);
    b += __shfl_xor_sync(kFull, b, sh);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sa[w] = a;
    sb[w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0.0;
    b = 0.0;
    for (int i = 0; i < kResidThreads / 32; ++i) {
      a += sa[i];
      b += sb[i];
    }
  }
}

// blockIdx.y = matrix of a batch (a + y*stride_a, l + y*stride_l); partials of matrix y at
// partial + 2*gridDim.x*y.
__global__ void __launch_bounds__(kResidThreads)
band_residual_kernel(int n, int kd, const double* __restrict__ a, int lda, const double* __restrict__ l, int ldl,
                     double* __restrict__ partial, int64_t stride_a = 0, int64_t stride_l = 0) {
  a += (int64_t)blockIdx.y * stride_a;
  l += (int64_t)blockIdx.y * stride_l;
  partial += (size_t)2 * gridDim.x * blockIdx.y;
  double num = 0.0, den = 0.0;
  for (int j = blockIdx.x; j < n; j += gridDim.x) {
    for (int d = threadIdx.x; d <= kd; d += kResidThreads) {
      if (j + d >= n) continue;
      const int smax = min(kd - d, j);
      double r0 = 0.0, r1 = 0.0;
      int s = 0;
      for (; s + 1 <= smax; s += 2) {
        const double* c0 = l + (int64_t)(j - s) * ldl;
        const double* c1 = c0 - ldl;
        r0 = fma(c0[d + s], c0[s], r0);
        r1 = fma(c1[d + s + 1], c1[s + 1], r1);
      }
      if (s <= smax) {
        const double* c0 = l + (int64_t)(j - s) * ldl;
        r0 = fma(c0[d + s], c0[s], r0);
      }
      const double av = a[(int64_t)j * lda + d];
      const double diff = av - (r0 + r1);
      const double w = d == 0 ? 1.0 : 2.0;
      num = fma(w * diff, diff, num);
      den = fma(w * av, av, den);
    }
  }
  block_sum2(num, den);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = num;
    partial[2 * blockIdx.x + 1] = den;
  }
}

// one thread per matrix (batch of `count`): partials summed in block order
__global__ void band_residual_finish(const double* __restrict__ partial, int blocks, double* __restrict__ out,
                                     int count = 1) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= count) return;
  partial += (size_t)2 * blocks * y;
  out += y;
  double num = 0.0, den = 0.0;
  for (int i = 0; i < blocks; ++i) {
    num += partial[2 * i];
    den += partial[2 * i + 1];
  }
  out[0] = den == 0.0 ? (num == 0.0 ? 0.0 : __longlong_as_double(0x7ff0000000000000LL)) : sqrt(num / den);
}

}  // namespace bcg
