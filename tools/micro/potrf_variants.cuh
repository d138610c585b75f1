#pragma once
template <int V> constexpr int variant_n() { return 16; }
template <int V> constexpr int variant_ld() { return LD; }
template <int V>
__device__ __forceinline__ void run_variant(const double* A, double* D, double* lbuf, double eps, double& carry) {
  potrf_v0(A, D, lbuf, eps, carry);
}
