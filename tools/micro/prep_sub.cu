// Cycles of one prep substitution (band_sweep.cuh prep_forward / prep_backward), one warp
// alone on an SM, n calls back to back (each call's output feeds the next call's input).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2305_04635_b200/csrc -o prep_sub tools/micro/prep_sub.cu
#include <cstdio>
#include "band_sweep.cuh"

__global__ void __launch_bounds__(256, 2) k(const double* g, double* out, long long* cyc, int n, int ldab, int kd) {
  extern __shared__ __align__(16) double sm[];
  for (int i = threadIdx.x; i < 16 * ldab * 2 + 2 * 16 * bcg::kLinvLd; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x, j = lane & 15;
  const bool second = lane >= 16;
  double* o = sm + 32 * ldab;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    bcg::prep_forward<true>(sm + 16 * ldab, sm, true, 16, kd, ldab, j, second, o + (second ? 16 * bcg::kLinvLd : 0));
    __syncwarp();
  }
  long long t1 = clock64();
  for (int it = 0; it < n; ++it) {
    bcg::prep_backward<true>(sm, 16, 16, kd, ldab, j, second, o + (second ? 16 * bcg::kLinvLd : 0));
    __syncwarp();
  }
  long long t2 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  out[lane] = o[lane];
}

int main() {
  const int ldab = 101, kd = 100, n = 256;
  const int words = 16 * ldab * 2 + 2 * 16 * bcg::kLinvLd;
  double* h = new double[words];
  for (int i = 0; i < words; ++i) h[i] = (i % ldab == 0) ? 4.0 : 0.01 * ((i * 7) % 13 - 6);
  double *g, *o;
  long long* c;
  cudaMalloc(&g, words * 8);
  cudaMalloc(&o, 256 * 8);
  cudaMalloc(&c, 16);
  cudaMemcpy(g, h, words * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 8);
  k<<<1, 32, words * 8>>>(g, o, c, 4, ldab, kd);
  k<<<1, 32, words * 8>>>(g, o, c, n, ldab, kd);
  cudaDeviceSynchronize();
  long long r[2];
  cudaMemcpy(r, c, 16, cudaMemcpyDeviceToHost);
  if (cudaGetLastError() != cudaSuccess) { printf("cuda error\n"); return 1; }
  printf("{\"prep_forward\": %.1f, \"prep_backward\": %.1f}\n", (double)r[0] / n, (double)r[1] / n);
  return 0;
}
