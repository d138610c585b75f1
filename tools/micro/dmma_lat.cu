// DMMA m8n8k4 f64 latency on B200: dependent chain, 4 interleaved chains, and a 16x16x16
// tile update from shared memory (8 accumulator loads, 16 operand loads, 16 DMMA, 8 stores),
// one warp alone on the SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sm[4096];
  const int lane = threadIdx.x;
  for (int i = lane; i < 4096; i += 32) sm[i] = 1e-3 * (i % 7);
  __syncwarp();
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0, c6 = 0, c7 = 0;
  double a = lane * 1e-3, b = 1 - a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(c0, c1, a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { dmma(c0, c1, a, b); dmma(c2, c3, a, b); dmma(c4, c5, a, b); dmma(c6, c7, a, b); }
  long long t2 = clock64();
  const int gr = lane >> 2, gc = lane & 3;
  for (int i = 0; i < n; ++i) {
    double acc[8];
    const int base = (i & 7) * 256;
    for (int j = 0; j < 8; ++j) acc[j] = sm[base + j * 32 + lane];
    for (int k0 = 0; k0 < 16; k0 += 4) {
      const double* pk = sm + 2048 + (k0 + gc) * 20;
      const double a0 = pk[gr], a1 = pk[8 + gr], b0 = pk[gr + 2], b1 = pk[10 + gr];
      dmma(acc[0], acc[1], a0, b0); dmma(acc[2], acc[3], a1, b0); dmma(acc[4], acc[5], a0, b1); dmma(acc[6], acc[7], a1, b1);
    }
    for (int j = 0; j < 8; ++j) sm[base + j * 32 + lane] = acc[j];
    __syncwarp();
  }
  long long t3 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
  out[lane] = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  const int n = 1024;
  k<<<1, 32>>>(o, c, 16); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, n); cudaDeviceSynchronize();
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("{\"dmma_dep_latency\": %.1f, \"dmma_4chain_per_instr\": %.1f, \"tile16_update_cycles\": %.1f}\n",
         (double)h[0] / n, (double)h[1] / (4.0 * n), (double)h[2] / n);
  return 0;
}
