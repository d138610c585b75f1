// Microbenchmark: cycles of the warp POTRF (CtaBand::potrf_diag) in the kernel's setting:
// window in shared memory, 256-thread CTA with __launch_bounds__(256, 2).
#include <cstdio>
#include "../../paper_2305_04635_b200/csrc/band_cta.cuh"
using namespace bcg;

template <int NB>
__global__ void __launch_bounds__(256, 2) k(double* out, long long* cyc, int reps, int nbrt) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double D[NB * NB], Dinv[NB], lbuf[32];
  CtaGeom g;
  g.n = 1 << 20; g.kd = 100; g.ldab = 101; g.lds = 101; g.nslot = 120; g.pld = 116;
  CtaBand<NB, false> w{g};
  w.ab = nullptr; w.rhs = nullptr; w.win = sm; w.P = sm + 120 * 101; w.D = D; w.Dinv = Dinv; w.lbuf = lbuf;
  double* win = sm;
  for (int i = threadIdx.x; i < 120 * 101; i += 256) win[i] = (i % 101 == 0) ? 200.0 : 0.01 * ((i * 7) % 13);
  __syncthreads();
  long long tot = 0;
  int f = 0;
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x < 32) {
      long long t0 = clock64();
      f += w.template potrf_diag<true>(0, 0, nbrt);
      long long t1 = clock64();
      tot += t1 - t0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NB * 101; i += 256) win[i] = (i % 101 == 0) ? 200.0 : 0.01 * ((i * 7) % 13);
    __syncthreads();
  }
  if (threadIdx.x == 0) { cyc[0] = tot / reps; out[0] = f; }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  long long h;
  size_t sm = (120 * 101 + 16 * 116) * 8;
  cudaFuncSetAttribute(k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<16><<<1, 256, sm>>>(out, cyc, 50, 16); cudaDeviceSynchronize();
  k<16><<<1, 256, sm>>>(out, cyc, 50, 16); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"potrf16_cycles\": %lld, \"err\": \"%s\"}\n", h, cudaGetErrorString(cudaGetLastError()));
  size_t sm32 = (120 * 101 + 32 * 116) * 8;
  cudaFuncSetAttribute(k<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm32);
  k<32><<<1, 256, sm32>>>(out, cyc, 50, 32); cudaDeviceSynchronize();
  k<32><<<1, 256, sm32>>>(out, cyc, 50, 32); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"potrf32_cycles\": %lld, \"err\": \"%s\"}\n", h, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
