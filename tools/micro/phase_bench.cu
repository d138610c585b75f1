// Microbenchmark: cycles of the one-CTA kernel's phases in isolation (window in smem,
// 256 threads, __launch_bounds__(256, 2)); plus DMMA / DFMA dependent-chain latency.
#include <cstdio>
#include "../../paper_2305_04635_b200/csrc/band_cta.cuh"
using namespace bcg;

__global__ void lat_dmma(long long* cyc, double* out) {
  double d0 = threadIdx.x, d1 = 1.0, a = 0.5, b = 0.25;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) dmma884(d0, d1, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
  out[threadIdx.x] = d0 + d1;
}

template <int NB>
__global__ void __launch_bounds__(256, 2) k(double* out, long long* cyc, int reps, int which, CtaGeom g, int s0p, int j0p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(16) double D[NB * NB], Dinv[NB], lbuf[32];
  CtaBand<NB, false> w{g};
  w.ab = nullptr; w.rhs = nullptr; w.win = sm; w.P = sm + 116 * 101; w.D = D; w.Dinv = Dinv; w.lbuf = lbuf;
  for (int i = threadIdx.x; i < 116 * 101; i += 256) sm[i] = (i % 101 == 0) ? 200.0 : 0.01 * ((i * 7) % 13);
  for (int i = threadIdx.x; i < NB * 116; i += 256) w.P[i] = 0.001 * (i % 17);
  for (int i = threadIdx.x; i < NB * NB; i += 256) D[i] = (i % (NB + 1) == 0) ? 2.0 : 0.01;
  if (threadIdx.x < NB) Dinv[threadIdx.x] = 0.5;
  __syncthreads();
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    long long t0 = clock64();
    if (which == 0) w.trsm_panel(0, 0, NB, 100);
    if (which == 1) w.update_tiles(0, 0, NB, 100, 0, NB / 16, 0);
    if (which == 2) w.update_tiles(0, 0, NB, 100, NB / 16, 1 << 20, 1);
    if (which == 3) w.update_tiles(0, 0, NB, 100, 0, 1 << 20, 0);
    if (which == 7) {
      // the kernel's per-step code mix: TRSM, part-1 update, then POTRF || rest update
      w.trsm_panel(0, 0, NB, 100);
      __syncthreads();
      w.update_tiles(0, 0, NB, 100, 0, NB / 16, 0);
      __syncthreads();
      if (threadIdx.x < 32) {
        long long a0 = clock64();
        w.template potrf_diag<true>(0, 0, NB);
        long long a1 = clock64();
        if (threadIdx.x == 0) tot += a1 - a0;
      } else {
        w.update_tiles(0, 0, NB, 100, NB / 16, 1 << 20, 1);
      }
    }
    if (which >= 4 && which < 7) {
      // POTRF timed alone on warp 0 while the other warps do: 4 = nothing, 5 = DMMA updates,
      // 6 = DFMA register work
      if (threadIdx.x < 32) {
        long long a0 = clock64();
        w.template potrf_diag<false>(s0p, j0p, NB);
        long long a1 = clock64();
        if (threadIdx.x == 0) tot += a1 - a0;
      } else if (which == 5 && (threadIdx.x >> 5) != 4) {
        for (int q = 0; q < 3; ++q) w.update_tiles(0, 0, NB, 100, NB / 16, 1 << 20, 1);
      } else if (which == 6 && (threadIdx.x >> 5) != 4) {
        double x = threadIdx.x, y = 1.0;
        for (int q = 0; q < 2000; ++q) { x = fma(x, 0.999, 1e-3); y = fma(y, 0.999, 1e-3); }
        if (x == 12345.0) sm[0] = x + y;
      }
    }
    __syncthreads();
    long long t1 = clock64();
    if (which < 4) tot += t1 - t0;
    if (which == 7) {  // restore an SPD window for the next round
      for (int i = threadIdx.x; i < 116 * 101; i += 256) sm[i] = (i % 101 == 0) ? 200.0 : 0.01 * ((i * 7) % 13);
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) { cyc[0] = tot / reps; out[0] = sm[5]; }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  long long h;
  lat_dmma<<<1, 32>>>(cyc, out); cudaDeviceSynchronize();
  lat_dmma<<<1, 32>>>(cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"dmma_dep_latency\": %lld}\n", h);
  size_t sm = (116 * 101 + 16 * 116) * 8;
  cudaFuncSetAttribute(k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const char* names[] = {"trsm", "update_part1", "update_rest_6warps", "update_all_8warps",
                         "potrf_alone", "potrf_with_dmma", "potrf_with_dfma", "potrf_in_step_mix"};
  CtaGeom g;
  g.n = 1 << 20; g.kd = 100; g.ldab = 101; g.lds = 101; g.nslot = 116; g.pld = 116;
  for (int wh = 0; wh < 8; ++wh) {
    k<16><<<1, 256, sm>>>(out, cyc, 20, wh, g, 5, 16*37); cudaDeviceSynchronize();
    k<16><<<1, 256, sm>>>(out, cyc, 20, wh, g, 5, 16*37); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"%s_cycles\": %lld, \"err\": \"%s\"}\n", names[wh], h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
