// potrf_lab.cu -- one warp factoring a 16x16 (or 32x32) SPD block again and again: cycles per
// POTRF of the pivot-chain variants, each checked against a serial Cholesky.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2305_04635_b200/csrc \
//      -o potrf_lab tools/micro/potrf_lab.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "band_cta.cuh"
using namespace bcg;

constexpr int LD = 20;

// V0: the production scheme (CtaBand::potrf_diag): lanes 0-15 rows, lanes 16-31 the inverse.
__device__ __forceinline__ void potrf_v0(const double* A, double* D, double* lbuf, double eps, double& carry) {
  constexpr int NB = 16;
  const int r = threadIdx.x & 31;
  const bool inv = r >= NB;
  double row[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const double v = A[c * LD + ((c <= r && !inv) ? r : 0)] + eps * carry;
    row[c] = inv ? (c == r - NB ? 1.0 : 0.0) : v;
  }
  double p = __shfl_sync(kFull, row[0], 0);
  double alpha = __shfl_sync(kFull, row[0], 1);
  double beta = __shfl_sync(kFull, row[1], 1);
  double rs = rsqrt_nr(p);
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const double lrc = row[c] * rs;
    const double l1 = alpha * rs;
    const double pn = fma(-l1, l1, beta);
    const double rsn = rsqrt_nr(pn);
    if (c + 1 < NB) row[c + 1 < NB ? c + 1 : 0] = fma(-lrc, l1, row[c + 1 < NB ? c + 1 : 0]);
    double alpha_n = 0.0, beta_n = 0.0;
    if (c + 2 < NB) {
      const double bn = fma(-lrc, lrc, row[c + 2 < NB ? c + 2 : 0]);
      alpha_n = shfl_early(row[c + 1 < NB ? c + 1 : 0], c + 2);
      beta_n = shfl_early(bn, c + 2);
    }
    row[c] = lrc;
    double* dc = D + c * LD;
    *(inv ? lbuf + (r - NB) : dc + r) = lrc;
    __syncwarp();
#pragma unroll
    for (int h = 0; h < NB / 2; ++h) {
      if (2 * h + 1 >= c + 2) {
        const double2 l2 = reinterpret_cast<const double2*>(dc)[h];
        if (2 * h >= c + 2) row[2 * h] = fma(-lrc, l2.x, row[2 * h]);
        row[2 * h + 1] = fma(-lrc, l2.y, row[2 * h + 1]);
      }
    }
    p = pn;
    rs = rsn;
    alpha = alpha_n;
    beta = beta_n;
  }
  carry = row[15];
}

#ifndef VARIANT
#define VARIANT 0
#endif
#include "potrf_variants.cuh"

// noise: what the six worker warps of the factorization do beside the pivot warp
//   bit 0: DMMA chains (4 accumulators), bit 1: shared-memory fragment loads/stores
__device__ __forceinline__ void noise_loop(int mode, volatile int* stop, double* buf, double* sink) {
  const int lane = threadIdx.x & 31, gr = lane >> 2, gc = lane & 3;
  double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  double a0 = 1e-3 * lane, a1 = 2e-3, b0 = 1e-3, b1 = 3e-3;
  int it = 0;
  if (mode & 12) {
    double f[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    while (!*stop) {
      if (mode & 8) {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const double2 p2 = *reinterpret_cast<const double2*>(buf + c * 36 + 2 * (lane & 15));
          f[c & 3] = fma(p2.x, 1e-3, f[c & 3]);
          f[4 + (c & 3)] = fma(p2.y, 1e-3, f[4 + (c & 3)]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) f[c & 7] = fma(f[c & 7], 0.999, 1e-3);
      }
      ++it;
    }
    sink[threadIdx.x] = f[0] + f[1] + f[2] + f[3] + f[4] + f[5] + f[6] + f[7];
    if (lane == 0) sink[512 + (threadIdx.x >> 5)] = (double)it;
    return;
  }
  while (!*stop) {
    if (mode & 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u) { acc[u][0] = 1e-9 * acc[u][0] + buf[(u * 8 + gr) + 36 * (2 * gc)]; acc[u][1] = 1e-9 * acc[u][1] + buf[(u * 8 + gr) + 36 * (2 * gc + 1)]; }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (mode & 2) { a0 = buf[(4 * k + gc) * 36 + gr]; a1 = buf[(4 * k + gc) * 36 + 8 + gr]; b0 = buf[(4 * k + gc) * 36 + 16 + gr]; b1 = buf[(4 * k + gc) * 36 + 24 + gr]; }
      if (mode & 1) {
        dmma884n(acc[0][0], acc[0][1], a0, b0);
        dmma884n(acc[1][0], acc[1][1], a1, b0);
        dmma884n(acc[2][0], acc[2][1], a0, b1);
        dmma884n(acc[3][0], acc[3][1], a1, b1);
      }
    }
    if (mode & 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u) { buf[(u * 8 + gr) + 36 * (2 * gc)] = acc[u][0]; buf[(u * 8 + gr) + 36 * (2 * gc + 1)] = acc[u][1]; }
    }
    ++it;
  }
  sink[threadIdx.x] = acc[0][0] + acc[1][1] + acc[2][0] + acc[3][1];
  if (lane == 0) sink[512 + (threadIdx.x >> 5)] = (double)it;
}

template <int V>
__global__ void lab(const double* gA, double* gL, long long* cyc, int iters, double eps, int noise) {
  __shared__ __align__(16) double A[32 * 36];
  __shared__ __align__(16) double D[2][32 * 36];
  __shared__ __align__(16) double lbuf[64];
  extern __shared__ __align__(16) double nbuf_all[];
  __shared__ int stop, piv;
  if (threadIdx.x == 0) { stop = 0; unsigned h; asm volatile("mov.u32 %0, %%warpid;" : "=r"(h)); piv = h & 3; }
  if (noise) for (int t = threadIdx.x; t < 8 * 1024; t += blockDim.x) nbuf_all[t] = 1e-6 * (t % 13);
  __syncthreads();
  if (threadIdx.x >= 32) {
    const int w = threadIdx.x >> 5;
    unsigned hw;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(hw));
    if ((noise >> (4 + ((hw - piv) & 3))) & 1) noise_loop(noise & 15, &stop, nbuf_all + w * 1024, gL + 2048);
    return;
  }
  const int lane = threadIdx.x;
  for (int t = lane; t < 32 * 36; t += 32) { A[t] = 0; D[0][t] = 0; D[1][t] = 0; }
  __syncwarp();
  constexpr int N = variant_n<V>();
  constexpr int ld = variant_ld<V>();
  for (int t = lane; t < N * N; t += 32) A[(t / N) * ld + (t % N)] = gA[t];
  __syncwarp();
  double carry = 0.0;
  // warm
  run_variant<V>(A, D[0], lbuf, eps, carry);
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    run_variant<V>(A, D[it & 1], lbuf, eps, carry);
  }
  long long t1 = clock64();
  __syncwarp();
  if (lane == 0) cyc[0] = (t1 - t0) / iters;
  stop = 1;
  for (int t = lane; t < N * N; t += 32) gL[t] = D[(iters - 1) & 1][(t / N) * ld + (t % N)];
  if (lane == 0) gL[N * N] = carry;
}

// dependent-chain latencies of the pivot warp's communication primitives under the same noise
__global__ void latprobe(long long* out, int noise, int iters) {
  extern __shared__ __align__(16) double nbuf_all[];
  __shared__ int stop, piv;
  __shared__ double sbuf[64];
  if (threadIdx.x == 0) { stop = 0; unsigned h; asm volatile("mov.u32 %0, %%warpid;" : "=r"(h)); piv = h & 3; }
  if (noise) for (int t = threadIdx.x; t < 8 * 1024; t += blockDim.x) nbuf_all[t] = 1e-6 * (t % 13);
  if (threadIdx.x < 64) sbuf[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x >= 32) {
    const int w = threadIdx.x >> 5;
    unsigned hw;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(hw));
    if ((noise >> (4 + ((hw - piv) & 3))) & 1) noise_loop(noise & 15, &stop, nbuf_all + w * 1024, (double*)(out + 64));
    return;
  }
  const int lane = threadIdx.x;
  double x = lane;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = __shfl_sync(kFull, x, (lane + 1) & 31) + 1e-9;
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) {
    sbuf[lane] = x;
    __syncwarp();
    x = sbuf[(lane + 1) & 31] + 1e-9;
    __syncwarp();
  }
  long long t2 = clock64();
  int idx = lane;
  for (int it = 0; it < iters; ++it) idx = (int)sbuf[32 + (idx & 31)] - 32 + lane - (idx & 31) ;
  long long t3 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, 0.999, 1e-3);
  long long t4 = clock64();
  if (lane == 0) { out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters; out[3] = (t4 - t3) / iters; }
  stop = 1;
  out[8 + lane] = (long long)x + idx;
}

// the production function itself (CtaBand<16,100>::potrf_diag) on a real ring window: prologue
// (rows from the ring), column loop, epilogue (L back to the ring, L^-1 to D)
__global__ void lab_prod(const double* gA, long long* cyc, int iters, int s0, int noise) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int stop, piv;
  CtaGeom g;
  g.n = 1 << 20; g.kd = 100; g.ldab = 101; g.lds = 101; g.nslot = 116; g.pld = 100;
  CtaBand<16, 100> w{g};
  w.win = sm;
  w.P = sm + 116 * 101;
  w.D = w.P + 1600;
  w.lbuf = w.D + 640;
  double* nbuf = w.lbuf + 64;
  if (threadIdx.x == 0) { stop = 0; unsigned h; asm volatile("mov.u32 %0, %%warpid;" : "=r"(h)); piv = h & 3; }
  if (noise) for (int t = threadIdx.x; t < 8 * 1024; t += blockDim.x) nbuf[t] = 1e-6 * (t % 13);
  __syncthreads();
  if (threadIdx.x >= 32) {
    const int wq = threadIdx.x >> 5;
    unsigned hw;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(hw));
    if ((noise >> (4 + ((hw - piv) & 3))) & 1) noise_loop(noise & 15, &stop, nbuf + wq * 1024, (double*)(cyc + 64));
    return;
  }
  const int r = threadIdx.x;
  auto fill = [&]() {
    if (r < 16)
      for (int c = 0; c <= r; ++c) {
        const int sl = (s0 + c) % 116;
        w.win[sl * 101 + (r - c)] = gA[c * 16 + r];
      }
    __syncwarp();
  };
  fill();
  int f = w.potrf_diag(s0, 4096, 16);
  long long tf = 0, tp = 0;
  for (int it = 0; it < iters; ++it) {
    long long t0 = clock64();
    fill();
    long long t1 = clock64();
    f += w.potrf_diag(s0, 4096, 16);
    long long t2 = clock64();
    tf += t1 - t0;
    tp += t2 - t1;
  }
  if (r == 0) { cyc[0] = tp / iters; cyc[1] = tf / iters; cyc[2] = f; }
  stop = 1;
}

template <int V>
void run(const char* name, int noise = 0) {
  constexpr int N = variant_n<V>();
  std::vector<double> a(N * N), l(N * N, 0.0), out(N * N + 1);
  srand(1);
  for (int c = 0; c < N; ++c)
    for (int r = 0; r < N; ++r) a[c * N + r] = 0;
  for (int c = 0; c < N; ++c)
    for (int r = c + 1; r < N; ++r) { double v = 2.0 * rand() / RAND_MAX - 1.0; a[c * N + r] = v; a[r * N + c] = v; }
  for (int r = 0; r < N; ++r) { double s = 1.0; for (int c = 0; c < N; ++c) if (c != r) s += fabs(a[c * N + r]); a[r * N + r] = s; }
  // serial cholesky (column-major a[c*N + r])
  std::vector<double> w = a;
  for (int c = 0; c < N; ++c) {
    double d = sqrt(w[c * N + c]);
    for (int r = c; r < N; ++r) w[c * N + r] /= d;
    for (int c2 = c + 1; c2 < N; ++c2)
      for (int r = c2; r < N; ++r) w[c2 * N + r] -= w[c * N + r] * w[c * N + c2];
  }
  double *dA, *dL; long long* dc;
  cudaMalloc(&dA, sizeof(double) * N * N); cudaMalloc(&dL, sizeof(double) * 4096); cudaMemset(dL, 0, sizeof(double) * 4096); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, a.data(), sizeof(double) * N * N, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(lab<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  lab<V><<<1, noise ? 256 : 32, noise ? 65536 : 0>>>(dA, dL, dc, 2000, 0.0, noise);
  cudaError_t e = cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(out.data(), dL, sizeof(double) * (N * N + 1), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int c = 0; c < N; ++c) for (int r = c; r < N; ++r) err = fmax(err, fabs(out[c * N + r] - w[c * N + r]));
  std::vector<double> aux(4096, 0.0);
  cudaMemcpy(aux.data(), dL, sizeof(double) * 4096, cudaMemcpyDeviceToHost);
  double nit = 0; for (int w = 0; w < 8; ++w) nit += aux[2048 + 512 + w];
  printf("[noise dmma/cycle(SM) %.3f] ", nit * 16.0 / (2000.0 * cyc));
  printf("%-28s noise=%02x N=%d  %6lld cycles/potrf  %6.1f /col   maxerr %.2e  (%s)\n", name, noise, N, cyc, (double)cyc / N, err, cudaGetErrorString(e));
  cudaFree(dA); cudaFree(dL); cudaFree(dc);
}

void probe(int noise) {
  long long* d; cudaMalloc(&d, 8 * 4096); cudaMemset(d, 0, 8 * 4096);
  cudaFuncSetAttribute(latprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  latprobe<<<1, noise ? 256 : 32, 65536>>>(d, noise, 2000);
  cudaDeviceSynchronize();
  long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("latency noise=%02x: shfl %lld  sts+sync+lds %lld  lds-chase %lld  dfma %lld\n", noise, h[0], h[1], h[2], h[3]);
  cudaFree(d);
}

int main() {
  for (int m : {0x00, 0xe2, 0xe3, 0xe1, 0x12, 0xf3}) probe(m);
  {
    const int N = 16;
    std::vector<double> a(N * N);
    srand(1);
    for (int c = 0; c < N; ++c)
      for (int r2 = c + 1; r2 < N; ++r2) { double v = 2.0 * rand() / RAND_MAX - 1.0; a[c * N + r2] = v; a[r2 * N + c] = v; }
    for (int r2 = 0; r2 < N; ++r2) { double sum = 1.0; for (int c = 0; c < N; ++c) if (c != r2) sum += fabs(a[c * N + r2]); a[r2 * N + r2] = sum; }
    double* dA; long long* dc;
    cudaMalloc(&dA, sizeof(double) * N * N); cudaMalloc(&dc, 8 * 4096);
    cudaMemcpy(dA, a.data(), sizeof(double) * N * N, cudaMemcpyHostToDevice);
    const int smem = (116 * 101 + 1600 + 640 + 64 + 8 * 1024) * 8;
    cudaFuncSetAttribute(lab_prod, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int s0 : {0, 96, 108})
      for (int nz : {0x00, 0xe3}) {
        cudaMemset(dc, 0, 8 * 4096);
        lab_prod<<<1, nz ? 256 : 32, smem>>>(dA, dc, 2000, s0, nz);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[3]; cudaMemcpy(h, dc, 24, cudaMemcpyDeviceToHost);
        printf("production potrf_diag on the ring: s0=%3d noise=%02x  %lld cycles/potrf (+ %lld refill)  fail-sum %lld (%s)\n",
               s0, nz, h[0], h[1], h[2], cudaGetErrorString(e));
      }
    cudaFree(dA); cudaFree(dc);
  }
  const int masks[] = {0x00, 0xe1, 0x11, 0x14, 0xe2, 0xe3, 0xf3};
  for (int m : masks) run<0>("v0 production", m);
  for (int m : masks) run<1>("v2 three-row lookahead", m);
  return 0;
}
