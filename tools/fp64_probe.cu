// FP64 microbenchmarks for B200 (sm_100a): the numbers the band-Cholesky roofline
// and the pivot-chain bound are built on.
//   * DFMA throughput (FP64 pipe), full chip
//   * DMMA m8n8k4 throughput (legacy warp-level FP64 tensor path), full chip
//   * latencies of the operations on the factorization's sequential pivot chain:
//     dependent DFMA, sqrt, rsqrt, 1/x, __drcp_rn, 64-bit shuffle, smem round trip
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dfma_tput(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_tput(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - a;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

// latency probes: one thread, dependent chain, clock64 around N links
template <int OP>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[64];
  double x = x0;
  sm[threadIdx.x] = x0;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = fma(x, 0.9999999, 1e-9);
    if (OP == 1) x = sqrt(x) + 1.0;          // correctly rounded sqrt (+ dep add)
    if (OP == 2) x = rsqrt(x) + 1.0;
    if (OP == 3) x = 1.0 / x + 1.0;          // IEEE division
    if (OP == 4) x = __drcp_rn(x) + 1.0;
    if (OP == 5) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
    if (OP == 6) { sm[threadIdx.x] = x; __syncwarp(); x = sm[(threadIdx.x + 1) & 31] + 1e-9; __syncwarp(); }
    if (OP == 7) x = x * 1.0000001;          // dependent DMUL
    if (OP == 8) x = x + 1e-9;               // dependent DADD
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}

template <int OP>
int run_lat(const char* name, double x0, int threads) {
  double* d; long long* c; long long h;
  CK(cudaMalloc(&d, 8)); CK(cudaMalloc(&c, 8));
  const int n = 4096;
  lat<OP><<<1, threads>>>(d, c, x0, n);  // warm
  lat<OP><<<1, threads>>>(d, c, x0, n);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("{\"probe\":\"latency\",\"op\":\"%s\",\"cycles_per_link\":%.2f}\n", name, (double)h / n);
  cudaFree(d); cudaFree(c);
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"probe\":\"device\",\"name\":\"%s\",\"sms\":%d,\"smem_optin\":%zu,\"clock_khz\":%d,\"l2\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, clk_khz, p.l2CacheSize);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    int iters = 4096;
    dfma_tput<<<blocks, tpb>>>(out, 16);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_tput<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 64.0 * iters * (double)blocks * tpb;
    printf("{\"probe\":\"dfma_tput\",\"tpb\":%d,\"blocks\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", tpb, blocks, best, flops / best / 1e9);
  }
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (2048 / tpb);
    int iters = 1024;
    dmma_tput<<<blocks, tpb>>>(out, 16);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_tput<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256.0 * 32.0 * iters * (double)blocks * (tpb / 32);  // 8x8x4 MACs per mma
    printf("{\"probe\":\"dmma_tput\",\"tpb\":%d,\"blocks\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", tpb, blocks, best, flops / best / 1e9);
  }
  run_lat<0>("dfma", 1.0, 32);
  run_lat<7>("dmul", 1.0, 32);
  run_lat<8>("dadd", 1.0, 32);
  run_lat<1>("sqrt+add", 2.0, 32);
  run_lat<2>("rsqrt+add", 2.0, 32);
  run_lat<3>("div+add", 2.0, 32);
  run_lat<4>("drcp_rn+add", 2.0, 32);
  run_lat<5>("shfl64+add", 1.0, 32);
  run_lat<6>("smem_roundtrip+add", 1.0, 32);
  return 0;
}
