// Cost of the pieces of one streamed-solve chain step (band_sweep.cuh), one warp alone on
// an SM (cycles per iteration, every iteration data-dependent on the previous one):
//   prod     16 LDS operands + 16 broadcast LDS + 16 DFMA in 4 chains + 3 DADD
//   wait     mbarrier try_wait on an already-completed phase
//   arrive   mbarrier arrive (no waiter)
//   stsld    STS, __syncwarp, LDS round trip
//   stgsync  STG then __syncwarp
//   step     the forward step's sequence: prod, 3 waits, 2 LDS, STS + sync + prod, STS, sync,
//            3 arrives, STG
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_step tools/micro/chain_step.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void marrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void mwait(unsigned long long* b, unsigned ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                   su(b)), "r"(ph) : "memory");
}

__global__ void k(double* gout, long long* cyc, int n) {
  __shared__ __align__(16) double sm[4096];
  __shared__ __align__(8) unsigned long long bars[4];
  const int lane = threadIdx.x, i = lane & 15;
  for (int t = lane; t < 4096; t += 32) sm[t] = 1e-3 * (t % 7);
  if (lane < 4) minit(&bars[lane], 1);
  __syncwarp();
  if (lane == 0) marrive(&bars[0]);  // phase 0 of bars[0..2] complete
  if (lane == 0) marrive(&bars[1]);
  if (lane == 0) marrive(&bars[2]);
  if (lane == 0) minit(&bars[3], (1 << 20) - 1);
  __syncwarp();
  double x = 0.25;
  auto prod = [&](int off) {
    double l[16], v[16];
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) l[kk] = sm[off + kk * 100 + i];
#pragma unroll
    for (int kk = 0; kk < 16; kk += 2) {
      const double2 t = *reinterpret_cast<const double2*>(sm + 2048 + off + kk);
      v[kk] = t.x;
      v[kk + 1] = t.y;
    }
    double a[4] = {0, 0, 0, 0};
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) a[kk & 3] = fma(l[kk], v[kk], a[kk & 3]);
    return (a[0] + a[1]) + (a[2] + a[3]);
  };
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) x = prod(((int)x) & 7) * 1e-3;
  long long t1 = clock64();
  for (int it = 0; it < n; ++it) mwait(&bars[((int)x) & 1], 0), x += 1e-9;
  long long t2 = clock64();
  for (int it = 0; it < n; ++it) {
    if (lane == 0) marrive(&bars[3]);
    x += 1e-9;
  }
  long long t3 = clock64();
  for (int it = 0; it < n; ++it) {
    sm[3000 + lane + (((int)x) & 1)] = x;
    __syncwarp();
    x = sm[3000 + ((lane + 1) & 31)] * 0.5;
  }
  long long t4 = clock64();
  for (int it = 0; it < n; ++it) {
    gout[lane + 32 * (it & 63)] = x;
    __syncwarp();
    x += 1e-9;
  }
  long long t5 = clock64();
  for (int it = 0; it < n; ++it) {
    const int off = ((int)x) & 7;
    double u = prod(off);
    mwait(&bars[0], 0);
    mwait(&bars[1], 0);
    mwait(&bars[2], 0);
    double v = sm[1000 + i + off] + sm[1100 + i] - u;
    sm[1200 + off + i] = v;
    __syncwarp();
    double o = prod(off + 200);
    sm[1400 + i] = o;
    __syncwarp();
    if (lane == 0) { marrive(&bars[3]); marrive(&bars[3]); marrive(&bars[3]); }
    gout[lane + 32 * (it & 63)] = o;
    x = o * 1e-3;
  }
  long long t6 = clock64();
  if (lane == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
  gout[4096 + lane] = x;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8 * 8192);
  cudaMalloc(&c, 64);
  const int n = 2048;
  k<<<1, 32>>>(o, c, 16);
  cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, n);
  cudaDeviceSynchronize();
  long long h[6];
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  if (cudaGetLastError() != cudaSuccess) { printf("cuda error\n"); return 1; }
  printf("{\"prod\": %.1f, \"wait_complete\": %.1f, \"arrive\": %.1f, \"sts_sync_lds\": %.1f, \"stg_sync\": %.1f, "
         "\"step\": %.1f}\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n, (double)h[5] / n);
  return 0;
}
