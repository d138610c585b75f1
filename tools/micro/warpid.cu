// Which SM sub-partition does each warp land on?  2 CTAs x 8 warps per SM (113 KB smem each,
// as the C5 kernel), prints (block, warp, smid, %warpid) for the first SMs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) k(int* out) {
  extern __shared__ double sm[];
  unsigned smid, wid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if ((threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    out[(blockIdx.x * 8 + w) * 2] = smid;
    out[(blockIdx.x * 8 + w) * 2 + 1] = wid;
  }
  sm[threadIdx.x] = 1;
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) {}
}
int main() {
  int* d; cudaMalloc(&d, 296 * 8 * 2 * 4);
  size_t smem = 113 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<296, 256, smem>>>(d); cudaDeviceSynchronize();
  static int h[296 * 16]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int mism = 0;
  for (int b = 0; b < 296; ++b) {
    if (b < 0) {
      printf("block %d smid %d warpids", b, h[b * 16]);
      for (int w = 0; w < 8; ++w) printf(" %d", h[(b * 8 + w) * 2 + 1]);
      printf("\n");
    }
    for (int w = 0; w < 8; ++w) if ((h[(b * 8 + w) * 2 + 1] & 3) != (w & 3)) ++mism;
  }
  for (int sm = 0; sm < 3; ++sm) {
    printf("SM %d:", sm);
    for (int b = 0; b < 296; ++b) if (h[b * 16] == sm) {
      printf(" [block %d:", b);
      for (int w = 0; w < 8; ++w) printf(" %d", h[(b * 8 + w) * 2 + 1]);
      printf("]");
    }
    printf("\n");
  }
  int same = 0;
  for (int b = 0; b < 148; ++b) same += h[b * 16] == h[(b + 148) * 16];
  printf("warps whose %%warpid%%4 != w%%4: %d; blocks b, b+148 on the same SM: %d of 148\n", mism, same);
  return 0;
}
