// Launch-gap micro-test: event-timed duration of an empty 148 x 512 kernel holding 192 KB of
// dynamic shared memory, launched after (a) cudaMemsetAsync, (b) the same kernel, (c) a reset
// kernel that prefers the maximum shared-memory carveout. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k_big(unsigned* out) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0) { sm[0] = 1; if (blockIdx.x == 0) out[0] = sm[0]; }
}
__global__ void k_reset(unsigned* p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 0;
}
__global__ void k_sleep(unsigned long long ns) {
  unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); if (t - t0 > ns) break; }
}
int main() {
  const int smem = 3 * 65536;
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned* buf; cudaMalloc(&buf, 64 << 20);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int variant = 0; variant < 4; ++variant) {
    if (variant == 3) cudaFuncSetAttribute(k_reset, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    float tot = 0; int n = 0;
    for (int it = 0; it < 30; ++it) {
      k_sleep<<<1, 32, 0, s>>>(100000);
      if (variant == 0) cudaMemsetAsync(buf, 0, 1 << 20, s);
      else if (variant == 1) k_big<<<148, 512, smem, s>>>(buf + 1024);
      else if (variant == 2) k_reset<<<148, 512, 0, s>>>(buf + 4096, 1 << 18);
      else k_reset<<<148, 512, 0, s>>>(buf + 4096, 1 << 18);
      cudaEventRecord(a, s);
      k_big<<<148, 512, smem, s>>>(buf);
      cudaEventRecord(b, s);
      cudaStreamSynchronize(s);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it >= 5) { tot += ms; ++n; }
    }
    const char* names[] = {"after memset", "after same kernel", "after reset kernel (default carveout)", "after reset kernel (carveout 100)"};
    printf("%-42s %.2f us\n", names[variant], 1000 * tot / n);
  }
  // baseline variant 3 done with carveout already set; add default-carveout reset for comparison
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
