// Launch-cost micro-test: event-timed duration of an empty 148-CTA kernel as a function of
// the kernel-parameter size (__grid_constant__ struct of 16 B .. 4 KB), the CTA size and the
// dynamic shared memory. Decides whether the comm kernel's ~2.7 KB CommArgs should move to
// device memory. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/exp_launch.bin tools/exp_launch.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int BYTES>
struct Args {
  unsigned char b[BYTES];
};
template <int BYTES>
__global__ void __launch_bounds__(512, 1) k_empty(const __grid_constant__ Args<BYTES> a, unsigned* out) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0) {
    sm[0] = a.b[BYTES - 1];
    if (blockIdx.x == 0) out[0] = sm[0];
  }
}
__global__ void k_sleep(unsigned long long ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > ns) break;
  }
}
template <int BYTES>
void run(int threads, int smem, cudaStream_t s, unsigned* buf) {
  cudaFuncSetAttribute(k_empty<BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  Args<BYTES> a{};
  a.b[BYTES - 1] = 3;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float tot = 0;
  int n = 0;
  for (int it = 0; it < 40; ++it) {
    k_sleep<<<1, 32, 0, s>>>(100000);
    cudaEventRecord(e0, s);
    k_empty<BYTES><<<148, threads, smem, s>>>(a, buf);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 5) {
      tot += ms;
      ++n;
    }
  }
  printf("params %5d B  threads %4d  smem %6d B : %.2f us  (%s)\n", BYTES, threads, smem, 1000 * tot / n,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned* buf;
  cudaMalloc(&buf, 1 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int smem : {16, 3 * 65536}) {
    for (int threads : {128, 512}) {
      run<16>(threads, smem, s, buf);
      run<512>(threads, smem, s, buf);
      run<2816>(threads, smem, s, buf);
      run<1024>(threads, smem, s, buf);
    }
  }
}
