// NVLink peer-copy probe: per-SM and aggregate throughput of the ways a CTA can move data
// between two GPUs (device 0 runs the kernels; device 1 holds the peer buffer).
//   st     : ld.global.v4 local -> st.global.v4 peer (push by registers)
//   bulk   : cp.async.bulk local -> smem -> cp.async.bulk peer (push by TMA; S stages in flight)
//   ld     : ld.global.v4 peer -> st.global.v4 local (pull by registers)
//   bulkld : cp.async.bulk peer -> smem -> cp.async.bulk local (pull by TMA)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_probe.bin tools/p2p_probe.cu
// ./tools/p2p_probe.bin   (prints one line per method x CTA count x stage count)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512) k_st(const float4* __restrict__ src, float4* dst, uint64_t n4) {
  const uint64_t per = (n4 / gridDim.x) & ~7ull;
  const float4* s = src + per * blockIdx.x;
  float4* d = dst + per * blockIdx.x;
  for (uint64_t i = threadIdx.x; i < per; i += 4 * blockDim.x) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * blockDim.x < per) v[u] = s[i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * blockDim.x < per) d[i + u * blockDim.x] = v[u];
  }
}

// one thread drives a ring of `stages` chunks of `chunk` bytes: load (bulk, mbarrier) then store (bulk group)
__global__ void k_bulk(const uint8_t* src, uint8_t* dst, uint64_t bytes, uint32_t chunk, uint32_t stages) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x != 0) return;
  const uint64_t per = (bytes / gridDim.x) & ~(uint64_t)(chunk - 1);  // (chunks are powers of two)
  const uint8_t* s = src + per * blockIdx.x;
  uint8_t* d = dst + per * blockIdx.x;
  for (uint32_t i = 0; i < stages; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t nchunks = per / chunk;
  uint32_t phase[16] = {0};
  auto load = [&](uint64_t c) {
    const uint32_t st = c % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(sm + (size_t)st * chunk)), "l"(s + c * chunk), "r"(chunk), "r"(smem_u32(&bar[st])) : "memory");
  };
  for (uint64_t c = 0; c < nchunks && c < stages; ++c) load(c);
  for (uint64_t c = 0; c < nchunks; ++c) {
    const uint32_t st = c % stages;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(smem_u32(&bar[st])), "r"(phase[st]) : "memory");
    phase[st] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + c * chunk),
                 "r"(smem_u32(sm + (size_t)st * chunk)), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the previous chunk's stage is reloaded once its store has read it (all groups but the
    // newest), so one store's read overlaps the next chunk's wait
    if (c >= 1 && c - 1 + stages < nchunks) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(c - 1 + stages);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  printf("peer access 0->1: %d\n", can);
  const uint64_t bytes = 512ull << 20;
  uint8_t *loc, *rem;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&rem, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&loc, bytes));
  CK(cudaMemset(loc, 1, bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int ctas_list[] = {1, 2, 4, 8, 16, 32, 64, 148};
  for (int method = 0; method < 4; ++method) {
    const char* name[] = {"st", "bulk", "ld", "bulkld"};
    for (int ctas : ctas_list) {
      std::vector<std::pair<uint32_t, uint32_t>> cfgs;
      if (method == 0 || method == 2) cfgs.push_back({0, 0});
      else for (uint32_t chunk : {16384u, 32768u, 65536u}) for (uint32_t st : {2u, 3u, 6u}) if ((uint64_t)chunk * st <= 196608) cfgs.push_back({chunk, st});
      for (auto [chunk, st] : cfgs) {
        const uint64_t b = std::min<uint64_t>(bytes, (uint64_t)ctas * (8ull << 20));
        const uint8_t* src = method < 2 ? loc : rem;
        uint8_t* dst = method < 2 ? rem : loc;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaEventRecord(e0));
          if (method == 0 || method == 2)
            k_st<<<ctas, 512>>>((const float4*)src, (float4*)dst, b / 16);
          else
            k_bulk<<<ctas, 32, chunk * st>>>(src, dst, b, chunk, st);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          CK(cudaGetLastError());
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (rep) best = std::min(best, ms);
        }
        printf("P2P {\"method\": \"%s\", \"ctas\": %d, \"chunk\": %u, \"stages\": %u, \"MB\": %.0f, \"GBps\": %.1f, \"GBps_per_cta\": %.2f}\n",
               name[method], ctas, chunk, st, b / 1e6, b / best / 1e6, b / best / 1e6 / ctas);
      }
    }
  }
  // bidirectional: both GPUs push to each other at the same time (the N=2 exchange pattern)
  {
    uint8_t *loc1, *rem0;  // device 1's source, device 0's receive buffer
    CK(cudaSetDevice(1));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaMalloc(&loc1, bytes));
    CK(cudaMemset(loc1, 2, bytes));
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaEvent_t f0, f1;
    CK(cudaEventCreate(&f0));
    CK(cudaEventCreate(&f1));
    CK(cudaSetDevice(0));
    CK(cudaMalloc(&rem0, bytes));
    for (int method = 0; method < 2; ++method)
      for (int ctas : {32, 64, 148}) {
        float best0 = 1e30f, best1 = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaSetDevice(0));
          CK(cudaDeviceSynchronize());
          CK(cudaSetDevice(1));
          CK(cudaDeviceSynchronize());
          for (int dev = 0; dev < 2; ++dev) {
            CK(cudaSetDevice(dev));
            const uint8_t* src = dev == 0 ? loc : loc1;
            uint8_t* dst = dev == 0 ? rem : rem0;
            CK(cudaEventRecord(dev == 0 ? e0 : f0));
            if (method == 0)
              k_st<<<ctas, 512>>>((const float4*)src, (float4*)dst, bytes / 16);
            else
              k_bulk<<<ctas, 32, 65536 * 3>>>(src, dst, bytes, 65536, 3);
            CK(cudaEventRecord(dev == 0 ? e1 : f1));
          }
          float m0, m1;
          CK(cudaSetDevice(0));
          CK(cudaEventSynchronize(e1));
          CK(cudaEventElapsedTime(&m0, e0, e1));
          CK(cudaSetDevice(1));
          CK(cudaEventSynchronize(f1));
          CK(cudaEventElapsedTime(&m1, f0, f1));
          CK(cudaGetLastError());
          if (rep) { best0 = std::min(best0, m0); best1 = std::min(best1, m1); }
        }
        printf("P2P {\"method\": \"bidir_%s\", \"ctas\": %d, \"chunk\": 65536, \"stages\": 3, \"MB\": %.0f, \"GBps\": %.1f, \"GBps_dev1\": %.1f, \"GBps_per_cta\": %.2f}\n",
               method == 0 ? "st" : "bulk", ctas, bytes / 1e6, bytes / best0 / 1e6, bytes / best1 / 1e6, bytes / best0 / 1e6 / ctas);
      }
  }
  return 0;
}
