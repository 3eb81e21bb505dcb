// NVLS multicast probe (one process, every visible GPU): is CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED
// set, can a multicast object span the GPUs, and does multimem.st from GPU 0 land in every
// GPU's bound memory? Also times a multimem.st broadcast against N-1 unicast peer stores.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe.bin tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s = nullptr; cuGetErrorString(r, &s); \
  printf("CU error %d (%s) at line %d: %s\n", (int)r, s ? s : "?", __LINE__, #x); return 1; } } while (0)
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_mc_store(float* mc, uint64_t n4, float v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    float* p = mc + 4 * i;
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
  }
}
__global__ void k_uni_store(float4* const* dst, int nd, uint64_t n4, float v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < nd; ++d) dst[d][i] = make_float4(v, v, v, v);
}

int main() {
  CU(cuInit(0));
  int n = 0;
  CU(cuDeviceGetCount(&n));
  printf("devices %d\n", n);
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    CU(cuDeviceGet(&dev, d));
    int mc = 0;
    CU(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("dev %d multicast_supported %d\n", d, mc);
  }
  if (n < 2) return 0;
  const size_t bytes = 256ull << 20;
  CUmulticastObjectProp prop = {};
  prop.numDevices = n;
  prop.size = bytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("multicast granularity %zu\n", gran);
  prop.size = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mch;
  CU(cuMulticastCreate(&mch, &prop));
  std::vector<CUdevice> devs(n);
  for (int d = 0; d < n; ++d) {
    CU(cuDeviceGet(&devs[d], d));
    CU(cuMulticastAddDevice(mch, devs[d]));
  }
  std::vector<CUdeviceptr> uc(n);
  std::vector<CUcontext> ctx(n);
  for (int d = 0; d < n; ++d) {
    CU(cuDevicePrimaryCtxRetain(&ctx[d], devs[d]));
    CU(cuCtxSetCurrent(ctx[d]));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g2 = 0;
    CU(cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    const size_t sz = (prop.size + g2 - 1) / g2 * g2;
    CUmemGenericAllocationHandle h;
    CU(cuMemCreate(&h, sz, &ap, 0));
    CU(cuMulticastBindMem(mch, 0, h, 0, prop.size, 0));
    CU(cuMemAddressReserve(&uc[d], sz, g2, 0, 0));
    CU(cuMemMap(uc[d], sz, 0, h, 0));
    std::vector<CUmemAccessDesc> ads(n);  // every GPU may access it (the unicast baseline)
    for (int q = 0; q < n; ++q) {
      ads[q] = {};
      ads[q].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ads[q].location.id = q;
      ads[q].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    CU(cuMemSetAccess(uc[d], sz, ads.data(), n));
    CU(cuMemsetD8(uc[d], 0, sz));
  }
  // map the multicast object on device 0
  CU(cuCtxSetCurrent(ctx[0]));
  CUdeviceptr mcva;
  CU(cuMemAddressReserve(&mcva, prop.size, gran, 0, 0));
  CU(cuMemMap(mcva, prop.size, 0, mch, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(mcva, prop.size, &ad, 1));
  const uint64_t n4 = bytes / 16;
  k_mc_store<<<148, 512>>>((float*)mcva, n4, 3.5f);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  for (int d = 0; d < n; ++d) {
    CU(cuCtxSetCurrent(ctx[d]));
    float h[4];
    CU(cuMemcpyDtoH(h, uc[d] + bytes - 16, 16));
    printf("dev %d tail value %.2f (want 3.50)\n", d, h[0]);
  }
  CU(cuCtxSetCurrent(ctx[0]));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int ctas : {32, 64, 148, 296}) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      CK(cudaEventRecord(e0));
      k_mc_store<<<ctas, 512>>>((float*)mcva, n4, (float)rep);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep) best = ms < best ? ms : best;
    }
    printf("NVLS {\"mode\": \"multimem.st\", \"ctas\": %d, \"MB\": %.0f, \"ms\": %.4f, \"GBps_source\": %.1f, \"GBps_delivered_peers\": %.1f}\n", ctas,
           bytes / 1e6, best, bytes / best / 1e6, bytes * (n - 1) / best / 1e6);
  }
  // unicast baseline: device 0 stores the same bytes into every peer's memory (peer access)
  float4** dl;
  CK(cudaMalloc(&dl, sizeof(float4*) * n));
  std::vector<float4*> hd(n - 1);
  for (int d = 1; d < n; ++d) hd[d - 1] = (float4*)uc[d];
  CK(cudaMemcpy(dl, hd.data(), sizeof(float4*) * (n - 1), cudaMemcpyHostToDevice));
  for (int ctas : {64, 148}) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      CK(cudaEventRecord(e0));
      k_uni_store<<<ctas, 512>>>(dl, n - 1, n4, (float)rep);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep) best = ms < best ? ms : best;
    }
    printf("NVLS {\"mode\": \"unicast x%d\", \"ctas\": %d, \"MB\": %.0f, \"ms\": %.4f, \"GBps_source\": %.1f, \"GBps_delivered_peers\": %.1f}\n", n - 1, ctas,
           bytes / 1e6, best, bytes * (n - 1) / best / 1e6, bytes * (n - 1) / best / 1e6);
  }
  return 0;
}
