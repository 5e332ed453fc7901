// mc_probe.cu — can this process create an NVLink-SHARP (NVLS) multicast object over its one GPU,
// bind memory to it, and store through the multicast address with multimem.st?  (measurement /
// capability probe; the multi-GPU gather uses the same driver calls across ranks)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro/mc_probe tools/micro/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %d (%s)\n", #x, (int)r, s); return 1; } } while (0)
__global__ void mc_store(uint32_t* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint32_t v = 0x3f803f80u + (uint32_t)i;
    asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(mc + i), "r"(v) : "memory");
  }
}
int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  int mc = 0;
  CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("MULTICAST_SUPPORTED = %d\n", mc);
  if (!mc) return 0;
  CUmulticastObjectProp prop = {};
  prop.numDevices = 1;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  prop.size = 2 << 20;
  CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  prop.size = (prop.size + gran - 1) / gran * gran;
  printf("granularity %zu size %zu\n", gran, prop.size);
  CUmemGenericAllocationHandle mch;
  {
    const unsigned long long hts[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC, 0};
    CUresult r = CUDA_ERROR_UNKNOWN;
    for (int nd = 1; nd <= 2 && r != CUDA_SUCCESS; ++nd)
      for (unsigned long long ht : hts) {
        prop.numDevices = nd;
        prop.handleTypes = ht;
        size_t g2 = 0;
        cuMulticastGetGranularity(&g2, &prop, CU_MULTICAST_GRANULARITY_MINIMUM);
        r = cuMulticastCreate(&mch, &prop);
        printf("cuMulticastCreate(numDevices=%d, handleTypes=%llu, min gran %zu) -> %d\n", nd, ht, g2, (int)r);
        if (r == CUDA_SUCCESS) break;
      }
    if (r != CUDA_SUCCESS) return 1;
    if (prop.numDevices != 1) { printf("only numDevices > 1 works: a single process cannot complete it\n"); return 0; }
  }
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)prop.handleTypes;
  CUmemGenericAllocationHandle mh;
  CK(cuMemCreate(&mh, prop.size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, mh, 0, prop.size, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0));
  CK(cuMemMap(uc, prop.size, 0, mh, 0));
  CK(cuMemAddressReserve(&mcp, prop.size, gran, 0, 0));
  CK(cuMemMap(mcp, prop.size, 0, mch, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, prop.size, &ad, 1));
  CK(cuMemSetAccess(mcp, prop.size, &ad, 1));
  const int n = 1 << 16;
  cudaMemset((void*)uc, 0, n * 4);
  mc_store<<<n / 256, 256>>>((uint32_t*)mcp, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("multimem.st kernel: %s\n", cudaGetErrorString(e));
  uint32_t h[4];
  cudaMemcpy(h, (void*)uc, 16, cudaMemcpyDeviceToHost);
  printf("unicast view after multimem.st: %08x %08x %08x %08x (expect 3f803f80 3f803f81 ...)\n", h[0], h[1], h[2], h[3]);
  return 0;
}
