// Which kernel features limit occupancy to one CTA per SM on sm_100a? (cudaOccupancy queries only)
#include <cstdio>
#include <cstdint>
__global__ void k_plain(int* p) { if (p) p[threadIdx.x] = 1; }
__global__ void k_mbar(int* p) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
  __syncthreads();
  if (p) p[threadIdx.x] = 1;
}
__global__ void k_tmem(int* p) {
  __shared__ uint32_t holder;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((unsigned)__cvta_generic_to_shared(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(holder));
  if (p) p[threadIdx.x] = 1;
}
__global__ void k_pdl(int* p) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p) p[threadIdx.x] = 1;
}
__global__ void k_cluster_sync(int* p) {
  asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
  if (p) p[threadIdx.x] = 1;
}
int main() {
  const void* ks[] = {(const void*)k_plain, (const void*)k_mbar, (const void*)k_tmem, (const void*)k_pdl, (const void*)k_cluster_sync};
  const char* nm[] = {"plain", "mbarrier", "tcgen05.alloc", "griddepcontrol", "barrier.cluster"};
  for (int i = 0; i < 5; ++i) {
    int b = -1;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ks[i], 192, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, ks[i]);
    printf("%-16s blocks/SM %d (%s) regs %d\n", nm[i], b, cudaGetErrorString(e), fa.numRegs);
  }
}
