// Per-SM L2 -> SMEM throughput: cp.async.bulk rings (16 KiB x 12 stages, one CTA per SM) over an
// L2-resident buffer, grids of 48 / 96 / 148 CTAs, PDL-chained launches (no dependency wait).
// Question answered: can 96 CTAs pull W* from L2 at > 80 GB/s each (decode kernel, K4)?
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int STAGE, int S>
__global__ void __launch_bounds__(128) bulk_kernel(const uint8_t* __restrict__ p, size_t per, unsigned* out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[S];
  const uint8_t* base = p + per * blockIdx.x;
  int nst = (int)(per / STAGE);
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&full[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  auto issue = [&](int t) {
    int s = t % S; size_t off = (size_t)t * STAGE;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s])), "r"(STAGE));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su32(sm + s * STAGE)), "l"(base + off), "r"(STAGE), "r"(su32(&full[s])) : "memory");
  };
  if (threadIdx.x == 0) for (int t = 0; t < nst && t < S; ++t) issue(t);
  uint32_t acc = 0;
  for (int t = 0; t < nst; ++t) {
    int s = t % S; uint32_t ph = (t / S) & 1;
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" :: "r"(su32(&full[s])), "r"(ph) : "memory");
    acc ^= reinterpret_cast<const uint32_t*>(sm + s * STAGE)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && t + S < nst) issue(t + S);
  }
  if (acc == 0x12345678u) out[0] = acc;
}
template <typename K, typename... A>
void launch_pdl(K k, int grid, int block, size_t smem, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(block); cfg.dynamicSmemBytes = smem; cfg.stream = 0;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}
int main() {
  const size_t per = 512 << 10;  // bytes per CTA (the decode kernel's per-CTA W* slice at S = 2)
  uint8_t* buf; cudaMalloc(&buf, 148 * per); cudaMemset(buf, 1, 148 * per);
  unsigned* out; cudaMalloc(&out, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(bulk_kernel<16384, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
  cudaFuncSetAttribute(bulk_kernel<32768, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  for (int grid : {16, 48, 96, 120, 148}) {
    for (int v = 0; v < 2; ++v) {
      auto f = [&]() { if (v == 0) launch_pdl(bulk_kernel<16384, 12>, grid, 128, 12 * 16384, (const uint8_t*)buf, per, out);
                       else launch_pdl(bulk_kernel<32768, 6>, grid, 128, 6 * 32768, (const uint8_t*)buf, per, out); };
      for (int i = 0; i < 20; ++i) f();
      cudaEventRecord(a); for (int i = 0; i < 200; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); double us = ms * 1e3 / 200;
      printf("L2-resident %s grid=%3d: %6.2f us/launch  %6.1f GB/s per CTA  %7.0f GB/s total (%s)\n", v ? "32Kx6 " : "16Kx12", grid, us,
             per / us / 1e3, grid * per / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
