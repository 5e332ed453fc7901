// Microbenchmark: how fast can 148 CTAs stream S bytes from HBM on this B200?
// (1) LDG.128 grid-stride with unroll, (2) cp.async.bulk into a smem ring per CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(512) ldg_kernel(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  uint32_t acc = 0;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  for (; i < n16; i += stride) acc ^= p[i].x;
  if (acc == 0x12345678u) out[0] = acc;
}
template <int STAGE, int S, int NT = 128, int SPLIT = 1, bool PDL = false, bool WAIT = false, bool LATE = false, bool STORE = false>
__global__ void __launch_bounds__(NT) bulk_kernel(const uint8_t* __restrict__ p, size_t bytes, unsigned* out) {
  if (PDL && (!LATE || threadIdx.x < 32)) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[S];
  size_t per = (bytes / gridDim.x) & ~(size_t)15;
  const uint8_t* base = p + per * blockIdx.x;
  int nst = (int)((per + STAGE - 1) / STAGE);
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&full[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  auto issue = [&](int t) {
    int s = t % S; size_t off = (size_t)t * STAGE; uint32_t b = (uint32_t)((per - off) < STAGE ? (per - off) : STAGE);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s])), "r"(b));
    const int nsplit = (b == STAGE) ? SPLIT : 1;
    for (int q = 0; q < nsplit; ++q) { uint32_t bb = b / nsplit;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su32(sm + s * STAGE + q * bb)), "l"(base + off + q * bb), "r"(bb), "r"(su32(&full[s])) : "memory"); }
  };
  if (threadIdx.x == 0) for (int t = 0; t < nst && t < S; ++t) issue(t);
  if (WAIT) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (PDL && LATE && threadIdx.x >= 32) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint32_t acc = 0;
  for (int t = 0; t < nst; ++t) {
    int s = t % S; uint32_t ph = (t / S) & 1;
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" :: "r"(su32(&full[s])), "r"(ph) : "memory");
    acc ^= reinterpret_cast<const uint32_t*>(sm + s * STAGE)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && t + S < nst) issue(t + S);
  }
  if (STORE) out[1 + blockIdx.x * NT + threadIdx.x] = acc;
  else if (acc == 0x12345678u) out[0] = acc;
}
__global__ void __launch_bounds__(512) ldg_pdl_kernel(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint32_t acc = 0;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  for (; i < n16; i += stride) acc ^= p[i].x;
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
  int sms = 148;
  for (size_t MB : {50, 200}) {
    size_t bytes = MB << 20;
    uint8_t* buf[4]; for (int i = 0; i < 4; ++i) { cudaMalloc(&buf[i], bytes); cudaMemset(buf[i], 1, bytes); }
    unsigned* out; cudaMalloc(&out, 4 * (1 + 148 * 512));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto fnc) {
      for (int i = 0; i < 10; ++i) fnc(i);
      cudaEventRecord(a); for (int i = 0; i < 200; ++i) fnc(i); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); double us = ms * 1e3 / 200;
      printf("%-28s %4zu MB: %8.2f us  %7.0f GB/s  (%s)\n", name, MB, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    run("ldg128 x8 grid=148x512", [&](int i) { ldg_kernel<<<sms, 512>>>((const uint4*)buf[i % 4], bytes / 16, out); });
    run("ldg128 x8 grid=296x512", [&](int i) { ldg_kernel<<<2 * sms, 512>>>((const uint4*)buf[i % 4], bytes / 16, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("bulk 32K x6 grid=148", [&](int i) { bulk_kernel<32768, 6><<<sms, 128, 6 * 32768>>>(buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<16384, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
    run("bulk 16K x12 grid=148", [&](int i) { bulk_kernel<16384, 12><<<sms, 128, 12 * 16384>>>(buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<65536, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    run("bulk 64K x3 grid=148", [&](int i) { bulk_kernel<65536, 3><<<sms, 128, 3 * 65536>>>(buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<65536, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
    run("bulk 64K x2 grid=148", [&](int i) { bulk_kernel<65536, 2><<<sms, 128, 2 * 65536>>>(buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<65536, 2, 512, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536 + 65536);
    run("bulk 64Kx2 512thr split8", [&](int i) { bulk_kernel<65536, 2, 512, 8><<<sms, 512, 2 * 65536 + 65536>>>(buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 4, 512, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 65536);
    run("bulk 32Kx4 512thr split8", [&](int i) { bulk_kernel<32768, 4, 512, 8><<<sms, 512, 4 * 32768 + 65536>>>(buf[i % 4], bytes, out); });
    run("PDL ldg128 x8 grid=148x512", [&](int i) { launch_pdl(ldg_pdl_kernel, sms, 512, 0, (const uint4*)buf[i % 4], bytes / 16, out); });
    run("PDL ldg128 x8 grid=296x512", [&](int i) { launch_pdl(ldg_pdl_kernel, 2 * sms, 512, 0, (const uint4*)buf[i % 4], bytes / 16, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 3, 128, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768);
    run("PDL bulk 32K x3 grid=148", [&](int i) { launch_pdl(bulk_kernel<32768, 3, 128, 1, true>, sms, 128, 3 * 32768, (const uint8_t*)buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 6, 128, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("PDL bulk 32K x6 grid=148", [&](int i) { launch_pdl(bulk_kernel<32768, 6, 128, 1, true>, sms, 128, 6 * 32768, (const uint8_t*)buf[i % 4], bytes, out); });
    run("PDL bulk 32K x3 grid=296", [&](int i) { launch_pdl(bulk_kernel<32768, 3, 128, 1, true>, 2 * sms, 128, 3 * 32768, (const uint8_t*)buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 6, 128, 1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("PDL+wait bulk 32K x6 grid=148", [&](int i) { launch_pdl(bulk_kernel<32768, 6, 128, 1, true, true>, sms, 128, 6 * 32768, (const uint8_t*)buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 3, 128, 1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768);
    run("PDL+wait bulk 32K x3 grid=296", [&](int i) { launch_pdl(bulk_kernel<32768, 3, 128, 1, true, true>, 2 * sms, 128, 3 * 32768, (const uint8_t*)buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 6, 512, 1, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("PDL+wait+late 32Kx6 512thr", [&](int i) { launch_pdl(bulk_kernel<32768, 6, 512, 1, true, true, true>, sms, 512, 6 * 32768, (const uint8_t*)buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 6, 512, 1, true, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("PDL+wait+late+store 32Kx6 512", [&](int i) { launch_pdl(bulk_kernel<32768, 6, 512, 1, true, true, true, true>, sms, 512, 6 * 32768, (const uint8_t*)buf[i % 4], bytes, out); });
    cudaFuncSetAttribute(bulk_kernel<32768, 6, 512, 1, true, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("PDL+wait+store 32Kx6 512", [&](int i) { launch_pdl(bulk_kernel<32768, 6, 512, 1, true, true, false, true>, sms, 512, 6 * 32768, (const uint8_t*)buf[i % 4], bytes, out); });
    run("empty kernel", [&](int i) { ldg_kernel<<<sms, 512>>>((const uint4*)buf[i % 4], 0, out); });
    for (int i = 0; i < 4; ++i) cudaFree(buf[i]);
  }
}
