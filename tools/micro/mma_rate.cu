// mma_rate.cu — tcgen05.mma (cta_group::1, kind::f16, SS) issue rate vs shape, one CTA per SM, all SMs:
// how many W* bytes per clock the tensor core consumes from SMEM when W* is the A operand (decode
// today: M = 128 W* rows, N = 16 tokens) vs the B operand (M = 128 or 64 token rows, N = 64..256 W* rows).
// Measurement tool only.  build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_09577_b200/csrc -o tools/micro/mma_rate tools/micro/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define FN_DEVICE __device__ __forceinline__
#include "common.cuh"
using namespace fn;

__global__ void __launch_bounds__(128, 1) k(int M, int N, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;              // 128 rows x 64 k bf16, SW128 (16 KiB)
  uint8_t* sB = sm + 16384;      // 256 rows x 64 k bf16, SW128 (32 KiB)
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_holder;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) {
    tmem_alloc(&tmem_holder, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(M, N);
    const uint64_t ad = make_sw128_desc(smem_u32(sA)), bd = make_sw128_desc(smem_u32(sB));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (it | kk) != 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  const int smem = 49152 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct { int M, N; const char* what; int wbytes; } cfg[] = {
      {128, 16, "A = W* (128 rows), B = 16 tokens   [decode today]", 128 * 16 * 2},
      {128, 32, "A = W* (128 rows), B = 32 tokens", 128 * 16 * 2},
      {128, 64, "A = 128 tokens,    B = W* 64 rows", 64 * 16 * 2},
      {128, 128, "A = 128 tokens,    B = W* 128 rows", 128 * 16 * 2},
      {128, 256, "A = 128 tokens,    B = W* 256 rows", 256 * 16 * 2},
      {64, 128, "A = 64 tokens,     B = W* 128 rows", 128 * 16 * 2},
      {64, 256, "A = 64 tokens,     B = W* 256 rows", 256 * 16 * 2},
  };
  const int iters = 4096;
  for (auto& c : cfg) {
    k<<<sms, 128, smem>>>(c.M, c.N, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("M=%d N=%d: %s\n", c.M, c.N, cudaGetErrorString(e)); return 1; }
    long long h[256];
    cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double mx = 0, sum = 0;
    for (int i = 0; i < sms; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    const double per = sum / sms / (iters * 4.0);
    printf("M=%3d N=%3d %-50s %6.1f cycles/MMA  %6.1f W* B/clk/SM  (%.0f flop/clk/SM)\n", c.M, c.N, c.what, per,
           c.wbytes / per, 2.0 * c.M * c.N * 16 / per);
  }
  return 0;
}
