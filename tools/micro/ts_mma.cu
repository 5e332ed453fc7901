// ts_mma.cu — tcgen05.mma with the A operand in TENSOR MEMORY (".kind::f16 [d], [a_tmem], b_desc"):
// checks the layout (one A row per TMEM lane, 2 bf16 per 32-bit column, k ascending, written with
// tcgen05.st 32x32b) against a host matmul, then measures its issue rate for M = 128, N = 16
// (the decode shape: W* as A, 16 tokens as B from SMEM).  Measurement tool only.  build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_09577_b200/csrc -o tools/micro/ts_mma tools/micro/ts_mma.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#define FN_DEVICE __device__ __forceinline__
#include "common.cuh"
using namespace fn;

FN_DEVICE void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
FN_DEVICE void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  tmem_wait_ld();
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// A [128][64] bf16 (one 64-k stage of W* rows), B [16][64] bf16 tokens -> D [128][16] fp32
__global__ void __launch_bounds__(128, 1) ts_check(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int iters,
                                                   long long* cyc) {
  __shared__ __align__(1024) uint8_t sB[2048];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t holder;
  const int t = threadIdx.x, warp = t >> 5;
  // B in SW128 K-major: row r's 16-byte chunk c at r*128 + ((c ^ (r & 7)) * 16)
  for (int i = t; i < 16 * 8; i += 128) {
    const int r = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sB + r * 128 + ((c ^ (r & 7)) * 16)) = reinterpret_cast<const uint4*>(B + r * 64)[c];
  }
  fence_proxy_async_smem();
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&holder, 256); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  // A row t -> TMEM lane t, columns [128, 160): 2 bf16 per column, k ascending
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = reinterpret_cast<const uint32_t*>(A + t * 64)[i];
  tmem_st_32x32b_x32(tm + lane_base + 128, r);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint32_t idesc = make_idesc_bf16(128, 16);
    const uint64_t bd = make_sw128_desc(smem_u32(sB));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int kk = 0; kk < 4; ++kk) umma_ts(tm, tm + 128 + 8 * kk, bd + 2 * kk, idesc, (it | kk) != 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  float v[16];
  tmem_ld16(tm + lane_base + 0, v);
  if (blockIdx.x == 0)
    for (int n = 0; n < 16; ++n) D[t * 16 + n] = v[n];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 256); }
}

int main() {
  std::vector<__nv_bfloat16> hA(128 * 64), hB(16 * 64);
  std::vector<float> fA(128 * 64), fB(16 * 64);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 9) & 0xFFFF) / 32768.0f - 1.0f; };
  for (int i = 0; i < 128 * 64; ++i) { hA[i] = __float2bfloat16(rnd()); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < 16 * 64; ++i) { hB[i] = __float2bfloat16(rnd()); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB; float* dD; long long* dc;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dD, 128 * 16 * 4); cudaMalloc(&dc, 160 * 8);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  ts_check<<<1, 128>>>(dA, dB, dD, 1, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("check: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> hD(128 * 16);
  cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      double ref = 0;
      for (int k = 0; k < 64; ++k) ref += (double)fA[m * 64 + k] * fB[n * 64 + k];
      maxerr = fmax(maxerr, fabs(ref - hD[m * 16 + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("TS MMA layout check (A in TMEM, one row per lane, 2 bf16 per column): max |err| %.3g (max |ref| %.3g) -> %s\n",
         maxerr, maxref, maxerr < 1e-3 * maxref ? "MATCH" : "MISMATCH");
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  ts_check<<<sms, 128>>>(dA, dB, dD, iters, dc);
  cudaDeviceSynchronize();
  std::vector<long long> hc(sms);
  cudaMemcpy(hc.data(), dc, sms * 8, cudaMemcpyDeviceToHost);
  double sum = 0; for (auto x : hc) sum += x;
  const double per = sum / sms / (iters * 4.0);
  printf("TS MMA M=128 N=16 K=16: %.1f cycles/MMA = %.1f W* bytes/clk/SM (A from TMEM)\n", per, 4096.0 / per);
  return 0;
}
