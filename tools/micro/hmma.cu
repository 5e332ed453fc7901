// mma.sync.m16n8k16 bf16 -> f32 on this GPU: dependent-chain latency and per-SM throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int CH>
__global__ void k(int iters, float* out, long long* cyc) {
  uint32_t a = threadIdx.x * 0x00010001u;
  float d[CH][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) mma(d[c], a, a + 1, a + 2, a + 3, a + 4, a + 5);
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 1024 * 4 * 4); long long* cyc; cudaMalloc(&cyc, 8);
  const int iters = 4096;
  auto run = [&](const char* name, auto kern, int ch, int warps) {
    kern<<<1, 32, 0>>>(16, out, cyc); cudaDeviceSynchronize();
    kern<<<1, 32 * warps>>>(iters, out, cyc); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-10s warps/SM=%2d: %.1f cycles per mma per warp-chain step, %.2f mma/clk/SM\n", name, warps,
           (double)c / iters, (double)iters * ch * warps / c);
  };
  run("1 chain", k<1>, 1, 1);
  run("4 chains", k<4>, 4, 1);
  run("8 chains", k<8>, 8, 1);
  run("1 chain", k<1>, 1, 4);
  run("4 chains", k<4>, 4, 4);
  run("4 chains", k<4>, 4, 16);
  run("1 chain", k<1>, 1, 16);
  run("8 chains", k<8>, 8, 16);
}
