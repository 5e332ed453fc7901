// host_cost.cu — host-side cost per decode call (config 2, M = 1) through the C ABI, against a bare
// cudaLaunchKernelEx of an empty kernel with the same launch attributes (cluster of 2, PDL).
// Measurement tool only.  build (after python -m paper_2407_09577_b200.build):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/micro/host_cost \
//        tools/micro/host_cost.cu -L paper_2407_09577_b200 -lflashnorm -Xlinker -rpath=$PWD/paper_2407_09577_b200
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include "flashnorm.h"
#include <cuda.h>

__global__ void __cluster_dims__(2, 1, 1) empty_k() {}
__global__ void empty_big(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1, const float* p0,
                          void* p1, int a, int b, int c, float d, float e, int f, int g, int h, const float* p2,
                          int4 r0, int4 r1, int4 r2, int i, int j, int k, const void* p3, const void* p4) {}

int main() {
  const int K = 4096, N = 6144, M = 1, R = 4000;
  void *a, *w, *z;
  cudaMalloc(&a, (size_t)16 * K * 2);
  cudaMalloc(&w, (size_t)N * K * 2);
  cudaMalloc(&z, (size_t)16 * N * 2);
  cudaMemset(a, 0, (size_t)16 * K * 2);
  cudaMemset(w, 0, (size_t)N * K * 2);
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int i = 0; i < 50; ++i)
    flashnorm_linear_ws(a, w, nullptr, M, K, N, 1e-5f, 0.5f, FN_RMSNORM, FN_BF16, z, FN_PATH_AUTO, nullptr, 0, st);
  cudaStreamSynchronize(st);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < R; ++i)
    flashnorm_linear_ws(a, w, nullptr, M, K, N, 1e-5f, 0.5f, FN_RMSNORM, FN_BF16, z, FN_PATH_AUTO, nullptr, 0, st);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  auto t2 = std::chrono::steady_clock::now();
  const double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / R;
  const double us_all = std::chrono::duration<double, std::micro>(t2 - t0).count() / R;
  printf("flashnorm_linear_ws (decode, M=1): %.2f us/call host, %.2f us/call incl. drain\n", us, us_all);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(96);
  cfg.blockDim = dim3(192);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int i = 0; i < 50; ++i) cudaLaunchKernelEx(&cfg, empty_k);
  cudaStreamSynchronize(st);
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < R; ++i) cudaLaunchKernelEx(&cfg, empty_k);
  t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  printf("bare cudaLaunchKernelEx (cluster 2 + PDL, empty kernel): %.2f us/call host\n",
         std::chrono::duration<double, std::micro>(t1 - t0).count() / R);
  // the decode kernel's launch shape: runtime cluster of 2, PDL, 226 KiB dynamic SMEM, ~400 B of params
  cudaFuncSetAttribute(empty_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 231488);
  cudaLaunchAttribute at2[2];
  at2[0] = at[0];
  at2[1].id = cudaLaunchAttributeClusterDimension;
  at2[1].val.clusterDim.x = 2;
  at2[1].val.clusterDim.y = 1;
  at2[1].val.clusterDim.z = 1;
  cfg.attrs = at2;
  cfg.numAttrs = 2;
  cfg.dynamicSmemBytes = 231488;
  CUtensorMap m{};
  const float* fp = nullptr;
  void* vp = nullptr;
  int4 r{};
  for (int i = 0; i < 50; ++i) cudaLaunchKernelEx(&cfg, empty_big, m, m, fp, vp, 1, 2, 3, 1.f, 1.f, 1, 1, 1, fp, r, r, r, 1, 1, 1, (const void*)vp, (const void*)vp);
  cudaStreamSynchronize(st);
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < R; ++i)
    cudaLaunchKernelEx(&cfg, empty_big, m, m, fp, vp, 1, 2, 3, 1.f, 1.f, 1, 1, 1, fp, r, r, r, 1, 1, 1, (const void*)vp, (const void*)vp);
  t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  printf("bare launch, decode shape (runtime cluster 2 + PDL + 226 KiB dyn SMEM + ~400 B params): %.2f us/call host (%s)\n",
         std::chrono::duration<double, std::micro>(t1 - t0).count() / R, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
