// host_cost.cu — host-side cost per decode call (config 2, M = 1) through the C ABI, against a bare
// cudaLaunchKernelEx of an empty kernel with the same launch attributes (cluster of 2, PDL).
// Measurement tool only.  build (after python -m paper_2407_09577_b200.build):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/micro/host_cost \
//        tools/micro/host_cost.cu -L paper_2407_09577_b200 -lflashnorm -Xlinker -rpath=$PWD/paper_2407_09577_b200
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include "flashnorm.h"

__global__ void __cluster_dims__(2, 1, 1) empty_k() {}

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
  return 0;
}
