// fp64_rate.cu — DADD/DFMA latency and throughput per SM on this part (measurement tool).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/fp64_rate tools/micro/fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, int n, double x) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, x);
  long long t1 = clock64();
  if (threadIdx.x == 0) printf("DADD dependent latency: %.1f cycles\n", (double)(t1 - t0) / n);
  out[threadIdx.x] = a;
}
template <int CH>
__global__ void thr(double* out, int n, double x) {
  double a[CH];
  for (int c = 0; c < CH; ++c) a[c] = x + c;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = __fma_rn(a[c], x, 1.0);
  double s = 0;
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* d;
  cudaMalloc(&d, 1 << 24);
  lat<<<1, 32>>>(d, 4096, 1.0);
  cudaDeviceSynchronize();
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {256, 1024}) {
    const int n = 4096;
    thr<8><<<sms, threads>>>(d, n, 1.0000001);
    cudaEventRecord(a);
    thr<8><<<sms, threads>>>(d, n, 1.0000001);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fmas = (double)sms * threads * n * 8;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("DFMA throughput (%d thr/SM): %.2f T/s = %.1f per clk per SM at %.0f MHz (max clock)\n", threads,
           fmas / (ms * 1e-3) / 1e12, fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
  }
  return 0;
}
