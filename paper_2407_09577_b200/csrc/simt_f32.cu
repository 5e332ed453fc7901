// simt_f32.cu — K5: the fp32 FlashNorm linear (FFMA only, no TF32 — reading c13).
//
//   rms/ln : z = fma( sum_k a_k W*t[j][k],  rsqrt(sum_k a_k^2 / K + eps),  c*_j )
//   dyt    : z = sum_k tanhf(alpha a_k) W*t[j][k] + c*_j                           reading c10
//   none   : z = sum_k a_k W*t[j][k] + c*_j
//
// Tiny shapes (BASELINE config 1: M=8, K=64, N=64) are latency-bound; one warp
// per output element, lanes split K (coalesced along the K-contiguous W*t row),
// the RMS of the row is reduced by the same warp alongside the dot product
// (the "parallel" RMS of PAPER.md:20 at warp granularity).  Accurate tanhf.
#include "common.cuh"
#include "kernels.h"

namespace fn {

template <int MODE>
__global__ void __launch_bounds__(256)
    linear_f32_kernel(const float* __restrict__ a, const float* __restrict__ Wt, const float* __restrict__ cstar,
                      float* __restrict__ z, int M, int K, int N, float eps, float alpha) {
  const int lane = threadIdx.x & 31;
  const int n = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int m = blockIdx.y;
  if (n >= N || m >= M) return;
  const float* arow = a + (size_t)m * K;
  const float* wrow = Wt + (size_t)n * K;
  float dot = 0.f, ssq = 0.f;
  for (int k = lane; k < K; k += 32) {
    float x = arow[k];
    if (MODE == MODE_RMS) ssq = fmaf(x, x, ssq);
    if (MODE == MODE_DYT) x = tanhf(alpha * x);
    dot = fmaf(x, wrow[k], dot);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    dot += __shfl_xor_sync(0xffffffffu, dot, off);
    if (MODE == MODE_RMS) ssq += __shfl_xor_sync(0xffffffffu, ssq, off);
  }
  if (lane == 0) {
    const float cb = cstar != nullptr ? cstar[n] : 0.f;
    float r = 1.f;
    if (MODE == MODE_RMS) r = 1.0f / sqrtf(ssq / (float)K + eps);
    z[(size_t)m * N + n] = fmaf(dot, r, cb);
  }
}

cudaError_t launch_linear_f32(const float* a, const float* Wt, const float* cstar, float* z, int M, int K, int N,
                              float eps, float alpha, int mode, cudaStream_t stream) {
  const dim3 grid((unsigned)((N + 7) / 8), (unsigned)M);
  if (mode == MODE_RMS) linear_f32_kernel<MODE_RMS><<<grid, 256, 0, stream>>>(a, Wt, cstar, z, M, K, N, eps, alpha);
  else if (mode == MODE_DYT) linear_f32_kernel<MODE_DYT><<<grid, 256, 0, stream>>>(a, Wt, cstar, z, M, K, N, eps, alpha);
  else linear_f32_kernel<MODE_NONE><<<grid, 256, 0, stream>>>(a, Wt, cstar, z, M, K, N, eps, alpha);
  return cudaGetLastError();
}

}  // namespace fn
