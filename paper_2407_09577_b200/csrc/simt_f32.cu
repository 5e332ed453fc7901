// simt_f32.cu — K5: the fp32 FlashNorm linear (FFMA only, no TF32 — reading c13).
//
//   rms/ln : z = fma( sum_k a_k W*t[j][k],  rsqrt(sum_k a_k^2 / K + eps),  c*_j )
//   dyt    : z = sum_k tanhf(alpha a_k) W*t[j][k] + c*_j                           reading c10
//   none   : z = sum_k a_k W*t[j][k] + c*_j
//   ln (u != NULL, rms mode): z = fma( dot - mu u_j, rsqrt(var + eps), c*_j ), mu = mean(a),
//            var = mean((a - a0)^2) - mean(a - a0)^2 (shift a0 = a_0): LayerNorm deferred past
//            the contraction (NEXT-4, reading c29)
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
                      float* __restrict__ z, int M, int K, int N, float eps, float alpha,
                      const float* __restrict__ u) {
  const int lane = threadIdx.x & 31;
  const int n = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int m = blockIdx.y;
  if (n >= N || m >= M) return;
  const float* arow = a + (size_t)m * K;
  const float* wrow = Wt + (size_t)n * K;
  float dot = 0.f, ssq = 0.f, s1 = 0.f;
  const bool ln = MODE == MODE_RMS && u != nullptr;
  const float a0 = ln ? arow[0] : 0.f;
  for (int k = lane; k < K; k += 32) {
    float x = arow[k];
    if (MODE == MODE_RMS) {
      const float d = x - a0;
      ssq = fmaf(d, d, ssq);
      s1 += d;
    }
    if (MODE == MODE_DYT) x = tanhf(alpha * x);
    dot = fmaf(x, wrow[k], dot);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    dot += __shfl_xor_sync(0xffffffffu, dot, off);
    if (MODE == MODE_RMS) ssq += __shfl_xor_sync(0xffffffffu, ssq, off);
    if (MODE == MODE_RMS && ln) s1 += __shfl_xor_sync(0xffffffffu, s1, off);
  }
  if (lane == 0) {
    const float cb = cstar != nullptr ? cstar[n] : 0.f;
    float r = 1.f;
    if (MODE == MODE_RMS && ln) {
      const float m1 = s1 / (float)K;
      const float var = fmaxf(ssq / (float)K - m1 * m1, 0.0f);
      r = 1.0f / sqrtf(var + eps);
      dot = fmaf(-(a0 + m1), u[n], dot);
    } else if (MODE == MODE_RMS) {
      r = 1.0f / sqrtf(ssq / (float)K + eps);
    }
    z[(size_t)m * N + n] = fmaf(dot, r, cb);
  }
}

cudaError_t launch_linear_f32(const float* a, const float* Wt, const float* cstar, float* z, int M, int K, int N,
                              float eps, float alpha, int mode, cudaStream_t stream, const float* u) {
  const dim3 grid((unsigned)((N + 7) / 8), (unsigned)M);
  if (mode == MODE_RMS) linear_f32_kernel<MODE_RMS><<<grid, 256, 0, stream>>>(a, Wt, cstar, z, M, K, N, eps, alpha, u);
  else if (mode == MODE_DYT) linear_f32_kernel<MODE_DYT><<<grid, 256, 0, stream>>>(a, Wt, cstar, z, M, K, N, eps, alpha, u);
  else linear_f32_kernel<MODE_NONE><<<grid, 256, 0, stream>>>(a, Wt, cstar, z, M, K, N, eps, alpha, u);
  return cudaGetLastError();
}

}  // namespace fn
