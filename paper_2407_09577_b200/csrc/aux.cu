// aux.cu — K6 (unfused baseline normalization) and K7 (column-gather permute).
//
// K6 is a measurement comparator, not the method: Fig 1(a)'s first half,
//   rms : y = RN(a / RMSe(a) * g + b)
//   ln  : y = RN((a - mu) / RMSe(a - mu) * g + b)
//   dyt : y = RN(g * tanh(alpha a) + b)      reading c10
// written to HBM and then consumed by flashnorm_linear(mode = none) on the
// ORIGINAL W — the two-kernel variant BASELINE.json:5 asks for.
//
// K7 moves P column shards z_parts[P][M][N/P] (after an all-gather) into z[M][N].
#include "common.cuh"
#include "kernels.h"

#include <cstring>

namespace fn {

template <typename T>
FN_DEVICE float to_f(T x);
template <>
FN_DEVICE float to_f<float>(float x) { return x; }
template <>
FN_DEVICE float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
FN_DEVICE T from_f(float x);
template <>
FN_DEVICE float from_f<float>(float x) { return x; }
template <>
FN_DEVICE __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

FN_DEVICE float block_sum(float v, float* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

template <typename T, int KIND>
__global__ void __launch_bounds__(256)
    baseline_norm_kernel(const T* __restrict__ a, const float* __restrict__ g, const float* __restrict__ b, int K,
                         float eps, float alpha, T* __restrict__ y) {
  __shared__ float red[8];
  const T* row = a + (size_t)blockIdx.x * K;
  T* out = y + (size_t)blockIdx.x * K;
  float mu = 0.f, r = 1.f;
  if (KIND != 2) {
    if (KIND == 1) {
      float s = 0.f;
      for (int k = threadIdx.x; k < K; k += blockDim.x) s += to_f(row[k]);
      mu = block_sum(s, red) / (float)K;
    }
    float q = 0.f;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      const float x = to_f(row[k]) - mu;
      q = fmaf(x, x, q);
    }
    r = rsqrtf(block_sum(q, red) / (float)K + eps);
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float x = to_f(row[k]);
    float v = KIND == 2 ? tanhf(alpha * x) : (x - mu) * r;
    if (g != nullptr) v *= g[k];
    if (b != nullptr) v += b[k];
    out[k] = from_f<T>(v);
  }
}

cudaError_t launch_baseline_norm(const void* a, const float* g, const float* b, int64_t M, int64_t K, float eps,
                                 int kind, float alpha, int dtype, void* y, cudaStream_t stream) {
  const dim3 grid((unsigned)M);
#define FN_BN(T, KD)                                                                                        \
  baseline_norm_kernel<T, KD><<<grid, 256, 0, stream>>>(static_cast<const T*>(a), g, b, (int)K, eps, alpha, \
                                                        static_cast<T*>(y))
  if (dtype == 0) {
    if (kind == 0) FN_BN(__nv_bfloat16, 0);
    else if (kind == 1) FN_BN(__nv_bfloat16, 1);
    else FN_BN(__nv_bfloat16, 2);
  } else {
    if (kind == 0) FN_BN(float, 0);
    else if (kind == 1) FN_BN(float, 1);
    else FN_BN(float, 2);
  }
#undef FN_BN
  return cudaGetLastError();
}

__global__ void gather_columns_kernel(const uint4* __restrict__ parts, int64_t P, int64_t M, int64_t nl16,
                                      uint4* __restrict__ z) {
  // one thread per 16-byte chunk of z; z row m = [part 0 | part 1 | ... ]
  const int64_t total = P * M * nl16;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / (P * nl16);
    const int64_t rem = i - m * P * nl16;
    const int64_t p = rem / nl16;
    const int64_t q = rem - p * nl16;
    z[i] = parts[(p * M + m) * nl16 + q];
  }
}

cudaError_t launch_gather_columns(const void* parts, int64_t P, int64_t M, int64_t Nl, int elem_bytes, void* z,
                                  cudaStream_t stream) {
  const int64_t nl16 = Nl * elem_bytes / 16;
  const int64_t total = P * M * nl16;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  gather_columns_kernel<<<(unsigned)blocks, 256, 0, stream>>>(static_cast<const uint4*>(parts), P, M, nl16,
                                                              static_cast<uint4*>(z));
  return cudaGetLastError();
}

// Debug check behind FN_DEBUG_LAYERNORM (include/flashnorm.h, FN_LAYERNORM): the LayerNorm mode
// trusts that its input was mean-centered by a V* fold.  One CTA per row measures
// |mean(a_m)| / rms(a_m) (fp32) and folds it into a device-wide maximum (non-negative floats
// order like their bit patterns, so atomicMax on the bits is a float max).
__device__ unsigned g_ln_center_max;

template <typename T>
__global__ void __launch_bounds__(256) layernorm_center_check_kernel(const T* __restrict__ a, int K) {
  __shared__ float red[8];
  const T* row = a + (size_t)blockIdx.x * K;
  float s = 0.f, q = 0.f;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float x = to_f(row[k]);
    s += x;
    q = fmaf(x, x, q);
  }
  s = block_sum(s, red);
  q = block_sum(q, red);
  if (threadIdx.x == 0) {
    const float mean = s / (float)K, rms = sqrtf(q / (float)K);
    const float ratio = rms > 0.f ? fabsf(mean) / rms : 0.f;
    atomicMax(&g_ln_center_max, __float_as_uint(ratio));
  }
}

cudaError_t layernorm_center_check(const void* a, int64_t M, int64_t K, int dtype, cudaStream_t stream,
                                   float* max_ratio) {
  void* dptr = nullptr;
  cudaError_t e = cudaGetSymbolAddress(&dptr, g_ln_center_max);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(dptr, 0, sizeof(unsigned), stream)) != cudaSuccess) return e;
  if (dtype == 0)
    layernorm_center_check_kernel<__nv_bfloat16><<<(unsigned)M, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(a), (int)K);
  else
    layernorm_center_check_kernel<float><<<(unsigned)M, 256, 0, stream>>>(static_cast<const float*>(a), (int)K);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  unsigned bits = 0;
  if ((e = cudaMemcpyAsync(&bits, dptr, sizeof(bits), cudaMemcpyDeviceToHost, stream)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return e;
  memcpy(max_ratio, &bits, sizeof(bits));
  return cudaSuccess;
}

}  // namespace fn
