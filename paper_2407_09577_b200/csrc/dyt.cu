// dyt.cu — K8: DyT activation pre-pass  y = RN_bf16(tanh(alpha * a))  (reading c10).
//
// Why a pre-pass exists at all: the A-tile prologue of the GEMM (gemm*_sm100.cu) recomputes
// tanh(alpha a) once per N tile, i.e. N/256 times per element, and the MUFU tanh unit delivers
// only ~16 values/clk/SM on sm_100a for BOTH tanh.approx.f32 and tanh.approx.bf16x2
// (tools/micro/mufu.cu, measured 4.6 Tvalues/s).  A 128x64 bf16 A stage is 8192 tanh values =
// 512 MUFU cycles, the same as the 512 cycles the tensor core spends on that stage at BN=256,
// so the prologue caps DyT near half of the GEMM rate.  Computing tanh ONCE per element here
// (HBM-bound: 2 bytes read + 2 bytes written per element, the output stays in the 126 MB L2
// for the GEMM that follows) and running the GEMM in mode NONE removes that cap.
//
// Arithmetic is bit-identical to the in-kernel prologue: x = a (bf16x2) * alpha (bf16x2, RN),
// y = tanh.approx.bf16x2(x), so z matches flashnorm_linear's in-kernel DyT bit for bit.
#include "common.cuh"
#include "kernels.h"

namespace fn {

namespace {

constexpr int DYT_THREADS = 256;
constexpr int DYT_UNROLL = 4;  // 16-byte vectors in flight per thread

FN_DEVICE uint32_t dyt2(uint32_t v, __nv_bfloat162 alpha2) {
  __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&v);
  x = __hmul2(x, alpha2);
  return tanh_approx_bf16x2(*reinterpret_cast<uint32_t*>(&x));
}

FN_DEVICE uint4 dyt8(uint4 v, __nv_bfloat162 alpha2) {
  return make_uint4(dyt2(v.x, alpha2), dyt2(v.y, alpha2), dyt2(v.z, alpha2), dyt2(v.w, alpha2));
}

__global__ void __launch_bounds__(DYT_THREADS) dyt_prepass_kernel(const uint4* __restrict__ a, uint4* __restrict__ y,
                                                                  int64_t n16, float alpha) {
  const __nv_bfloat162 alpha2 = __floats2bfloat162_rn(alpha, alpha);
  const int64_t stride = (int64_t)gridDim.x * DYT_THREADS;
  int64_t i = (int64_t)blockIdx.x * DYT_THREADS + threadIdx.x;
  // main loop: DYT_UNROLL independent 16-byte loads issued before any MUFU work
  for (; i + (DYT_UNROLL - 1) * stride < n16; i += DYT_UNROLL * stride) {
    uint4 v[DYT_UNROLL];
#pragma unroll
    for (int u = 0; u < DYT_UNROLL; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < DYT_UNROLL; ++u) y[i + u * stride] = dyt8(v[u], alpha2);
  }
  for (; i < n16; i += stride) y[i] = dyt8(__ldcs(a + i), alpha2);
}

}  // namespace

cudaError_t launch_dyt_prepass(const __nv_bfloat16* a, __nv_bfloat16* y, int64_t n, float alpha, int num_sms,
                               cudaStream_t stream) {
  const int64_t n16 = n / 8;  // n % 8 == 0 (K % 8 == 0 is validated by the caller)
  int64_t blocks = (n16 + DYT_THREADS * DYT_UNROLL - 1) / (DYT_THREADS * DYT_UNROLL);
  const int64_t cap = (int64_t)num_sms * 8;  // 8 x 256 threads resident per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  dyt_prepass_kernel<<<(unsigned)blocks, DYT_THREADS, 0, stream>>>(reinterpret_cast<const uint4*>(a),
                                                                   reinterpret_cast<uint4*>(y), n16, alpha);
  return cudaGetLastError();
}

}  // namespace fn
