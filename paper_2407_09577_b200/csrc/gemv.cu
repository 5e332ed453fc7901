// gemv.cu — K4: decode-shaped FlashNorm linear (M <= 16 tokens), bf16, HBM-bound.
//
//   z[m][j] = RN( fma( sum_k a[m][k] W*t[j][k], r_m, c*_j ) ),  r_m = rsqrt(ssq_m/K + eps)
//
// The whole cost is streaming W* (K*N*2 bytes) once from HBM.
// PAPER.md:145-154 (§5, Fig 8): at batch 1 the RMS is a vector-unit bottleneck
// in front of the matrix unit; with deferred normalization (Fig 8(c)) the W*
// stream starts immediately, ssq is computed while the first W* loads are in
// flight, and the scale is applied at the very end.
//
// Work split (one persistent CTA of 16 warps per SM):
//  * CTA c owns the contiguous OUTPUT ROWS [c*N/G, (c+1)*N/G) of W*t — byte-balanced
//    across SMs; 8-row mma tiles at the range ends are shared with the neighbour
//    CTA, each side loading/storing only its own rows.
//  * inside a CTA the 16 warps split K (warp w owns 32-wide K chunks w, w+16, ...)
//    and walk ALL of the CTA's tiles as one flat load stream (two register
//    buffers of CH 16-byte loads per lane in flight) with no barrier inside.
//  * each lane streams 16-byte pieces of W*t straight into mma.sync.m16n8k16
//    B fragments (the K order inside a fragment is permuted consistently for A
//    and B — a dot product is order-free); the <=16 tokens are the A operand,
//    read from shared memory.  Tensor-core MMAs keep the ALU off the critical
//    path at M = 16 (FFMA cannot sustain HBM rate there).
//  * per-warp partial tiles go to shared memory; one barrier per segment of
//    <= SEG tiles, then a fixed-order reduction, * r + c*, bf16 store.
#include "common.cuh"
#include "kernels.h"

namespace fn {

namespace gv {
constexpr int WARPS = 16;
constexpr int THREADS = WARPS * 32;
constexpr int CH = 8;    // 16-byte loads per lane per buffer (two buffers in flight)
constexpr int SEG = 8;   // max 8-row tiles per segment (partials kept in shared memory)
}  // namespace gv

FN_DEVICE uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

FN_DEVICE void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                              uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

size_t gemv_smem_bytes(int M, int K) {
  const size_t a_bytes = ((size_t)M * (K + 32) * 2 + 15) / 16 * 16;
  return a_bytes + (size_t)gv::SEG * gv::WARPS * 128 * 4 + 16 * 4;
}

template <int MODE>
__global__ void __launch_bounds__(gv::THREADS, 1)
    flashnorm_gemv_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ Wt,
                          const float* __restrict__ cstar, __nv_bfloat16* __restrict__ z, int M, int K, int N,
                          float eps, float alpha) {
  using namespace gv;
  extern __shared__ __align__(16) uint8_t smem[];
  const int lda = K + 32;  // padded row stride (elements): the 8 rows of a fragment hit distinct banks
  __nv_bfloat16* a_s = reinterpret_cast<__nv_bfloat16*>(smem);
  float* part = reinterpret_cast<float*>(smem + ((size_t)M * lda * 2 + 15) / 16 * 16);  // [SEG][WARPS][128]
  float* r_s = part + SEG * WARPS * 128;                                                  // [16]

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int g = lane >> 2;
  const int kq = lane & 3;

  // byte-balanced contiguous row range of this CTA
  const int r0 = (int)(((long long)blockIdx.x * N) / gridDim.x);
  const int r1 = (int)(((long long)(blockIdx.x + 1) * N) / gridDim.x);
  const int t0 = r0 >> 3;
  const int ntiles = r1 > r0 ? ((r1 - 1) >> 3) - t0 + 1 : 0;
  const int kchunks = (K + 31) >> 5;
  const int cpw = (kchunks - warp + WARPS - 1) / WARPS;  // chunks of this warp per tile (warp-uniform)

  // flat per-warp stream over (tile, chunk) of the current segment
  auto load_group = [&](int seg_t0, int item0, int items, uint4 (&w)[CH]) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      w[i] = make_uint4(0u, 0u, 0u, 0u);
      const int it = item0 + i;
      if (it < items) {
        const int tile = seg_t0 + it / cpw;
        const int c = warp + WARPS * (it % cpw);
        const int n = (t0 + tile) * 8 + g;
        const int k = c * 32 + kq * 8;
        if (n >= r0 && n < r1 && k < K) w[i] = ldg_stream(Wt + (size_t)n * K + k);
      }
    }
  };

  uint4 wb0[CH], wb1[CH];
  const int seg0_tiles = ntiles < SEG ? ntiles : SEG;
  load_group(0, 0, seg0_tiles * cpw, wb0);  // the W* stream starts before the RMS (Fig 8(c))

  // stage the M tokens into shared memory (DyT: tanh prologue applied here, once)
  const int kv = K >> 3;
  for (int i = tid; i < M * kv; i += THREADS) {
    const int m = i / kv;
    const int k = (i - m * kv) * 8;
    uint4 v = *reinterpret_cast<const uint4*>(a + (size_t)m * K + k);
    if (MODE == MODE_DYT) {
      uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = tanh_approx_bf16x2(pack_bf16(bf16lo(w[q]) * alpha, bf16hi(w[q]) * alpha));
    }
    *reinterpret_cast<uint4*>(a_s + (size_t)m * lda + k) = v;
  }
  __syncthreads();

  // per-token sum of squares, overlapped with the W* loads already in flight
  if (MODE == MODE_RMS && warp < M) {
    float s0 = 0.f, s1 = 0.f;
    for (int k = lane * 8; k < K; k += 256) {
      const uint4 v = *reinterpret_cast<const uint4*>(a_s + (size_t)warp * lda + k);
      float x;
      x = bf16lo(v.x); s0 = fmaf(x, x, s0);
      x = bf16hi(v.x); s1 = fmaf(x, x, s1);
      x = bf16lo(v.y); s0 = fmaf(x, x, s0);
      x = bf16hi(v.y); s1 = fmaf(x, x, s1);
      x = bf16lo(v.z); s0 = fmaf(x, x, s0);
      x = bf16hi(v.z); s1 = fmaf(x, x, s1);
      x = bf16lo(v.w); s0 = fmaf(x, x, s0);
      x = bf16hi(v.w); s1 = fmaf(x, x, s1);
    }
    float s = s0 + s1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) r_s[warp] = rsqrtf(fmaf(s, 1.0f / (float)K, eps));
  }

  const bool row_lo = g < M;
  const bool row_hi = g + 8 < M;
  bool first = true;
  for (int seg_t0 = 0; seg_t0 < ntiles; seg_t0 += SEG) {
    const int seg_tiles = (ntiles - seg_t0) < SEG ? (ntiles - seg_t0) : SEG;
    const int items = seg_tiles * cpw;
    if (!first) load_group(seg_t0, 0, items, wb0);
    first = false;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};

    auto compute_group = [&](int item0, const uint4 (&w)[CH]) {
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int it = item0 + i;
        if (it < items) {  // warp-uniform
          const int c = warp + WARPS * (it % cpw);
          const int k = c * 32 + kq * 8;
          uint4 ra = make_uint4(0u, 0u, 0u, 0u), rb = make_uint4(0u, 0u, 0u, 0u);
          if (row_lo && k < K) ra = *reinterpret_cast<const uint4*>(a_s + (size_t)g * lda + k);
          if (row_hi && k < K) rb = *reinterpret_cast<const uint4*>(a_s + (size_t)(g + 8) * lda + k);
          mma_bf16_16816(acc, ra.x, rb.x, ra.y, rb.y, w[i].x, w[i].y);
          mma_bf16_16816(acc, ra.z, rb.z, ra.w, rb.w, w[i].z, w[i].w);
          if (it % cpw == cpw - 1) {  // last chunk of this warp for the tile: park the partial
            const int tile = it / cpw;
            *reinterpret_cast<float4*>(part + ((size_t)tile * WARPS + warp) * 128 + lane * 4) =
                make_float4(acc[0], acc[1], acc[2], acc[3]);
            acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
          }
        }
      }
    };

    for (int item0 = 0; item0 < items; item0 += 2 * CH) {
      load_group(seg_t0, item0 + CH, items, wb1);
      compute_group(item0, wb0);
      load_group(seg_t0, item0 + 2 * CH, items, wb0);
      compute_group(item0 + CH, wb1);
    }
    if (cpw == 0) {  // warp without K chunks (K < 16*32): contributes zero partials
      for (int tile = 0; tile < seg_tiles; ++tile)
        *reinterpret_cast<float4*>(part + ((size_t)tile * WARPS + warp) * 128 + lane * 4) =
            make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    // fixed-order reduction over the 16 warps, deferred scale, bias, bf16 store
    for (int e = tid; e < seg_tiles * 128; e += THREADS) {
      const int tile = e >> 7, slot = e & 127;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) s += part[((size_t)tile * WARPS + w) * 128 + slot];
      const int ln = slot >> 2, i = slot & 3;
      const int row = (ln >> 2) + (i >= 2 ? 8 : 0);
      const int col = (ln & 3) * 2 + (i & 1);
      const int n = (t0 + seg_t0 + tile) * 8 + col;
      if (row < M && n >= r0 && n < r1) {
        const float r = MODE == MODE_RMS ? r_s[row] : 1.0f;
        const float cb = cstar != nullptr ? __ldg(cstar + n) : 0.0f;
        z[(size_t)row * N + n] = __float2bfloat16_rn(fmaf(s, r, cb));
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_gemv(const __nv_bfloat16* a, const __nv_bfloat16* Wt, const float* cstar, __nv_bfloat16* z,
                        int M, int K, int N, float eps, float alpha, int mode, int num_sms, cudaStream_t stream) {
  const size_t smem = gemv_smem_bytes(M, K);
  const void* fptr = mode == MODE_RMS ? (const void*)flashnorm_gemv_kernel<MODE_RMS>
                     : mode == MODE_DYT ? (const void*)flashnorm_gemv_kernel<MODE_DYT>
                                        : (const void*)flashnorm_gemv_kernel<MODE_NONE>;
  static size_t attr_set[3] = {0, 0, 0};
  if (smem > 48 * 1024 && attr_set[mode] < smem) {
    cudaError_t e = cudaFuncSetAttribute(fptr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set[mode] = smem;
  }
  // one CTA per SM, but never fewer than ~8 output rows per CTA
  int grid = (N + 7) / 8;
  if (grid > num_sms) grid = num_sms;
  void* args[] = {(void*)&a, (void*)&Wt, (void*)&cstar, (void*)&z, (void*)&M, (void*)&K, (void*)&N, (void*)&eps,
                  (void*)&alpha};
  return cudaLaunchKernel(fptr, dim3(grid), dim3(gv::THREADS), args, smem, stream);
}

}  // namespace fn
