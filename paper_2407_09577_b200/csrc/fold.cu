// fold.cu — K1/K2: the offline FlashNorm weight folds, HBM-bound, 128-bit accesses.
//
// K1 fold_weights  (PAPER.md:25 Fig A, then PAPER.md:16 Fig 1(b)):
//    W*t[j][i] = RN_dtype(RN_f32(g_i * Wt[j][i]))
//    c*_j      = RN_f32(c_j + sum_i b_i * Wt[j][i])      (fp64, ORIGINAL W)
//    One warp per output row j: one pass over W reads Wt[j,:] once and writes
//    W*t[j,:] once.  The fp64 sum order is the contract in include/flashnorm.h.
//
// K2 fold_mean_center (Fig B):
//    pass 1  fp64 partial column sums of Vt over 32-row chunks   (s_i)
//    pass 1b s_i = fixed-order (lane-strided + xor butterfly) sum of the partials, one warp
//            per column; the same launch centers b_prev* = b_prev - mean(b_prev) (reading c7)
//    pass 2  V*t[j][i] = RN(Vt[j][i] - s_i/n)
//    The second read of Vt is L2-resident for the config-4 sizes (33.5 MB < 126 MB).
//
// All fp64 arithmetic uses __dmul_rn/__dadd_rn so no FMA contraction changes
// the rounding the CPU mirror reproduces.
#include "common.cuh"
#include "kernels.h"

namespace fn {

namespace fold {
constexpr int WARPS_PER_CTA = 8;  // K1
constexpr int ROWS_PER_WARP = 2;  // K1: rows sharing one g/b chunk load
constexpr int CHUNK_UNROLL = 4;   // K1: chunks per lane in flight
constexpr int COLSUM_ROWS = 32;  // rows per fp64 partial in K2 (contract constant)
constexpr int BPREV_THREADS = 256;
}  // namespace fold

FN_DEVICE uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// element e (0..E-1) of a 16-byte chunk as float
template <int DT>
FN_DEVICE float chunk_elem(const uint4& v, int e) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
  if (DT == 0) return (e & 1) ? bf16hi(w[e >> 1]) : bf16lo(w[e >> 1]);
  return __uint_as_float(w[e]);
}

template <int DT, bool HAS_G, bool HAS_B>
__global__ void __launch_bounds__(fold::WARPS_PER_CTA * 32)
    fold_weights_kernel(const uint8_t* __restrict__ Wt, int64_t N, int64_t K, const float* __restrict__ g,
                        const float* __restrict__ b, const float* __restrict__ c, uint8_t* __restrict__ Wt_star,
                        float* __restrict__ c_star) {
  // One warp per RPW consecutive rows: each lane loads its g/b chunk once and applies
  // it to RPW rows (RPW independent 16-byte W loads in flight per chunk); the c* sum of
  // every row keeps the contract order (lane l: its chunks ascending, then butterfly).
  constexpr int E = DT == 0 ? 8 : 4;       // elements per 16-byte chunk
  constexpr int ES = DT == 0 ? 2 : 4;      // element size
  constexpr int RPW = fold::ROWS_PER_WARP;
  const int lane = threadIdx.x & 31;
  const int64_t j0 = ((int64_t)blockIdx.x * fold::WARPS_PER_CTA + (threadIdx.x >> 5)) * RPW;
  if (j0 >= N) return;
  const int64_t nchunks = K / E;  // K % E == 0 enforced by the ABI
  double acc[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) acc[r] = 0.0;
  constexpr int U = fold::CHUNK_UNROLL;
  for (int64_t q0 = lane; q0 < nchunks; q0 += 32 * U) {
   uint4 vv[U][RPW];
#pragma unroll
   for (int u = 0; u < U; ++u)  // U x RPW independent 16-byte loads in flight
#pragma unroll
     for (int r = 0; r < RPW; ++r)
       if (q0 + u * 32 < nchunks && j0 + r < N) vv[u][r] = ld_nc_v4(Wt + ((j0 + r) * K + (q0 + u * 32) * E) * ES);
#pragma unroll
   for (int u = 0; u < U; ++u) {
    const int64_t q = q0 + u * 32;
    if (q >= nchunks) break;
    const uint4* v = vv[u];
    const int64_t i0 = q * E;
    float gv[E], bv[E];
    if (HAS_G) {
      const float4* g4 = reinterpret_cast<const float4*>(g + i0);
#pragma unroll
      for (int t = 0; t < E / 4; ++t) {
        const float4 x = __ldg(g4 + t);
        gv[4 * t] = x.x; gv[4 * t + 1] = x.y; gv[4 * t + 2] = x.z; gv[4 * t + 3] = x.w;
      }
    }
    if (HAS_B) {
      const float4* b4 = reinterpret_cast<const float4*>(b + i0);
#pragma unroll
      for (int t = 0; t < E / 4; ++t) {
        const float4 x = __ldg(b4 + t);
        bv[4 * t] = x.x; bv[4 * t + 1] = x.y; bv[4 * t + 2] = x.z; bv[4 * t + 3] = x.w;
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      if (j0 + r >= N) break;
      uint4 o;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float w = chunk_elem<DT>(v[r], e);
        if (HAS_B) acc[r] = __dadd_rn(acc[r], __dmul_rn((double)bv[e], (double)w));  // exact product, ordered sum
        const float ws = HAS_G ? __fmul_rn(gv[e], w) : w;
        if (DT == 0) {
          if (e & 1) ow[e >> 1] |= (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(ws)) << 16;
          else ow[e >> 1] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(ws));
        } else {
          ow[e] = __float_as_uint(ws);
        }
      }
      *reinterpret_cast<uint4*>(Wt_star + ((j0 + r) * K + q * E) * ES) = o;
    }
   }
  }
  if (c_star == nullptr) return;
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int64_t j = j0 + r;
    if (j >= N) break;
    if (!HAS_B) {
      if (lane == 0) c_star[j] = c != nullptr ? c[j] : 0.0f;  // c* = c exactly when b is absent
      continue;
    }
    double a2 = acc[r];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a2 = __dadd_rn(a2, __shfl_xor_sync(0xffffffffu, a2, off));
    if (lane == 0) {
      const double cj = c != nullptr ? (double)c[j] : 0.0;
      c_star[j] = __double2float_rn(__dadd_rn(cj, a2));
    }
  }
}

cudaError_t launch_fold_weights(const void* Wt, int64_t N, int64_t K, int dtype, const float* g, const float* b,
                                const float* c, void* Wt_star, float* c_star, cudaStream_t stream) {
  const int64_t rows_per_cta = fold::WARPS_PER_CTA * fold::ROWS_PER_WARP;
  const dim3 grid((unsigned)((N + rows_per_cta - 1) / rows_per_cta));
  const dim3 block(fold::WARPS_PER_CTA * 32);
  const uint8_t* src = static_cast<const uint8_t*>(Wt);
  uint8_t* dst = static_cast<uint8_t*>(Wt_star);
  const bool hg = g != nullptr, hb = b != nullptr;
#define FN_FOLD_LAUNCH(DT, G, B) fold_weights_kernel<DT, G, B><<<grid, block, 0, stream>>>(src, N, K, g, b, c, dst, c_star)
  if (dtype == 0) {
    if (hg && hb) FN_FOLD_LAUNCH(0, true, true);
    else if (hg) FN_FOLD_LAUNCH(0, true, false);
    else if (hb) FN_FOLD_LAUNCH(0, false, true);
    else FN_FOLD_LAUNCH(0, false, false);
  } else {
    if (hg && hb) FN_FOLD_LAUNCH(1, true, true);
    else if (hg) FN_FOLD_LAUNCH(1, true, false);
    else if (hb) FN_FOLD_LAUNCH(1, false, true);
    else FN_FOLD_LAUNCH(1, false, false);
  }
#undef FN_FOLD_LAUNCH
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K2

int64_t fold_mean_center_workspace(int64_t n_out, int64_t d_in) {
  const int64_t nchunk = (n_out + fold::COLSUM_ROWS - 1) / fold::COLSUM_ROWS;
  return (nchunk + 1) * d_in * (int64_t)sizeof(double);  // partials + s_i/n
}

// b_prev* = b_prev - mean(b_prev), one CTA of BPREV_THREADS threads (contract order)
FN_DEVICE void center_bias_block(const float* __restrict__ b_prev, int64_t n_out, float* __restrict__ b_star,
                                 double* wsum, double* mean_s) {
  const int t = threadIdx.x;
  double acc = 0.0;
  for (int64_t j = t; j < n_out; j += fold::BPREV_THREADS) acc = __dadd_rn(acc, (double)b_prev[j]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
  if ((t & 31) == 0) wsum[t >> 5] = acc;
  __syncthreads();
  if (t == 0) {
    double tot = 0.0;
    for (int w = 0; w < fold::BPREV_THREADS / 32; ++w) tot = __dadd_rn(tot, wsum[w]);
    *mean_s = __ddiv_rn(tot, (double)n_out);
  }
  __syncthreads();
  const double mean = *mean_s;
  for (int64_t j = t; j < n_out; j += fold::BPREV_THREADS)
    b_star[j] = __double2float_rn(__dsub_rn((double)b_prev[j], mean));
}

// pass 1b: one warp per column i: lane l sums partials c = l, l+32, ... ascending, the
// 32 lane sums are combined by the xor butterfly 16,8,4,2,1; mu_i = s_i / n.  The
// extra last CTA centers b_prev (independent work, same launch).
__global__ void __launch_bounds__(fold::BPREV_THREADS)
    colsum_reduce_kernel(const double* __restrict__ partial, int64_t nchunk, int64_t d_in, int64_t n_out,
                         double* __restrict__ mu, const float* __restrict__ b_prev, float* __restrict__ b_star) {
  __shared__ double wsum[fold::BPREV_THREADS / 32];
  __shared__ double mean_s;
  const int64_t ncol_blocks = (d_in + fold::BPREV_THREADS / 32 - 1) / (fold::BPREV_THREADS / 32);
  if ((int64_t)blockIdx.x == ncol_blocks) {
    if (b_prev != nullptr) center_bias_block(b_prev, n_out, b_star, wsum, &mean_s);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (fold::BPREV_THREADS / 32) + (threadIdx.x >> 5);
  if (i >= d_in) return;
  double v[8];
  double acc = 0.0;
  for (int64_t c0 = lane; c0 < nchunk; c0 += 32 * 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t c = c0 + u * 32;
      v[u] = c < nchunk ? partial[c * d_in + i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (c0 + u * 32 < nchunk) acc = __dadd_rn(acc, v[u]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
  if (lane == 0) mu[i] = __ddiv_rn(acc, (double)n_out);
}

// pass 1: partial[cidx][i] = sum_{j in chunk cidx, ascending} Vt[j][i]
// thread -> one 16-byte column group (E columns), block.y -> one 32-row chunk
template <int DT>
__global__ void __launch_bounds__(128)
    colsum_partial_kernel(const uint8_t* __restrict__ Vt, int64_t n_out, int64_t d_in, double* __restrict__ partial) {
  constexpr int E = DT == 0 ? 8 : 4;
  constexpr int ES = DT == 0 ? 2 : 4;
  const int64_t grp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ngrp = d_in / E;
  if (grp >= ngrp) return;
  const int64_t cidx = blockIdx.y;
  const int64_t j0 = cidx * fold::COLSUM_ROWS;
  const int64_t j1 = min(j0 + fold::COLSUM_ROWS, n_out);
  double acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.0;
  const uint8_t* p = Vt + (j0 * d_in + grp * E) * ES;
  for (int64_t j = j0; j < j1; j += 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j + u < j1) v[u] = ld_nc_v4(p + (j - j0 + u) * d_in * ES);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j + u >= j1) break;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = __dadd_rn(acc[e], (double)chunk_elem<DT>(v[u], e));
    }
  }
  double* out = partial + cidx * d_in + grp * E;
#pragma unroll
  for (int e = 0; e < E; ++e) out[e] = acc[e];
}

// pass 2: V*t = RN(Vt - s_i/n).  block.y -> 32-row chunk (second read of Vt: L2-resident).
template <int DT>
__global__ void __launch_bounds__(128)
    center_kernel(const uint8_t* __restrict__ Vt, int64_t n_out, int64_t d_in, const double* __restrict__ mu_g,
                  uint8_t* __restrict__ Vt_star) {
  constexpr int E = DT == 0 ? 8 : 4;
  constexpr int ES = DT == 0 ? 2 : 4;
  const int64_t grp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ngrp = d_in / E;
  if (grp >= ngrp) return;
  double mu[E];
#pragma unroll
  for (int e = 0; e < E; ++e) mu[e] = mu_g[grp * E + e];
  const int64_t j0 = (int64_t)blockIdx.y * fold::COLSUM_ROWS;
  const int64_t j1 = min(j0 + fold::COLSUM_ROWS, n_out);
  for (int64_t j = j0; j < j1; j += 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)  // 8 independent 16-byte loads in flight
      if (j + u < j1) v[u] = ld_nc_v4(Vt + ((j + u) * d_in + grp * E) * ES);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j + u >= j1) break;
      uint4 o;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float r32 = __double2float_rn(__dsub_rn((double)chunk_elem<DT>(v[u], e), mu[e]));
        if (DT == 0) {
          const uint32_t hb = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(r32));
          if (e & 1) ow[e >> 1] |= hb << 16;
          else ow[e >> 1] = hb;
        } else {
          ow[e] = __float_as_uint(r32);
        }
      }
      *reinterpret_cast<uint4*>(Vt_star + ((j + u) * d_in + grp * E) * ES) = o;
    }
  }
}

cudaError_t launch_fold_mean_center(const void* Vt, int64_t n_out, int64_t d_in, int dtype, const float* b_prev,
                                    void* Vt_star, float* b_prev_star, void* workspace, cudaStream_t stream,
                                    int* launches) {
  const int E = dtype == 0 ? 8 : 4;
  const int64_t ngrp = d_in / E;
  const int64_t nchunk = (n_out + fold::COLSUM_ROWS - 1) / fold::COLSUM_ROWS;
  const dim3 grid((unsigned)((ngrp + 127) / 128), (unsigned)nchunk);
  double* partial = static_cast<double*>(workspace);
  const uint8_t* src = static_cast<const uint8_t*>(Vt);
  uint8_t* dst = static_cast<uint8_t*>(Vt_star);
  double* mu = partial + nchunk * d_in;
  const int64_t cols_per_cta = fold::BPREV_THREADS / 32;  // one warp per column
  const unsigned rgrid = (unsigned)((d_in + cols_per_cta - 1) / cols_per_cta + 1);  // + the b_prev CTA
  if (dtype == 0) {
    colsum_partial_kernel<0><<<grid, 128, 0, stream>>>(src, n_out, d_in, partial);
    colsum_reduce_kernel<<<rgrid, fold::BPREV_THREADS, 0, stream>>>(partial, nchunk, d_in, n_out, mu, b_prev,
                                                                     b_prev_star);
    center_kernel<0><<<grid, 128, 0, stream>>>(src, n_out, d_in, mu, dst);
  } else {
    colsum_partial_kernel<1><<<grid, 128, 0, stream>>>(src, n_out, d_in, partial);
    colsum_reduce_kernel<<<rgrid, fold::BPREV_THREADS, 0, stream>>>(partial, nchunk, d_in, n_out, mu, b_prev,
                                                                     b_prev_star);
    center_kernel<1><<<grid, 128, 0, stream>>>(src, n_out, d_in, mu, dst);
  }
  *launches = 3;
  return cudaGetLastError();
}

}  // namespace fn
