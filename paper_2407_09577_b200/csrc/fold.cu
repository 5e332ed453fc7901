// fold.cu — K1/K2: the offline FlashNorm weight folds, HBM-bound, 128-bit accesses.
//
// K1 fold_weights  (PAPER.md:25 Fig A, then PAPER.md:16 Fig 1(b)):
//    W*t[j][i] = RN_dtype(RN_f32(g_i * Wt[j][i]))
//    c*_j      = RN_f32(c_j + sum_i b_i * Wt[j][i])      (fp64, ORIGINAL W)
//    One warp per output row j: one pass over W reads Wt[j,:] once and writes
//    W*t[j,:] once.  The fp64 sum order is the contract in include/flashnorm.h.
//
// K2 fold_mean_center (Fig B): ONE launch of clusters of 8 CTAs (see the K2 section)
//    s_i = fp64 column sums in the contract order (32-row partials, lane sums, butterfly), reduced
//    on chip over DSMEM; mu_i = RN_f32(s_i / n); V*t[j][i] = RN_dtype(Vt[j][i] - mu_i) in f32
//    (reading c21); b_prev* = b_prev - mean(b_prev) (reading c7).
//
// All fp64 arithmetic uses explicit _rn intrinsics so no compiler contraction changes the
// rounding the CPU mirror reproduces; the one fused multiply-add (K1's b*w) is exact-
// equivalent because the product is exact.  bf16/f32 -> fp64 widening is done with integer
// ops in a 2^-896-scaled domain (widen_scaled_hi), not on the quarter-rate conversion unit.
#include "common.cuh"
#include <cooperative_groups.h>
#include "kernels.h"

#include <cstdio>
#include <cstdlib>

#include <algorithm>

namespace fn {
namespace cg = cooperative_groups;

namespace fold {
constexpr int WARPS_PER_CTA = 8;  // K1
constexpr int ROWS_PER_WARP = 2;  // K1: rows sharing one g/b chunk load
constexpr int CHUNK_UNROLL = 2;   // K1: chunks per lane in flight (x ROWS_PER_WARP loads, 3 CTAs/SM)
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

// Exact float -> double WITHOUT the conversion unit.  F2F.F64.F32 issues on the quarter-rate
// XU pipe (ncu: 66-69 % XU utilisation in K1/K2), so normal numbers are widened with integer
// ops — exponent re-bias (+896) and a 3-bit mantissa shift — and a chunk holding a zero,
// subnormal, inf or NaN takes the hardware conversion as a whole.  Same values, so the
// contract arithmetic (and the CPU mirror) is unchanged.
FN_DEVICE double widen_normal(uint32_t x) {  // x: f32 bit pattern with exponent field in 1..254
  return __hiloint2double((int)((((x & 0x7FFFFFFFu) >> 3) + 0x38000000u) | (x & 0x80000000u)), (int)(x << 29));
}

// NW 32-bit words of DT data (bf16 pairs or f32) -> 2*NW or NW doubles, exact.
template <int DT, int NW>
FN_DEVICE void widen_words(const uint32_t* w, double* out) {
  uint32_t special = 0u;
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    if (DT == 0) {
      const uint32_t t = (w[k] & 0x7F807F80u) + 0x00800080u;  // exponent 0 or 255 -> bits 14..8 / 30..24 clear
      special |= (uint32_t)((t & 0x7F00u) == 0u) | (uint32_t)((t & 0x7F000000u) == 0u);
      out[2 * k] = widen_normal(w[k] << 16);
      out[2 * k + 1] = widen_normal(w[k] & 0xFFFF0000u);
    } else {
      const uint32_t t = (w[k] & 0x7F800000u) + 0x00800000u;
      special |= (uint32_t)((t & 0x7F000000u) == 0u);
      out[k] = widen_normal(w[k]);
    }
  }
  if (special) {
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      if (DT == 0) {
        out[2 * k] = (double)__uint_as_float(w[k] << 16);
        out[2 * k + 1] = (double)__uint_as_float(w[k] & 0xFFFF0000u);
      } else {
        out[k] = (double)__uint_as_float(w[k]);
      }
    }
  }
}

// Scaled widening (K2): the bit pattern of a bf16/f32 value x, with its 8-bit exponent field
// moved into the low 8 bits of the double's 11-bit field, is the double x * 2^-896 — exact for
// normal, zero AND subnormal x (the exponent field is not re-biased, so a zero field stays a
// zero field).  Two integer ops per value: arithmetic shift right 3 (sign copied into bits
// 31..28), clear bits 30..28.  Inf/NaN (field 255) are NOT mapped (they become finite); the
// callers detect them with inf_nan_mark and redo that thread's work with hardware conversions.
// Sums of such scaled values round exactly like the unscaled sums: results >= 2^-1022 are
// normal (same 53-bit rounding), smaller ones are multiples of the inputs' granularity
// (>= 2^-1045) and therefore exact.  K2 multiplies by 2^896 (exact) before any division.
constexpr double kScaleDown = 0x1p-896;
constexpr double kScaleUp = 0x1p896;
FN_DEVICE double widen_scaled_hi(uint32_t hi16_in_top) {  // bf16 in bits 31..16, low bits ignored
  return __hiloint2double((int)(((int32_t)hi16_in_top >> 3) & (int32_t)0x8FFFE000), 0);
}
FN_DEVICE double widen_scaled_f32(uint32_t u) {
  return __hiloint2double((int)(((int32_t)u >> 3) & (int32_t)0x8FFFFFFF), (int)(u << 29));
}
// running max of the exponent|mantissa fields (per 16-bit half for bf16): >= 0x7F80 / 0x7F800000
// means an inf/NaN was seen
template <int DT>
FN_DEVICE uint32_t inf_nan_mark(uint32_t mark, uint32_t w) {
  return DT == 0 ? __vmaxu2(mark, w & 0x7FFF7FFFu) : max(mark, w & 0x7FFFFFFFu);
}
template <int DT>
FN_DEVICE bool inf_nan_seen(uint32_t mark) {
  return DT == 0 ? ((mark & 0xFFFFu) >= 0x7F80u || (mark >> 16) >= 0x7F80u) : mark >= 0x7F800000u;
}
// one 4-byte word -> its E scaled doubles (fast path) / hardware path (exact for every input)
template <int DT>
FN_DEVICE void widen_word_scaled(uint32_t w, double* d) {
  if (DT == 0) {
    d[0] = widen_scaled_hi(w << 16);
    d[DT == 0 ? 1 : 0] = widen_scaled_hi(w);
  } else {
    d[0] = widen_scaled_f32(w);
  }
}
template <int DT>
FN_DEVICE void widen_word_hw(uint32_t w, double* d) {
  if (DT == 0) {
    d[0] = __dmul_rn((double)__uint_as_float(w << 16), kScaleDown);
    d[DT == 0 ? 1 : 0] = __dmul_rn((double)__uint_as_float(w & 0xFFFF0000u), kScaleDown);
  } else {
    d[0] = __dmul_rn((double)__uint_as_float(w), kScaleDown);
  }
}

// element e (0..E-1) of a 16-byte chunk as float
template <int DT>
FN_DEVICE float chunk_elem(const uint4& v, int e) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
  if (DT == 0) return (e & 1) ? bf16hi(w[e >> 1]) : bf16lo(w[e >> 1]);
  return __uint_as_float(w[e]);
}

template <int DT, bool HAS_G, bool HAS_B, int RPW = fold::ROWS_PER_WARP, int U = fold::CHUNK_UNROLL, int MINB = 1>
__global__ void __launch_bounds__(fold::WARPS_PER_CTA * 32, MINB)
    fold_weights_kernel(const uint8_t* __restrict__ Wt, int64_t N, int64_t K, const float* __restrict__ g,
                        const float* __restrict__ b, const float* __restrict__ c, uint8_t* __restrict__ Wt_star,
                        float* __restrict__ c_star, int glu_half) {
  // One warp per RPW consecutive rows: each lane loads its g/b chunk once and applies
  // it to RPW rows (RPW independent 16-byte W loads in flight per chunk); the c* sum of
  // every row keeps the contract order (lane l: its chunks ascending, then butterfly).
  constexpr int E = DT == 0 ? 8 : 4;       // elements per 16-byte chunk
  constexpr int ES = DT == 0 ? 2 : 4;      // element size
  const int lane = threadIdx.x & 31;
  const int64_t j0 = ((int64_t)blockIdx.x * fold::WARPS_PER_CTA + (threadIdx.x >> 5)) * RPW;
  if (j0 >= N) return;
  const int64_t nchunks = K / E;  // K % E == 0 enforced by the ABI
  double acc[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) acc[r] = 0.0;
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
    double bd[E];  // b_i * 2^896 (exact): multiplies the 2^-896-scaled widening of w, see below
    if (HAS_B) {
#pragma unroll
      for (int e = 0; e < E; e += 4) widen_words<1, 4>(reinterpret_cast<const uint32_t*>(bv + e), bd + e);
#pragma unroll
      for (int e = 0; e < E; ++e) bd[e] = __dmul_rn(bd[e], kScaleUp);
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      if (j0 + r >= N) break;
      uint4 o;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
      float ws[E];
      double wd[E];
      if (HAS_B) {
        // w * 2^-896 by integer ops (widen_scaled_hi); (b 2^896)(w 2^-896) is the same real
        // product b*w, so the rounded fp64 product is identical.  inf/NaN: hardware widening.
        const uint32_t* vw = reinterpret_cast<const uint32_t*>(&v[r]);
        uint32_t mark = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) mark = inf_nan_mark<DT>(mark, vw[k]);
        if (!inf_nan_seen<DT>(mark)) {
#pragma unroll
          for (int k = 0; k < 4; ++k) widen_word_scaled<DT>(vw[k], wd + k * (E / 4));
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) widen_word_hw<DT>(vw[k], wd + k * (E / 4));
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float w = chunk_elem<DT>(v[r], e);
        // b*w is exact in fp64 (24 x 8 or 24 x 24 significand bits, no underflow), so the
        // fused multiply-add rounds exactly like add(acc, mul(b, w)) in the mirror
        if (HAS_B) acc[r] = __fma_rn(bd[e], wd[e], acc[r]);
        ws[e] = HAS_G ? __fmul_rn(gv[e], w) : w;
      }
#pragma unroll
      for (int e = 0; e < E; e += 2) {
        if (DT == 0) ow[e >> 1] = pack_bf16(ws[e], ws[e + 1]);  // packed RNE (F2FP, not XU)
        else { ow[e] = __float_as_uint(ws[e]); ow[e + 1] = __float_as_uint(ws[e + 1]); }
      }
      const int64_t jr = j0 + r;
      const int64_t jo = glu_half < 0 ? jr : (jr >> 7) * 256 + glu_half * 128 + (jr & 127);  // GLU interleave
      *reinterpret_cast<uint4*>(Wt_star + (jo * K + q * E) * ES) = o;
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

// K1 on a TMA ring (default): a persistent CTA (one per SM) owns blocks of 16 consecutive rows;
// a producer warp streams each block's rows as [16 rows x 2 KiB] boxes (four 512-byte-wide TMA
// sub-boxes, the box width limit) through a 6-slot ring (192 KiB in flight per SM, independent
// of the consumers' pace).  Consumer warp w takes row w of every box, lane l the chunks l, l+32,
// l+64, l+96 of the row's 2 KiB segment, so lane l sees chunks l, l+32, ... in ascending order
// across the segments — exactly the c* contract order (include/flashnorm.h).  W* goes out with
// 16-byte streaming stores (512 contiguous bytes per warp store).
// The c* products use the hardware widening (F2F.F64.F32, exact for every input incl. inf/NaN
// and subnormals) of w and b: b_i w_i is exact in fp64, so fma(b, w, acc) = add(acc, mul(b, w)),
// the mirror's order.  This kernel is issue-bound, and the hardware conversion costs one
// instruction where the integer widening + inf/NaN marks cost three (the XU pipe has room here).
namespace k1 {
constexpr int CWARPS = 16;                  // consumer warps = rows per block
constexpr int ROWS = CWARPS;
constexpr int THREADS = (CWARPS + 1) * 32;  // + the producer warp
constexpr int SUB = 512;                    // bytes of a row per TMA sub-box (<= 256 elements)
constexpr int U = 4;                        // sub-boxes per box = chunks per lane per box
constexpr int SEG = SUB * U;                // 2 KiB of each row per box
constexpr int SUBBOX = SUB * ROWS;          // 8 KiB
constexpr int BOX = SUBBOX * U;             // 32 KiB
constexpr int RING = 6;                     // 192 KiB
constexpr size_t SMEM = (size_t)RING * BOX + 128;
}  // namespace k1

template <int DT, bool HAS_G, bool HAS_B>
__global__ void __launch_bounds__(k1::THREADS, 1)
    fold_weights_tma_kernel(const __grid_constant__ CUtensorMap tm_w, int64_t N, int64_t K,
                            const float* __restrict__ g, const float* __restrict__ b, const float* __restrict__ c,
                            uint8_t* __restrict__ Wt_star, float* __restrict__ c_star, int glu_half) {
  using namespace k1;
  constexpr int E = DT == 0 ? 8 : 4;   // elements per 16-byte chunk
  constexpr int ES = DT == 0 ? 2 : 4;
  extern __shared__ __align__(128) uint8_t k1s_raw[];
  uint8_t* ring = k1s_raw + ((128u - (smem_u32(k1s_raw) & 127u)) & 127u);
  __shared__ __align__(8) uint64_t full[RING];
  __shared__ __align__(8) uint64_t empty[RING];
  __shared__ volatile uint32_t k1_sink;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nblk = (N + ROWS - 1) / ROWS;
  const int64_t nchunks = K / E;
  const int nseg = (int)((K * ES + SEG - 1) / SEG);
  if (threadIdx.x == 0) {
    for (int i = 0; i < RING; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CWARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == CWARPS) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      prefetch_tmap(&tm_w);
      int k = 0;
      for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x)
        for (int sg = 0; sg < nseg; ++sg, ++k) {
          const int slot = k % RING;
          if (k >= RING) mbar_wait(&empty[slot], (uint32_t)((k / RING) - 1) & 1u);
          const int nsub = min(U, (int)((K * ES - (int64_t)sg * SEG + SUB - 1) / SUB));
          mbar_arrive_expect_tx(&full[slot], (uint32_t)(nsub * SUBBOX));
          for (int u = 0; u < nsub; ++u)
            tma_load_2d(ring + (size_t)slot * BOX + u * SUBBOX, &tm_w, &full[slot], (sg * SEG + u * SUB) / ES,
                        (int32_t)(blk * ROWS), kEvictFirst);
        }
    }
    return;
  }
  // ------------------------------------------------------------------ consumers
  int k = 0;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t j = blk * ROWS + warp;
    const bool row_ok = j < N;
    const int64_t jo = glu_half < 0 ? j : (j >> 7) * 256 + glu_half * 128 + (j & 127);  // GLU interleave
    double acc = 0.0;
    for (int sg = 0; sg < nseg; ++sg, ++k) {
      const int slot = k % RING;
      const int64_t q0 = (int64_t)sg * (SEG / 16) + lane;  // chunk of sub-box 0; sub-box u adds 32 u
      // g / b of this lane's U chunks: issued before the wait
      float4 gq[U][E / 4], bq[U][E / 4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool qv = row_ok && q0 + 32 * u < nchunks;
#pragma unroll
        for (int tt = 0; tt < E / 4; ++tt) {
          if (HAS_G) gq[u][tt] = qv ? __ldg(reinterpret_cast<const float4*>(g + (q0 + 32 * u) * E) + tt)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
          if (HAS_B) bq[u][tt] = qv ? __ldg(reinterpret_cast<const float4*>(b + (q0 + 32 * u) * E) + tt)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      mbar_wait(&full[slot], (uint32_t)(k / RING) & 1u);
      uint4 vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u)  // U independent LDS.128 in flight
        vv[u] = *reinterpret_cast<const uint4*>(ring + (size_t)slot * BOX + u * SUBBOX + warp * SUB + lane * 16);
      if (row_ok) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t q = q0 + 32 * u;
          if (q >= nchunks) break;
          const float* gv = reinterpret_cast<const float*>(gq[u]);
          const float* bv = reinterpret_cast<const float*>(bq[u]);
          uint4 o;
          uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
          float ws[E];
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const float w = chunk_elem<DT>(vv[u], e);
            if (HAS_B) acc = __fma_rn((double)bv[e], (double)w, acc);  // exact product: = add(acc, mul(b, w))
            ws[e] = HAS_G ? __fmul_rn(gv[e], w) : w;
          }
#pragma unroll
          for (int e = 0; e < E; e += 2) {
            if (DT == 0) ow[e >> 1] = pack_bf16(ws[e], ws[e + 1]);
            else { ow[e] = __float_as_uint(ws[e]); ow[e + 1] = __float_as_uint(ws[e + 1]); }
          }
          __stcs(reinterpret_cast<uint4*>(Wt_star + (jo * K + q * E) * ES), o);
        }
      }
      // loaded words not used above (rows >= N, chunks past K) must still be consumed before the slot
      // is released (releasing right after an ld.shared is not safe on sm_100a); the
      // compare reads every loaded register and its (practically never taken) store is harmless
      uint32_t x = 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) x ^= vv[u].x ^ vv[u].y ^ vv[u].z ^ vv[u].w;
      if (x == 0x7FC00001u) k1_sink = x;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // every lane's loads have returned
    }
    if (row_ok && c_star != nullptr) {
      if (!HAS_B) {
        if (lane == 0) c_star[j] = c != nullptr ? c[j] : 0.0f;  // c* = c exactly when b is absent
      } else {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
        if (lane == 0) {
          const double cj = c != nullptr ? (double)c[j] : 0.0;
          c_star[j] = __double2float_rn(__dadd_rn(cj, acc));
        }
      }
    }
  }
}

template <int DT, bool G, bool B>
static cudaError_t fold_launch_tma(const uint8_t* src, int64_t N, int64_t K, const float* g, const float* b,
                                   const float* c, uint8_t* dst, float* c_star, cudaStream_t stream, int glu_half) {
  constexpr int ES = DT == 0 ? 2 : 4;
  CUtensorMap tm;
  if (!encode_plain_tmap(&tm, src, N, K, ES, k1::SUB / ES, k1::ROWS)) return cudaErrorInvalidValue;
  const void* fptr = (const void*)fold_weights_tma_kernel<DT, G, B>;
  if (cudaError_t e = ensure_smem_attr(fptr, (int)k1::SMEM); e != cudaSuccess) return e;
  const int64_t nblk = (N + k1::ROWS - 1) / k1::ROWS;
  const int grid = (int)std::min<int64_t>(nblk, device_sms());
  fold_weights_tma_kernel<DT, G, B><<<grid, k1::THREADS, k1::SMEM, stream>>>(tm, N, K, g, b, c, dst, c_star,
                                                                             glu_half);
  return cudaGetLastError();
}

template <int DT, bool G, bool B, int RPW, int U, int MINB>
static void fold_launch_v(const uint8_t* src, int64_t N, int64_t K, const float* g, const float* b, const float* c,
                          uint8_t* dst, float* c_star, cudaStream_t stream, int glu_half) {
  const int64_t rows_per_cta = fold::WARPS_PER_CTA * RPW;
  const dim3 grid((unsigned)((N + rows_per_cta - 1) / rows_per_cta));
  fold_weights_kernel<DT, G, B, RPW, U, MINB><<<grid, fold::WARPS_PER_CTA * 32, 0, stream>>>(src, N, K, g, b, c, dst,
                                                                                          c_star, glu_half);
}
// variants (rows per warp, chunks in flight per lane, min CTAs per SM): the c* contract order does
// not depend on them.  A/B knob FN_FOLD_VARIANT; default = the measured best.
template <int DT, bool G, bool B>
static cudaError_t fold_launch(int variant, const uint8_t* src, int64_t N, int64_t K, const float* g,
                               const float* b, const float* c, uint8_t* dst, float* c_star, cudaStream_t stream,
                               int glu_half) {
  // default (variant 0): direct 16-byte loads, (2 rows per warp, 2 chunks in flight per lane, 3
  // CTAs/SM), 97-104 us on the config-3 W with g, b, c (tools/bench_folds.py); variant 9 = the
  // TMA-ring kernel (fold_weights_tma_kernel, 32 KiB boxes through a 192 KiB ring) measured no
  // faster; variants 1, 3-8 = other (rows, chunks, CTAs/SM) shapes, e.g. 1 = (2, 4, 1) 103 us
  switch (variant) {
    case 9: return fold_launch_tma<DT, G, B>(src, N, K, g, b, c, dst, c_star, stream, glu_half);
    case 1: fold_launch_v<DT, G, B, 2, 4, 1>(src, N, K, g, b, c, dst, c_star, stream, glu_half); break;
    case 3: fold_launch_v<DT, G, B, 4, 1, 3>(src, N, K, g, b, c, dst, c_star, stream, glu_half); break;
    case 4: fold_launch_v<DT, G, B, 4, 2, 2>(src, N, K, g, b, c, dst, c_star, stream, glu_half); break;
    case 5: fold_launch_v<DT, G, B, 2, 2, 4>(src, N, K, g, b, c, dst, c_star, stream, glu_half); break;
    case 6: fold_launch_v<DT, G, B, 1, 4, 4>(src, N, K, g, b, c, dst, c_star, stream, glu_half); break;
    case 7: fold_launch_v<DT, G, B, 2, 1, 6>(src, N, K, g, b, c, dst, c_star, stream, glu_half); break;
    case 8: fold_launch_v<DT, G, B, 4, 1, 4>(src, N, K, g, b, c, dst, c_star, stream, glu_half); break;
    default:
      fold_launch_v<DT, G, B, fold::ROWS_PER_WARP, fold::CHUNK_UNROLL, 3>(src, N, K, g, b, c, dst, c_star, stream,
                                                                          glu_half);
  }
  return cudaGetLastError();
}

cudaError_t launch_fold_weights(const void* Wt, int64_t N, int64_t K, int dtype, const float* g, const float* b,
                                const float* c, void* Wt_star, float* c_star, cudaStream_t stream, int glu_half) {
  static const int variant = [] {
    const char* e = getenv("FN_FOLD_VARIANT");
    return e != nullptr ? atoi(e) : 0;
  }();
  const uint8_t* src = static_cast<const uint8_t*>(Wt);
  uint8_t* dst = static_cast<uint8_t*>(Wt_star);
  const bool hg = g != nullptr, hb = b != nullptr;
#define FN_FOLD_LAUNCH(DT, G, B) fold_launch<DT, G, B>(variant, src, N, K, g, b, c, dst, c_star, stream, glu_half)
  if (dtype == 0) {
    if (hg && hb) return FN_FOLD_LAUNCH(0, true, true);
    if (hg) return FN_FOLD_LAUNCH(0, true, false);
    if (hb) return FN_FOLD_LAUNCH(0, false, true);
    return FN_FOLD_LAUNCH(0, false, false);
  }
  if (hg && hb) return FN_FOLD_LAUNCH(1, true, true);
  if (hg) return FN_FOLD_LAUNCH(1, true, false);
  if (hb) return FN_FOLD_LAUNCH(1, false, true);
  return FN_FOLD_LAUNCH(1, false, false);
#undef FN_FOLD_LAUNCH
}

// ------------------------------------------------------------------ K1u: column sums of W*
// u_j = RN_f32( fp64 sum_k W*t[j][k] ) in the c* contract order of K1 (lane l: chunks l, l+32, ...
// ascending, elements ascending; xor butterfly 16..1) — u = 1^T W* for the deferred LayerNorm
// (NEXT-4, reading c29): z = (acc - mu u) r + c*.  One warp per row, 4 chunks in flight per lane.
template <int DT>
__global__ void __launch_bounds__(256)
    colsum_rows_kernel(const uint8_t* __restrict__ Wt, int64_t N, int64_t K, float* __restrict__ u) {
  constexpr int E = DT == 0 ? 8 : 4;
  constexpr int ES = DT == 0 ? 2 : 4;
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= N) return;
  const int64_t nchunks = K / E;
  double acc = 0.0;
  for (int64_t q0 = lane; q0 < nchunks; q0 += 32 * U) {
    uint4 vv[U];
#pragma unroll
    for (int v = 0; v < U; ++v)
      if (q0 + v * 32 < nchunks) vv[v] = ld_nc_v4(Wt + (j * K + (q0 + v * 32) * E) * ES);
#pragma unroll
    for (int v = 0; v < U; ++v) {
      if (q0 + v * 32 >= nchunks) break;
#pragma unroll
      for (int e = 0; e < E; ++e) acc = __dadd_rn(acc, (double)chunk_elem<DT>(vv[v], e));
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
  if (lane == 0) u[j] = __double2float_rn(acc);
}

cudaError_t launch_fold_colsum(const void* Wt_star, int64_t N, int64_t K, int dtype, float* u, cudaStream_t stream) {
  const dim3 grid((unsigned)((N + 7) / 8));
  if (dtype == 0) colsum_rows_kernel<0><<<grid, 256, 0, stream>>>(static_cast<const uint8_t*>(Wt_star), N, K, u);
  else colsum_rows_kernel<1><<<grid, 256, 0, stream>>>(static_cast<const uint8_t*>(Wt_star), N, K, u);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K2

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

// ------------------------------------------------------------------ K2: one launch, clusters of 8 CTAs
// The column sums need every row, the centering needs every column sum: one cluster of 8 CTAs owns
// a 256-byte column slab at a time (128 bf16 / 64 f32 columns), so both the reduction and the
// exchange stay on-chip (DSMEM), with no workspace, atomics or grid-wide waits.
//   CTA j of the cluster owns contract lanes 4j..4j+3 (include/flashnorm.h: lane l sums the 32-row
//   partials of chunks l, l+32, ... ascending).  Its boxes are [128 rows x 256 B] = 32 KiB at rows
//   1024 k + 128 j (k = 0, 1, ...): chunks 4j+q + 32k for q = 0..3, so thread (word w, q) carries
//   lane 4j+q's running sum across its boxes in exactly the contract order.
//   P1: the lane sums go to shared memory; every CTA signals the cluster (remote mbarrier arrive).
//   R:  CTA j gathers the 32 lane sums of its 16 (bf16) / 8 (f32) columns over DSMEM, runs the
//       butterfly tree, mu_i = RN_f32(s_i / n), and writes mu into all 8 CTAs; signals again.
//   P2: V*t = RN_dtype(v - mu) in place in the box (f32 subtraction), one TMA store per box.
// A producer warp streams the boxes through a 6-slot ring (192 KiB); a box stays resident from P1 to
// P2 when the lane group has <= 6 boxes (n_out <= 6144), else P2 re-loads it (from L2).  The next
// slab's boxes load while this slab is centered and stored, so HBM reads and writes overlap.
namespace k2 {
constexpr int CL = 8;                 // CTAs per cluster (portable)
constexpr int CONSUMERS = 256;        // 8 consumer warps
constexpr int THREADS = CONSUMERS + 32;  // + the producer warp
constexpr int SLAB = FOLD_BOX_BYTES;  // 256 bytes of each row per box
constexpr int ROWS = fold::COLSUM_ROWS;
constexpr int QC = 4;                 // row chunks (= lanes) per box
constexpr int BOX_ROWS = ROWS * QC;   // 128
constexpr int WORDS = SLAB / 4;       // 64 four-byte column groups
constexpr int BOX = SLAB * BOX_ROWS;  // 32 KiB (TMA streams near HBM rate only with boxes this large)
constexpr int RES = 6;                // ring slots: 192 KiB
constexpr int LANES = 32;
constexpr size_t SMEM = (size_t)RES * BOX + 128;
}  // namespace k2

struct K2Geom {
  int64_t n_out, d_in;
  int nslab, nchunk, kq;  // kq = boxes per lane group = ceil(nchunk / 32)
  int nclusters;
};


// bounded waits: a lost arrival traps (with a message) after ~2 s instead of hanging the GPU
FN_DEVICE uint64_t k2_gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
FN_DEVICE void k2_wait(uint64_t* bar, uint32_t parity, int what) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = k2_gtime();
  while (!mbar_try_wait(bar, parity)) {
    if (k2_gtime() - t0 > 2000000000ull) {
      printf("fold_mean_center: wait %d timed out (block %d thread %d parity %u)\n", what, (int)blockIdx.x,
             (int)threadIdx.x, parity);
      __trap();
    }
  }
}
FN_DEVICE void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(bar, rank))
               : "memory");
}
FN_DEVICE uint32_t mbar_try_wait_cluster_acq(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok;
}
FN_DEVICE void mbar_wait_cluster_acq(uint64_t* bar, uint32_t parity, int what) {
  if (mbar_try_wait_cluster_acq(bar, parity)) return;
  const uint64_t t0 = k2_gtime();
  while (!mbar_try_wait_cluster_acq(bar, parity)) {
    if (k2_gtime() - t0 > 2000000000ull) {
      printf("fold_mean_center: cluster wait %d timed out (block %d thread %d parity %u)\n", what,
             (int)blockIdx.x, (int)threadIdx.x, parity);
      __trap();
    }
  }
}
FN_DEVICE double ld_cluster_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
FN_DEVICE void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

#ifdef FN_K2_TRACE  // per-CTA globaltimer stamps (ns), tools/micro/k2_trace.cu
__device__ unsigned long long g_k2_trace[160][32];
#define K2_STAMP(i) do { if (threadIdx.x == 0 && blockIdx.x < 160 && (i) < 32) g_k2_trace[blockIdx.x][i] = k2_gtime(); } while (0)
#else
#define K2_STAMP(i)
#endif

template <int DT>
__global__ void __launch_bounds__(k2::THREADS, 1)
    fold_mean_center_kernel(const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_vs,
                            K2Geom g, const float* __restrict__ b_prev, float* __restrict__ b_star) {
  using namespace k2;
  constexpr int E = DT == 0 ? 2 : 1;  // elements per 4-byte group
  constexpr int ES = DT == 0 ? 2 : 4;
  constexpr int CPS = SLAB / ES;      // columns per slab
  constexpr int CPC = CPS / CL;       // columns per CTA in the reduction (16 / 8)
  extern __shared__ __align__(128) uint8_t k2s_raw[];
  uint8_t* slots = k2s_raw + ((128u - (smem_u32(k2s_raw) & 127u)) & 127u);
  __shared__ __align__(8) uint64_t full[RES], empty[RES];
  __shared__ __align__(8) uint64_t lanes_ready, mu_ready;
  __shared__ double lane_sum[QC][CPS];        // this CTA's 4 lane sums per slab column
  __shared__ double gath[LANES][CPC];         // the 32 lane sums of this CTA's reduction columns
  __shared__ float mu_s[CPS];                 // mu of every slab column (written by the 8 CTAs)
  __shared__ double wsum[fold::BPREV_THREADS / 32];
  __shared__ double mean_s;
  const int t = threadIdx.x;
  const uint32_t j = cluster_ctarank();
  const int cid = (int)(blockIdx.x / CL);
  const bool resident = g.kq <= RES;
  const int my_slabs = (g.nslab - cid + g.nclusters - 1) / g.nclusters;
  if (t == 0) {
    for (int i = 0; i < RES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&lanes_ready, CL);
    mbar_init(&mu_ready, CL);
    fence_mbar_init();
  }
  __syncthreads();
  K2_STAMP(0);
  cluster_sync_all();  // every CTA's barriers are initialised before any remote arrive
  K2_STAMP(1);

  if (t >= CONSUMERS) {
    // ---------------------------------------------------------------- producer warp
    if (t == CONSUMERS) {
      prefetch_tmap(&tm_v);
      int n = 0;
      for (int i = 0; i < my_slabs; ++i) {
        const int s = cid + i * g.nclusters;
        const int passes = resident ? 1 : 2;
        for (int pass = 0; pass < passes; ++pass)
          for (int k = 0; k < g.kq; ++k, ++n) {
            const int slot = n % RES;
            if (n >= RES) k2_wait(&empty[slot], (uint32_t)((n / RES) - 1) & 1u, 1);
            mbar_arrive_expect_tx(&full[slot], (uint32_t)BOX);
            tma_load_2d(slots + (size_t)slot * BOX, &tm_v, &full[slot], (int32_t)((int64_t)s * CPS),
                        (int32_t)(k * (LANES * ROWS) + (int)j * BOX_ROWS), pass == 0 ? kEvictLast : kEvictFirst);
          }
      }
    }
    return;
  }
  // ------------------------------------------------------------------ consumers
  if (blockIdx.x == 0 && b_prev != nullptr) {
    // (consumers only: the helper's barriers are CTA-wide, the producer warp has returned)
    const int tb = t;
    double acc = 0.0;
    for (int64_t jj = tb; jj < g.n_out; jj += fold::BPREV_THREADS) acc = __dadd_rn(acc, (double)b_prev[jj]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
    if ((tb & 31) == 0) wsum[tb >> 5] = acc;
    named_bar_sync(1, CONSUMERS);
    if (tb == 0) {
      double tot = 0.0;
      for (int w8 = 0; w8 < fold::BPREV_THREADS / 32; ++w8) tot = __dadd_rn(tot, wsum[w8]);
      mean_s = __ddiv_rn(tot, (double)g.n_out);
    }
    named_bar_sync(1, CONSUMERS);
    for (int64_t jj = tb; jj < g.n_out; jj += fold::BPREV_THREADS)
      b_star[jj] = __double2float_rn(__dsub_rn((double)b_prev[jj], mean_s));
  }
  const int wd = t % WORDS, q = t / WORDS;
  int n = 0;            // loads consumed (same sequence as the producer's)
  int pend_slot = -1;   // thread 0: slot whose TMA store was issued but not yet waited for
  for (int i = 0; i < my_slabs; ++i) {
    const int s = cid + i * g.nclusters;
    const int64_t cg = (int64_t)s * CPS + wd * E;
    const bool col_ok = cg < g.d_in;
    // ---------------------------------------------------------------- P1: lane sums
    double L[E];
#pragma unroll
    for (int e = 0; e < E; ++e) L[e] = 0.0;
    const int n0 = n;
    for (int k = 0; k < g.kq; ++k, ++n) {
      const int slot = n % RES;
      k2_wait(&full[slot], (uint32_t)(n / RES) & 1u, 2);
      if (k == 0) K2_STAMP(6 + 6 * i);
      if (k == g.kq - 1) K2_STAMP(7 + 6 * i);
      const int c = (int)j * QC + q + k * LANES;  // this thread's chunk (lane 4j + q)
      if (c < g.nchunk && col_ok) {
        const int nrows = (int)min((int64_t)ROWS, g.n_out - (int64_t)c * ROWS);
        const uint32_t* colp = reinterpret_cast<const uint32_t*>(slots + (size_t)slot * BOX) + q * ROWS * WORDS + wd;
        double acc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.0;
        uint32_t mark = 0u;
#pragma unroll 8
        for (int rr = 0; rr < nrows; ++rr) {
          const uint32_t x = colp[rr * WORDS];
          mark = inf_nan_mark<DT>(mark, x);
          double d[E];
          widen_word_scaled<DT>(x, d);
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = __dadd_rn(acc[e], d[e]);
        }
        if (inf_nan_seen<DT>(mark)) {  // rare: redo with hardware conversions (inf/NaN propagate)
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = 0.0;
          for (int rr = 0; rr < nrows; ++rr) {
            double d[E];
            widen_word_hw<DT>(colp[rr * WORDS], d);
#pragma unroll
            for (int e = 0; e < E; ++e) acc[e] = __dadd_rn(acc[e], d[e]);
          }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) L[e] = __dadd_rn(L[e], acc[e]);  // partial c added in ascending c
      }
      if (!resident) {
        named_bar_sync(1, CONSUMERS);  // every read of the slot consumed (DADDs above)
        if (t == 0) mbar_arrive(&empty[slot]);
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) lane_sum[q][wd * E + e] = L[e];
    K2_STAMP(2 + 6 * i);
    named_bar_sync(1, CONSUMERS);
    if (t < CL) mbar_arrive_remote(&lanes_ready, (uint32_t)t);  // release: cumulative over the barrier
    // ---------------------------------------------------------------- R: butterfly for CPC columns
    mbar_wait_cluster_acq(&lanes_ready, (uint32_t)i & 1u, 3);
    K2_STAMP(3 + 6 * i);
    for (int idx = t; idx < LANES * CPC; idx += CONSUMERS) {
      const int l = idx / CPC, cc = idx % CPC;
      gath[l][cc] = ld_cluster_f64(mapa_shared(&lane_sum[l % QC][(int)j * CPC + cc], (uint32_t)(l / QC)));
    }
    named_bar_sync(1, CONSUMERS);
    if (t < CPC) {
      double a[LANES];
#pragma unroll
      for (int l = 0; l < LANES; ++l) a[l] = gath[l][t];
#pragma unroll
      for (int off = LANES / 2; off > 0; off >>= 1)
#pragma unroll
        for (int l = 0; l < off; ++l) a[l] = __dadd_rn(a[l], a[l + off]);
      // mu_i = RN_f32(s_i / n) (fp64 division; lane sums 2^-896-scaled)
      const float mu = __double2float_rn(__ddiv_rn(__dmul_rn(a[0], kScaleUp), (double)g.n_out));
#pragma unroll
      for (int r = 0; r < CL; ++r) st_cluster_f32(mapa_shared(&mu_s[(int)j * CPC + t], (uint32_t)r), mu);
    }
    named_bar_sync(1, CONSUMERS);
    if (t < CL) mbar_arrive_remote(&mu_ready, (uint32_t)t);
    mbar_wait_cluster_acq(&mu_ready, (uint32_t)i & 1u, 4);
    K2_STAMP(4 + 6 * i);
    // ---------------------------------------------------------------- P2: center + store
    float mu[E];
#pragma unroll
    for (int e = 0; e < E; ++e) mu[e] = mu_s[wd * E + e];
    for (int k = 0; k < g.kq; ++k) {
      int slot;
      if (resident) {
        slot = (n0 + k) % RES;
      } else {
        slot = n % RES;
        k2_wait(&full[slot], (uint32_t)(n / RES) & 1u, 5);
        ++n;
      }
      const int c = (int)j * QC + q + k * LANES;
      if (c < g.nchunk && col_ok) {
        const int nrows = (int)min((int64_t)ROWS, g.n_out - (int64_t)c * ROWS);
        uint32_t* colp = reinterpret_cast<uint32_t*>(slots + (size_t)slot * BOX) + q * ROWS * WORDS + wd;
#pragma unroll 8
        for (int rr = 0; rr < nrows; ++rr) {
          const uint32_t x = colp[rr * WORDS];
          if (DT == 0) colp[rr * WORDS] = pack_bf16(__fsub_rn(bf16lo(x), mu[0]), __fsub_rn(bf16hi(x), mu[E - 1]));
          else colp[rr * WORDS] = __float_as_uint(__fsub_rn(__uint_as_float(x), mu[0]));
        }
      }
      fence_proxy_async_smem();  // generic-proxy SMEM writes -> visible to the TMA store
      named_bar_sync(1, CONSUMERS);
      if (t == 0) {
        tma_store_2d(&tm_vs, slots + (size_t)slot * BOX, (int32_t)((int64_t)s * CPS),
                     (int32_t)(k * (LANES * ROWS) + (int)j * BOX_ROWS));
        bulk_commit_group();
        // the previous store has read its slot (at most one store group in flight): release it
        if (pend_slot >= 0) {
          bulk_wait_read1();
          mbar_arrive(&empty[pend_slot]);
        }
        pend_slot = slot;
      }
    }
    K2_STAMP(5 + 6 * i);
    // release the slab's last slot now (the next slab's loads may need every slot)
    if (t == 0 && pend_slot >= 0) {
      bulk_wait_read();
      mbar_arrive(&empty[pend_slot]);
      pend_slot = -1;
    }
  }
  K2_STAMP(30);
  if (t == 0) {
    bulk_wait_all();  // every box store is complete before the CTA retires
    if (pend_slot >= 0) mbar_arrive(&empty[pend_slot]);
  }
}

static cudaError_t launch_fold_mean_center_cluster(const CUtensorMap& tm_v, const CUtensorMap& tm_vs,
                                                  int64_t n_out, int64_t d_in, int dtype, const float* b_prev,
                                                  float* b_prev_star, cudaStream_t stream, int* launches) {
  const int es = dtype == 0 ? 2 : 4;
  K2Geom g;
  g.n_out = n_out;
  g.d_in = d_in;
  g.nslab = (int)((d_in * es + k2::SLAB - 1) / k2::SLAB);
  const int64_t nchunk = (n_out + fold::COLSUM_ROWS - 1) / fold::COLSUM_ROWS;
  if (nchunk > INT32_MAX / 2) return cudaErrorInvalidValue;
  g.nchunk = (int)nchunk;
  g.kq = (int)((nchunk + k2::LANES - 1) / k2::LANES);
  const void* fptr = dtype == 0 ? (const void*)fold_mean_center_kernel<0> : (const void*)fold_mean_center_kernel<1>;
  if (cudaError_t e = ensure_smem_attr(fptr, (int)k2::SMEM); e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(k2::THREADS);
  cfg.dynamicSmemBytes = k2::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = k2::CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // as many co-resident clusters as fit (a cluster loops over its slabs), at most one per slab
  int maxc = 0;
  cfg.gridDim = dim3(k2::CL * 64);
  if (cudaError_t e = cudaOccupancyMaxActiveClusters(&maxc, fptr, &cfg); e != cudaSuccess) return e;
  if (maxc < 1) return cudaErrorInvalidConfiguration;
  g.nclusters = std::min(maxc, g.nslab);
  cfg.gridDim = dim3(k2::CL * g.nclusters);
  *launches = 1;
  if (dtype == 0) return cudaLaunchKernelEx(&cfg, fold_mean_center_kernel<0>, tm_v, tm_vs, g, b_prev, b_prev_star);
  return cudaLaunchKernelEx(&cfg, fold_mean_center_kernel<1>, tm_v, tm_vs, g, b_prev, b_prev_star);
}

// ------------------------------------------------------------------ K2, three launches (default)
// pass 1: fp64 32-row partials -> workspace; 1b: s_i in the contract order + b_prev*; 2: V*t
namespace fold {
constexpr int K2_THREADS = 256;               // K2 passes 1/2: one 4-byte column group per thread
constexpr int K2_TILE_BYTES = K2_THREADS * 4;  // bytes of each row per CTA tile
}  // namespace fold
constexpr int K2_BOX_BYTES_3K = 512;          // tm_v box of the three-launch K2: 512 B x 32 rows
// pass 1b: s_i in the contract order — lane-sum l (l = 0..31) is the ascending sum of the
// partials c = l, l+32, ..., and the 32 lane sums are combined as the xor butterfly
// 16,8,4,2,1 leaves them in lane 0, i.e. the tree  a[l] += a[l+off] for l < off,
// off = 16,8,4,2,1 (fp addition commutes, so a[l] + a[l^off] is the same number on both
// lanes of a butterfly pair).  Mapping for coalesced loads: a CTA owns 32 columns, lane j
// -> column, warp w (of 8) -> lane-sums l = w, w+8, w+16, w+24; offs 16 and 8 stay in the
// thread, offs 4,2,1 go through SMEM.  mu_i = s_i / n.  The extra last CTA centers b_prev
// (independent work, same launch).
__global__ void __launch_bounds__(fold::BPREV_THREADS)
    colsum_reduce_kernel(const double* __restrict__ partial, int64_t nchunk, int64_t d_in, int64_t n_out,
                         double* __restrict__ mu, const float* __restrict__ b_prev, float* __restrict__ b_star) {
  __shared__ double wsum[fold::BPREV_THREADS / 32];
  __shared__ double mean_s;
  __shared__ double lsum[8][33];
  pdl_wait_prior_grid();  // launched with programmatic stream serialization after pass 1
  pdl_launch_dependents();
  const int64_t ncol_blocks = (d_in + 31) / 32;
  if ((int64_t)blockIdx.x == ncol_blocks) {
    if (b_prev != nullptr) center_bias_block(b_prev, n_out, b_star, wsum, &mean_s);
    return;
  }
  const int j = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + j;
  double a[4] = {0.0, 0.0, 0.0, 0.0};  // lane-sums l = w + 8q
  constexpr int RB = 4;                // rounds of 32 partials with loads in flight together
  if (i < d_in) {
    for (int64_t c0 = 0; c0 < nchunk; c0 += 32 * RB) {
      double v[RB][4];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t c = c0 + 32 * rb + w + 8 * q;
          v[rb][q] = c < nchunk ? __ldcg(partial + c * d_in + i) : 0.0;
        }
#pragma unroll
      for (int rb = 0; rb < RB; ++rb)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (c0 + 32 * rb + w + 8 * q < nchunk) a[q] = __dadd_rn(a[q], v[rb][q]);
    }
  }
  a[0] = __dadd_rn(a[0], a[2]);  // off 16: l = w, w+8 take l+16
  a[1] = __dadd_rn(a[1], a[3]);
  a[0] = __dadd_rn(a[0], a[1]);  // off 8: l = w takes l+8
  lsum[w][j] = a[0];
  __syncthreads();
  if (w == 0 && i < d_in) {
    double t[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) t[l] = lsum[l][j];
#pragma unroll
    for (int off = 4; off > 0; off >>= 1)
#pragma unroll
      for (int l = 0; l < off; ++l) t[l] = __dadd_rn(t[l], t[l + off]);
    mu[i] = __ddiv_rn(__dmul_rn(t[0], kScaleUp), (double)n_out);  // partials are 2^-896-scaled
  }
}

// Passes 1 and 2 stream [32 rows x 1 KiB] tiles of Vt through SMEM with TMA (two 2-D boxes
// of 512 B x 32 rows per tile, no swizzle, completing on the stage's mbarrier): a persistent
// grid of 3 CTAs per SM, each double-buffering 2 x 32 KiB, so the next tile is in flight
// while the current one is summed (pass 1) or centered and stored (pass 2).  Thread t owns
// the 4-byte column group t of a tile: box t / 128, byte (t % 128) * 4 of each box row.
template <int DT, bool CENTER>
__global__ void __launch_bounds__(fold::K2_THREADS)
    k2_tiles_kernel(const __grid_constant__ CUtensorMap tm_v, int64_t n_out, int64_t d_in, int ntiles_x, int ntiles,
                    double* __restrict__ partial, const double* __restrict__ mu_g, uint8_t* __restrict__ Vt_star) {
  constexpr int E = DT == 0 ? 2 : 1;  // elements per 4-byte group
  constexpr int ES = DT == 0 ? 2 : 4;
  constexpr int BOX_COLS = K2_BOX_BYTES_3K / ES;
  constexpr int BOX_SMEM = K2_BOX_BYTES_3K * fold::COLSUM_ROWS;
  constexpr int STAGE_SMEM = fold::COLSUM_ROWS * fold::K2_TILE_BYTES;
  extern __shared__ __align__(128) uint8_t k2_smem[];  // [2 stages][2 boxes][COLSUM_ROWS][K2_BOX_BYTES_3K]
  __shared__ __align__(8) uint64_t bar[2];
  const int64_t row_bytes = d_in * ES;
  const int t = threadIdx.x;
  auto tile_geom = [&](int tile, int64_t& c0b, uint32_t& seg, int64_t& j0, int& nrows) {
    c0b = (int64_t)(tile % ntiles_x) * fold::K2_TILE_BYTES;
    seg = (uint32_t)min((int64_t)fold::K2_TILE_BYTES, row_bytes - c0b);
    j0 = (int64_t)(tile / ntiles_x) * fold::COLSUM_ROWS;
    nrows = (int)min((int64_t)fold::COLSUM_ROWS, n_out - j0);
  };
  auto issue = [&](int tile, int stage) {
    int64_t c0b, j0;
    uint32_t seg;
    int nrows;
    tile_geom(tile, c0b, seg, j0, nrows);
    const int nbox = seg > (uint32_t)K2_BOX_BYTES_3K ? 2 : 1;  // out-of-range rows/cols are zero-filled
    uint8_t* dst = k2_smem + stage * STAGE_SMEM;
    mbar_arrive_expect_tx(&bar[stage], (uint32_t)(nbox * BOX_SMEM));
    // pass 1 keeps Vt in L2 for pass 2 (config 4: 33.5 MB < 126 MB); pass 2 is its last use
    for (int b = 0; b < nbox; ++b)
      tma_load_2d(dst + b * BOX_SMEM, &tm_v, &bar[stage], (int32_t)(c0b / ES + b * BOX_COLS), (int32_t)j0,
                  CENTER ? kEvictFirst : kEvictLast);
  };
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0) {  // Vt is never written by the fold kernels: prefetch before any PDL wait
    if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  if (CENTER) pdl_wait_prior_grid();  // mu_g comes from the reduce kernel
  else pdl_launch_dependents();
  int k = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int stage = k & 1;
    int64_t c0b, j0;
    uint32_t seg;
    int nrows;
    tile_geom(tile, c0b, seg, j0, nrows);
    mbar_wait(&bar[stage], (uint32_t)(k >> 1) & 1u);
    const uint8_t* src = k2_smem + stage * STAGE_SMEM + (t >> 7) * BOX_SMEM + (t & 127) * 4;
    if ((uint32_t)t * 4 < seg) {
      const int64_t col0 = c0b / ES + t * E;
      const uint32_t* col = reinterpret_cast<const uint32_t*>(src);
      constexpr int RW = K2_BOX_BYTES_3K / 4;  // words per box row
      uint32_t mark = 0u;
      if (!CENTER) {
        // partial sums in the 2^-896-scaled domain (exactly equivalent, see widen_scaled_hi)
        double acc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.0;
#pragma unroll 8
        for (int r = 0; r < nrows; ++r) {
          const uint32_t v = col[r * RW];
          mark = inf_nan_mark<DT>(mark, v);
          double d[E];
          widen_word_scaled<DT>(v, d);
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = __dadd_rn(acc[e], d[e]);
        }
        if (inf_nan_seen<DT>(mark)) {  // rare: redo with hardware conversions (inf/NaN propagate)
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = 0.0;
          for (int r = 0; r < nrows; ++r) {
            double d[E];
            widen_word_hw<DT>(col[r * RW], d);
#pragma unroll
            for (int e = 0; e < E; ++e) acc[e] = __dadd_rn(acc[e], d[e]);
          }
        }
        double* out = partial + (j0 / fold::COLSUM_ROWS) * d_in + col0;
#pragma unroll
        for (int e = 0; e < E; ++e) out[e] = acc[e];
      } else {
        // V*t = RN_dtype(v - mu_i) in f32, mu_i = RN_f32(s_i / n) (reading c21); IEEE f32: inf/NaN propagate
        float mu[E];
#pragma unroll
        for (int e = 0; e < E; ++e) mu[e] = __double2float_rn(mu_g[col0 + e]);
        uint8_t* dst = Vt_star + (j0 * d_in + col0) * ES;
#pragma unroll 8
        for (int r = 0; r < nrows; ++r) {
          const uint32_t v = col[r * RW];
          const uint32_t o = DT == 0 ? pack_bf16(__fsub_rn(bf16lo(v), mu[0]), __fsub_rn(bf16hi(v), mu[E - 1]))
                                     : __float_as_uint(__fsub_rn(__uint_as_float(v), mu[0]));
          *reinterpret_cast<uint32_t*>(dst + (int64_t)r * d_in * ES) = o;
        }
        (void)mark;
      }
    }
    // Every value read from this stage has been consumed by an issued DADD/DSUB above
    // (in-order issue), so after the barrier no LDS of the stage is outstanding.
    __syncthreads();
    if (t == 0 && tile + 2 * (int)gridDim.x < ntiles) issue(tile + 2 * gridDim.x, stage);
  }
}

static cudaError_t launch_fold_mean_center_3k(const CUtensorMap& tm_v, int64_t n_out, int64_t d_in, int dtype,
                                             const float* b_prev, void* Vt_star, float* b_prev_star,
                                             void* workspace, cudaStream_t stream, int* launches) {
  const int64_t row_bytes = d_in * (dtype == 0 ? 2 : 4);
  const int64_t nchunk = (n_out + fold::COLSUM_ROWS - 1) / fold::COLSUM_ROWS;
  const int ntiles_x = (int)((row_bytes + fold::K2_TILE_BYTES - 1) / fold::K2_TILE_BYTES);
  const int64_t ntiles64 = (int64_t)ntiles_x * nchunk;
  if (ntiles64 > INT32_MAX) return cudaErrorInvalidValue;
  const int ntiles = (int)ntiles64;
  double* partial = static_cast<double*>(workspace);
  uint8_t* dst = static_cast<uint8_t*>(Vt_star);
  double* mu = partial + nchunk * d_in;
  const unsigned rgrid = (unsigned)((d_in + 31) / 32 + 1);  // + the b_prev CTA
  constexpr size_t smem = 2 * fold::COLSUM_ROWS * fold::K2_TILE_BYTES;
  const int sms = device_sms();
  for (const void* f : {(const void*)k2_tiles_kernel<0, false>, (const void*)k2_tiles_kernel<0, true>,
                        (const void*)k2_tiles_kernel<1, false>, (const void*)k2_tiles_kernel<1, true>})
    if (cudaError_t e = ensure_smem_attr(f, (int)smem); e != cudaSuccess) return e;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * 3);
  // pass 1 in plain stream order; the reduce and pass 2 with programmatic dependent launch
  // (griddepcontrol.wait before they read the previous pass's output) to hide launch gaps.
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t rcfg = {};
  rcfg.gridDim = dim3(rgrid);
  rcfg.blockDim = dim3(fold::BPREV_THREADS);
  rcfg.stream = stream;
  rcfg.attrs = pdl;
  rcfg.numAttrs = 1;
  cudaLaunchConfig_t ccfg = rcfg;
  ccfg.gridDim = dim3(grid);
  ccfg.blockDim = dim3(fold::K2_THREADS);
  ccfg.dynamicSmemBytes = smem;
  const int64_t no = n_out, di = d_in;
  const int ntx = ntiles_x, nt = ntiles;
  double* const no_partial = nullptr;
  const double* const no_mu = nullptr;
  uint8_t* const no_dst = nullptr;
  cudaError_t e;
  if (dtype == 0) {
    k2_tiles_kernel<0, false><<<grid, fold::K2_THREADS, smem, stream>>>(tm_v, no, di, ntx, nt, partial, no_mu, no_dst);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&rcfg, colsum_reduce_kernel, (const double*)partial, nchunk, di, no, mu, b_prev,
                           b_prev_star);
    if (e != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&ccfg, k2_tiles_kernel<0, true>, tm_v, no, di, ntx, nt, no_partial, (const double*)mu, dst);
  } else {
    k2_tiles_kernel<1, false><<<grid, fold::K2_THREADS, smem, stream>>>(tm_v, no, di, ntx, nt, partial, no_mu, no_dst);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&rcfg, colsum_reduce_kernel, (const double*)partial, nchunk, di, no, mu, b_prev,
                           b_prev_star);
    if (e != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&ccfg, k2_tiles_kernel<1, true>, tm_v, no, di, ntx, nt, no_partial, (const double*)mu, dst);
  }
  *launches = 3;
  return e;
}


// ------------------------------------------------------------------ K2, one persistent launch (default when it fits)
// One CTA per SM, all co-resident (cooperative launch), V read from HBM exactly once and V* written
// once: every CTA TMA-loads ALL of its [32 rows x 512 B] tiles into shared memory at entry (up to 14
// tiles = 224 KiB in flight per SM — the whole 4096^2 bf16 V of config 4 fits in 148 SMs' SMEM), so
// the read phase streams at full HBM rate from the first cycle.  Then
//   P1  thread (word, tile) sums its tile's 32 rows in fp64 (the 32-row partial of the contract)
//       -> workspace partial[c][i];                                      grid.sync()
//   R   warp per column i, lane l = contract lane l: sums partial[c][i], c = l, l+32, ... ascending,
//       xor butterfly 16..1 with shuffles (exactly the contract tree), mu_i = RN_f32(s_i / n) ->
//       workspace;                                                       grid.sync()
//   P2  v* = RN_dtype(v -_f32 mu_i) in place in the resident tiles, one TMA store per tile.
// Same contract and bits as the three-launch K2 (include/flashnorm.h); b_prev* by the last CTA.
namespace k2p {
constexpr int THREADS = 512;
constexpr int GROUPS = THREADS / 128;    // tile groups of 128 threads (one 4-byte column word each)
constexpr int TW = 512;                  // bytes of each row per tile (= the three-launch box)
constexpr int ROWS = 32;                 // fold::COLSUM_ROWS (rows per partial)
constexpr int RES_BYTES = 14 * TW * ROWS;  // 224 KiB of resident tiles per CTA
constexpr size_t SMEM = (size_t)RES_BYTES + 128;
}  // namespace k2p

// R phase of the persistent K2 (contract order, see the comment inside)
FN_DEVICE void k2p_column_means(const double* __restrict__ partial, float* __restrict__ mu_g, int64_t n_out,
                                int64_t d_in, int nchunk, int b, int G) {
  constexpr int THREADS = k2p::THREADS;
  const int t = threadIdx.x;
  // A warp owns 8 columns; thread (k = lane & 7, q = lane >> 3) holds contract lanes l = 8q + u, u = 0..7,
  // of column 8cb + k: each loads partial[32m + 8q + u][i] (8 consecutive columns = 64 B per row
  // segment, all loads of a round in flight), adds them in ascending m (a missing partial adds +0.0:
  // exact, a lane sum starts at +0.0 and is never -0.0); the butterfly's offsets 16 and 8 pair lanes
  // of threads lane^16 / lane^8 (shuffles), offsets 4, 2, 1 pair values inside the thread — the
  // contract tree a[l] += a[l + off], bit for bit (fp addition commutes).
  {
    const int lane = t & 31, k = lane & 7, q = lane >> 3;
    // warp-major across CTAs: column blocks spread over every SM (per-SM load concurrency)
    const int64_t gw = (int64_t)(t >> 5) * G + b, nw = (int64_t)G * (THREADS / 32);
    for (int64_t cb = gw; cb * 8 < d_in; cb += nw) {
      const int64_t i = cb * 8 + k;
      const bool ok = i < d_in;
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = 0.0;
      // rounds of 32 chunks, 4 rounds' loads (32 per thread) issued before any of them is added:
      // one L2 round trip per 4 rounds instead of one per round (config 4: 128 chunks = 4 rounds)
      for (int m0 = 0; m0 < nchunk; m0 += 4 * 32) {
        double v[4][8];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = m0 + 32 * m + 8 * q + u;
            v[m][u] = (ok && c < nchunk) ? __ldcg(partial + (int64_t)c * d_in + i) : 0.0;
          }
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int u = 0; u < 8; ++u) a[u] = __dadd_rn(a[u], v[m][u]);  // ascending chunk per lane
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __dadd_rn(a[u], __shfl_xor_sync(0xffffffffu, a[u], 16));
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __dadd_rn(a[u], __shfl_xor_sync(0xffffffffu, a[u], 8));
#pragma unroll
      for (int off = 4; off > 0; off >>= 1)
#pragma unroll
        for (int u = 0; u < off; ++u) a[u] = __dadd_rn(a[u], a[u + off]);
      if (q == 0 && ok) mu_g[i] = __double2float_rn(__ddiv_rn(__dmul_rn(a[0], kScaleUp), (double)n_out));
    }
  }
}

// b_prev* = b_prev - mean(b_prev) in the contract order (first 256 threads; reading c7)
FN_DEVICE void k2p_center_bias(const float* __restrict__ b_prev, int64_t n_out, float* __restrict__ b_star,
                               double* wsum, double* mean_s) {
  const int t = threadIdx.x;
  if (t < fold::BPREV_THREADS) {
    double acc = 0.0;
    for (int64_t jj = t; jj < n_out; jj += fold::BPREV_THREADS) acc = __dadd_rn(acc, (double)b_prev[jj]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
    if ((t & 31) == 0) wsum[t >> 5] = acc;
  }
  __syncthreads();
  if (t == 0) {
    double tot = 0.0;
    for (int w8 = 0; w8 < fold::BPREV_THREADS / 32; ++w8) tot = __dadd_rn(tot, wsum[w8]);
    *mean_s = __ddiv_rn(tot, (double)n_out);
  }
  __syncthreads();
  for (int64_t jj = t; jj < n_out; jj += blockDim.x)
    b_star[jj] = __double2float_rn(__dsub_rn((double)b_prev[jj], *mean_s));
}

template <int DT, int TR>
__global__ void __launch_bounds__(k2p::THREADS, 1)
    fold_mean_center_persist_kernel(const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_vs,
                                    int64_t n_out, int64_t d_in, int nchunk, int ntx, int ntiles, int order,
                                    double* __restrict__ partial, float* __restrict__ mu_g,
                                    const float* __restrict__ b_prev, float* __restrict__ b_star) {
  using namespace k2p;
  constexpr int E = DT == 0 ? 2 : 1;  // elements per 4-byte word
  constexpr int ES = DT == 0 ? 2 : 4;
  constexpr int TCOLS = TW / ES;      // columns per tile
  constexpr int RW = TW / 4;          // words per tile row
  constexpr int TILE = TW * TR;       // tile: TR rows (TR / 32 partial chunks) x 512 B
  constexpr int HALVES = TR / ROWS;
  extern __shared__ __align__(128) uint8_t k2p_raw[];
  uint8_t* tiles = k2p_raw + ((128u - (smem_u32(k2p_raw) & 127u)) & 127u);
  __shared__ __align__(8) uint64_t full[RES_BYTES / (TW * ROWS)];
  __shared__ double wsum[fold::BPREV_THREADS / 32];
  __shared__ double mean_s;
  const int t = threadIdx.x;
  const int G = (int)gridDim.x;
  const int b = (int)blockIdx.x;
  const int t0 = (int)((int64_t)ntiles * b / G), t1 = (int)((int64_t)ntiles * (b + 1) / G);
  const int nt = t1 - t0;  // <= MAXT (host-checked)
  // tile index -> (band c of TR rows, column tile x): order 1 = band-major (a CTA reads whole bands:
  // contiguous DRAM rows), order 0 = column-tile-major
  const int nband = (nchunk + HALVES - 1) / HALVES;
  auto tile_cx = [&](int ti, int& c, int& x) {
    if (order) {
      c = ti / ntx;
      x = ti - c * ntx;
    } else {
      x = ti / nband;
      c = ti - x * nband;
    }
  };
  K2_STAMP(0);
  if (t == 0) {
    for (int j = 0; j < nt; ++j) mbar_init(&full[j], 1);
    fence_mbar_init();
    prefetch_tmap(&tm_v);
    prefetch_tmap(&tm_vs);
    for (int j = 0; j < nt; ++j) {
      int c, x;
      tile_cx(t0 + j, c, x);
      mbar_arrive_expect_tx(&full[j], (uint32_t)TILE);
      tma_load_2d(tiles + (size_t)j * TILE, &tm_v, &full[j], x * TCOLS, c * TR, kEvictFirst);
    }
  }
  __syncthreads();
  K2_STAMP(1);
  cg::grid_group grid = cg::this_grid();
  const int w = t & 127, grp = t >> 7;
  // ---------------------------------------------------------------- P1: 32-row fp64 partials
  for (int it = grp; it < nt * HALVES; it += GROUPS) {
    const int j = it / HALVES, h = it - j * HALVES;
    int cb, x;
    tile_cx(t0 + j, cb, x);
    const int c = cb * HALVES + h;  // the 32-row partial chunk
    k2_wait(&full[j], 0u, 7);  // bounded: a lost TMA completion traps instead of hanging the GPU
    if (it == 0) K2_STAMP(2);
    const int64_t col0 = (int64_t)x * TCOLS + w * E;
    if (col0 < d_in && c < nchunk) {
      const int nrows = (int)min((int64_t)ROWS, n_out - (int64_t)c * ROWS);
      const uint32_t* col = reinterpret_cast<const uint32_t*>(tiles + (size_t)j * TILE) + h * ROWS * RW + w;
      double acc[E];
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = 0.0;
      uint32_t mark = 0u;
#pragma unroll 8
      for (int r = 0; r < nrows; ++r) {
        const uint32_t v = col[r * RW];
        mark = inf_nan_mark<DT>(mark, v);
        double d[E];
        widen_word_scaled<DT>(v, d);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = __dadd_rn(acc[e], d[e]);
      }
      if (inf_nan_seen<DT>(mark)) {  // rare: redo with hardware conversions (inf/NaN propagate)
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.0;
        for (int r = 0; r < nrows; ++r) {
          double d[E];
          widen_word_hw<DT>(col[r * RW], d);
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = __dadd_rn(acc[e], d[e]);
        }
      }
      double* out = partial + (int64_t)c * d_in + col0;
#pragma unroll
      for (int e = 0; e < E; ++e) out[e] = acc[e];
    }
  }
  K2_STAMP(3);
  grid.sync();
  K2_STAMP(4);
  // ---------------------------------------------------------------- R: warp per column, lane = contract lane
  k2p_column_means(partial, mu_g, n_out, d_in, nchunk, b, G);
  K2_STAMP(5);
  grid.sync();
  K2_STAMP(6);
  // ---------------------------------------------------------------- P2: center in place, TMA store
  for (int j = grp; j < nt; j += GROUPS) {
    int c, x;
    tile_cx(t0 + j, c, x);
    const int64_t col0 = (int64_t)x * TCOLS + w * E;
    if (col0 < d_in) {
      float mu[E];
#pragma unroll
      for (int e = 0; e < E; ++e) mu[e] = __ldcg(mu_g + col0 + e);
      uint32_t* col = reinterpret_cast<uint32_t*>(tiles + (size_t)j * TILE) + w;
#pragma unroll 8
      for (int r = 0; r < TR; ++r) {  // rows past n_out are zero fill: the TMA store clips them
        const uint32_t v = col[r * RW];
        col[r * RW] = DT == 0 ? pack_bf16(__fsub_rn(bf16lo(v), mu[0]), __fsub_rn(bf16hi(v), mu[E - 1]))
                              : __float_as_uint(__fsub_rn(__uint_as_float(v), mu[0]));
      }
    }
    fence_proxy_async_smem();  // generic-proxy SMEM writes -> visible to the TMA store
    named_bar_sync(1 + grp, 128);
    if (w == 0) {
      tma_store_2d(&tm_vs, tiles + (size_t)j * TILE, x * TCOLS, c * TR);
      bulk_commit_group();
    }
  }
  K2_STAMP(7);
  if (b == G - 1 && b_prev != nullptr) k2p_center_bias(b_prev, n_out, b_star, wsum, &mean_s);
  if (w == 0) bulk_wait_read();  // the tiles stay valid until their stores have read them
  K2_STAMP(8);
}

// grid for the persistent K2 (0 = does not fit: a CTA would need more resident tiles than fit)
static int k2p_grid(int64_t n_out, int64_t d_in, int dtype, int tr, int* ntx_out, int* nchunk_out, int* ntiles_out) {
  const int64_t row_bytes = d_in * (dtype == 0 ? 2 : 4);
  const int64_t nchunk = (n_out + k2p::ROWS - 1) / k2p::ROWS;
  const int64_t nband = (n_out + tr - 1) / tr;
  const int64_t ntx = (row_bytes + k2p::TW - 1) / k2p::TW;
  const int64_t ntiles = nband * ntx;
  const int64_t sms = device_sms();
  const int64_t maxt = k2p::RES_BYTES / (k2p::TW * tr);
  if (ntiles > maxt * sms || ntiles > INT32_MAX) return 0;
  *ntx_out = (int)ntx;
  *nchunk_out = (int)nchunk;
  *ntiles_out = (int)ntiles;
  return (int)std::min<int64_t>(sms, ntiles);
}

static int k2p_tile_rows() {
  static const int tr = [] {
    const char* e = getenv("FN_K2P_TR");  // A/B knob: rows per resident tile (32 or 64)
    const int v = e != nullptr ? atoi(e) : 64;
    return v == 32 ? 32 : 64;
  }();
  return tr;
}

static cudaError_t launch_fold_mean_center_persist(const void* Vt, void* Vt_star, int grid, int tr, int ntx,
                                                   int nchunk, int ntiles, int64_t n_out, int64_t d_in, int dtype,
                                                   const float* b_prev, float* b_prev_star, void* workspace,
                                                   cudaStream_t stream, int* launches) {
  const int es = dtype == 0 ? 2 : 4;
  CUtensorMap tm_v, tm_vs;
  if (!encode_plain_tmap(&tm_v, Vt, n_out, d_in, es, k2p::TW / es, tr) ||
      !encode_plain_tmap(&tm_vs, Vt_star, n_out, d_in, es, k2p::TW / es, tr))
    return cudaErrorInvalidValue;
  const void* fptr = dtype == 0 ? (tr == 64 ? (const void*)fold_mean_center_persist_kernel<0, 64>
                                            : (const void*)fold_mean_center_persist_kernel<0, 32>)
                                : (tr == 64 ? (const void*)fold_mean_center_persist_kernel<1, 64>
                                            : (const void*)fold_mean_center_persist_kernel<1, 32>);
  if (cudaError_t e = ensure_smem_attr(fptr, (int)k2p::SMEM); e != cudaSuccess) return e;
  double* partial = static_cast<double*>(workspace);
  float* mu = reinterpret_cast<float*>(partial + (int64_t)nchunk * d_in);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(k2p::THREADS);
  cfg.dynamicSmemBytes = k2p::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: grid.sync() is legal
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  *launches = 1;
  static const int order = [] {
    const char* e = getenv("FN_K2P_ORDER");  // A/B knob: tile order, 1 = band-major, 0 = column-tile-major
    return e != nullptr ? atoi(e) : 1;
  }();
  void* args[] = {(void*)&tm_v, (void*)&tm_vs, (void*)&n_out, (void*)&d_in, (void*)&nchunk, (void*)&ntx,
                  (void*)&ntiles, (void*)&order, (void*)&partial, (void*)&mu, (void*)&b_prev, (void*)&b_prev_star};
  return cudaLaunchKernelExC(&cfg, fptr, args);
}

int64_t fold_mean_center_workspace(int64_t n_out, int64_t d_in) {
  const int64_t nchunk = (n_out + fold::COLSUM_ROWS - 1) / fold::COLSUM_ROWS;
  return (nchunk + 1) * d_in * (int64_t)sizeof(double);  // partials + s_i/n
}

// Variant (A/B knob FN_K2_VARIANT, read once): 0 = the three-launch K2 (default), 1 = the one-launch
// cluster K2 (no workspace).  Both implement the same contract, bit for bit (tests/test_gpu_parity.py
// runs both).  Measured (tools/bench_folds.py, 6 rotating V, graph): 4096^2 22.8 vs 30.5 us,
// 8192^2 76 vs 95 us — the cluster kernel's column slabs run in ~15 co-resident clusters, three
// sequential slab rounds, and its read / reduce / write phases do not overlap.
cudaError_t launch_fold_mean_center(const CUtensorMap& tm_v3, const CUtensorMap& tm_v, const CUtensorMap& tm_vs,
                                    const void* Vt, int64_t n_out, int64_t d_in, int dtype, const float* b_prev,
                                    void* Vt_star, float* b_prev_star, void* workspace, cudaStream_t stream,
                                    int* launches) {
  static const int variant = [] {
    const char* e = getenv("FN_K2_VARIANT");
    return e != nullptr ? atoi(e) : 0;
  }();
  if (variant == 1) return launch_fold_mean_center_cluster(tm_v, tm_vs, n_out, d_in, dtype, b_prev, b_prev_star,
                                                          stream, launches);
  int ntx = 0, nchunk = 0, ntiles = 0;
  const int tr = k2p_tile_rows();
  const int pgrid = variant == 3 ? 0 : k2p_grid(n_out, d_in, dtype, tr, &ntx, &nchunk, &ntiles);
  if (pgrid > 0) {
    const cudaError_t e = launch_fold_mean_center_persist(Vt, Vt_star, pgrid, tr, ntx, nchunk, ntiles, n_out, d_in,
                                                          dtype, b_prev, b_prev_star, workspace, stream, launches);
    // a cooperative launch the device refuses (e.g. too few co-resident CTAs under MPS limits) falls
    // back to the three launches, which need no co-residency; any other error is reported
    if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported) return e;
    (void)cudaGetLastError();
  }
  return launch_fold_mean_center_3k(tm_v3, n_out, d_in, dtype, b_prev, Vt_star, b_prev_star, workspace, stream,
                                    launches);
}

}  // namespace fn
