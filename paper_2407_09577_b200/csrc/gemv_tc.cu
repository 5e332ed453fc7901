// gemv_tc.cu — K4: decode-shaped FlashNorm linear (M <= 16 tokens) on the tcgen05 tensor core.
//
//   z[m][j] = RN( fma( sum_k a[m][k] W*t[j][k], r_m, c*_j ) ),  r_m = rsqrt(ssq_m/K + eps)
//   (Fig 1(c); the RMS is reduced beside the contraction, Fig 8(c))
//
// Decode is HBM-bound: the whole cost is streaming W* once.  The earlier mma.sync design
// split K over 15 warps and reduced every 8-row tile across warps through SMEM; on sm_100a
// that cross-warp reduction, not HBM, set the rate (~4 TB/s even with W* L2-resident,
// tools/decode_l2.py).  Here the contraction is "swap-AB" on tcgen05:
//
//   D[128 rows of W* x 16 tokens] (TMEM, fp32) += W*[128 x 16k] . a^T[16k x 16]
//
// one tcgen05.mma.cta_group::1 M=128 N=16 K=16 per 16 k, issued by one thread, accumulating
// over K in TMEM — no cross-warp reduction at all.  Work split: tile = 128 W* rows; each tile's
// K range is split over S CTAs (S*tiles <= #SMs, one tile-slice per CTA, so there is no tail
// and no scheduler).  The S partial accumulators (8 KiB each) and partial ssq vectors are
// summed in fixed rank order (deterministic):
//   * cluster mode (preferred): the S CTAs of a tile form a thread-block cluster and store their
//     partials into the leader's SMEM (DSMEM), one cluster barrier (~1 us tail).  S is the
//     largest size whose clusters are all co-resident: GPC shapes cap clusters of 3 at 45 on this
//     part, so config 2 (48 tiles) runs 48 clusters of 2;
//   * global mode (no cluster size > 1 fits): partials go to an L2-resident buffer and the CTA
//     arriving last on the tile's counter reduces (measured ~4 us tail, slower).
//
// Per CTA (192 threads): warp 0 TMA producer (W* [128 x 64] SW128 16 KiB + tokens [16 x 64]
// SW128 2 KiB per stage, 12-stage ring); warp 1 TMEM allocator + MMA issuer; warp 2 side warp
// (RMS: per-token partial ssq from the token stages; DyT: tanh(alpha a) in place before the
// MMA) then epilogue; warps 2-5 epilogue (TMEM lane quarter = warp % 4).
// Programmatic dependent launch: W* (a constant operand) streams into the ring BEFORE
// griddepcontrol.wait; the tokens (the previous kernel's output) are loaded after it.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <atomic>

namespace fn {

namespace dtc {
constexpr int ROWS = 128;               // W* rows per tile (MMA M)
constexpr int TOK = 16;                 // token rows (MMA N; rows >= M are TMA zero-fill)
constexpr int BK = 64;                  // k per stage (one SW128 atom row of bf16)
constexpr int STAGES = 12;  // 216 KiB ring: W* prefetched before griddepcontrol.wait
constexpr int W_STAGE = ROWS * BK * 2;  // 16 KiB
constexpr int T_STAGE = TOK * BK * 2;   // 2 KiB
constexpr int THREADS = 192;
constexpr int TMEM_COLS = 32;           // minimum allocation; D uses columns [0, 16)
constexpr int MAX_S = 8;                // K splits per tile
constexpr int MAX_CTAS = 160;           // tiles * S <= #SMs (148)
constexpr int SLOTS = 4;                // partial buffers, round robin over launches
constexpr size_t RECV = (size_t)ROWS * TOK * 4 + TOK * 4;  // one partial accumulator + ssq
constexpr size_t SMEM_MAX = 232448;                         // opt-in dynamic SMEM per CTA
constexpr size_t smem_bytes(int S, bool cluster) {
  return 1024 + (size_t)STAGES * (W_STAGE + T_STAGE) + (cluster ? (size_t)(S - 1) * RECV : 0) + 1024;
}
}  // namespace dtc

// split-K partials: [slot][CTA = tile * S + rank][row][token]; arrival counter per tile
__device__ float4 g_dtc_part[dtc::SLOTS][dtc::MAX_CTAS][dtc::ROWS * dtc::TOK / 4];
__device__ float4 g_dtc_ssq[dtc::SLOTS][dtc::MAX_CTAS][dtc::TOK / 4];
__device__ unsigned g_dtc_cnt[dtc::SLOTS][dtc::MAX_CTAS];

FN_DEVICE void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

#ifdef FN_GEMV_TC_TRACE  // tools/micro/gemv_tc_trace.cu: per-CTA timeline (globaltimer, ns)
__device__ unsigned long long g_tc_trace[2][160][8];
__device__ unsigned g_tc_launch;
FN_DEVICE unsigned long long tc_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TC_TRACE(ev) g_tc_trace[trace_par][blockIdx.x < 160 ? blockIdx.x : 159][(ev)] = tc_gtime()
#else
#define TC_TRACE(ev)
#endif

template <int MODE>
__global__ void __launch_bounds__(dtc::THREADS, 1)
    flashnorm_gemv_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_a,
                             const float* __restrict__ cstar, __nv_bfloat16* __restrict__ z, int M, int K, int N,
                             float eps, float alpha, int S, int slot, int use_cluster) {
  using namespace dtc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;                                  // [STAGES][128 x 64] SW128
  uint8_t* sT = sW + STAGES * W_STAGE;                 // [STAGES][16 x 64]  SW128
  float* recv = reinterpret_cast<float*>(sT + STAGES * T_STAGE);  // cluster mode: [S-1][128][16] (leader)
  float* recv_ssq = recv + (size_t)(use_cluster ? S - 1 : 0) * ROWS * TOK;  // [S-1][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(recv_ssq + (use_cluster ? S - 1 : 0) * TOK);
  uint64_t* full = bars;               // [STAGES] W* + tokens landed
  uint64_t* empty = bars + STAGES;     // [STAGES] stage consumed
  uint64_t* ready = bars + 2 * STAGES; // [STAGES] DyT: tokens transformed
  uint64_t* tfull = bars + 3 * STAGES; // accumulator complete
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tfull + 1);
  float* ssq_own = reinterpret_cast<float*>(tmem_holder + 4);  // [16]
  float* side_fence = ssq_own + TOK;                           // [32] load-completion fence
  int* last_flag = reinterpret_cast<int*>(side_fence + 32);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int rank = (int)(blockIdx.x % (unsigned)S);
  const int tile = (int)(blockIdx.x / (unsigned)S);
  const int n0 = tile * ROWS;
  const int nkb = (K + BK - 1) / BK;
  const int kb0 = (int)(((long long)rank * nkb) / S);
  const int kb1 = (int)(((long long)(rank + 1) * nkb) / S);
  const int my_kb = kb1 - kb0;  // >= 1 (S <= nkb)

  pdl_launch_dependents();  // the next call's CTAs may queue for free SMs right away
#ifdef FN_GEMV_TC_TRACE
  __shared__ int trace_par_s;
  if (threadIdx.x == 0) trace_par_s = (int)((atomicAdd(&g_tc_launch, 1u) / gridDim.x) & 1u);
  __syncthreads();
  const int trace_par = trace_par_s;
  if (threadIdx.x == 0) TC_TRACE(0);
#endif

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_w);
    prefetch_tmap(&tmap_a);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MODE == MODE_RMS ? 2 : 1);  // MMA commit (+ side warp)
      mbar_init(&ready[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const int pre = my_kb < STAGES ? my_kb : STAGES;
      // W* is constant: its first `pre` stages stream before the dependency wait
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], W_STAGE + T_STAGE);
        tma_load_2d(sW + i * W_STAGE, &tmap_w, &full[i], (kb0 + i) * BK, n0, kEvictFirst);
      }
      pdl_wait_prior_grid();  // tokens may be the previous kernel's output
      TC_TRACE(1);
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sT + i * T_STAGE, &tmap_a, &full[i], (kb0 + i) * BK, 0, kEvictLast);
      int stage = pre == STAGES ? 0 : pre;
      uint32_t phase = pre == STAGES ? 1u : 0u;
      for (int i = pre; i < my_kb; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], W_STAGE + T_STAGE);
        tma_load_2d(sW + stage * W_STAGE, &tmap_w, &full[stage], (kb0 + i) * BK, n0, kEvictFirst);
        tma_load_2d(sT + stage * T_STAGE, &tmap_a, &full[stage], (kb0 + i) * BK, 0, kEvictLast);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(ROWS, TOK);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < my_kb; ++i) {
        if (MODE == MODE_DYT) mbar_wait(&ready[stage], phase);
        else mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t adesc = make_sw128_desc(smem_u32(sW + stage * W_STAGE));
        const uint64_t bdesc = make_sw128_desc(smem_u32(sT + stage * T_STAGE));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) umma_bf16(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, (i | k) != 0);
        umma_commit(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      umma_commit(tfull);
    }
  } else {
    // ------------------------------------------------------------ side warp (warp 2), then epilogue
    if (warp == 2) {
      if (MODE == MODE_RMS) {
        // lane l: token row l/2, 16-byte chunks 4*(l&1) .. +3 of each stage (swizzled position)
        const int trow = (int)lane >> 1;
        float s0 = 0.f, s1 = 0.f;
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < my_kb; ++i) {
          mbar_wait_warp(&full[stage], phase);
          const uint4* row = reinterpret_cast<const uint4*>(sT + stage * T_STAGE + trow * 128);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 v = row[(4 * (lane & 1) + q) ^ (trow & 7)];
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
          // the store consumes every loaded value: it (and the arrive after it) issue only
          // once this warp's LDS of the stage have returned (WAR vs the TMA refill)
          side_fence[lane] = s0 + s1;
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        float s = s0 + s1;
        s += __shfl_xor_sync(0xffffffffu, s, 1);  // lanes 2r, 2r+1 -> token row r (fixed order)
        if ((lane & 1) == 0) ssq_own[lane >> 1] = s;
      } else if (MODE == MODE_DYT) {
        const __nv_bfloat162 alpha2 = __floats2bfloat162_rn(alpha, alpha);
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < my_kb; ++i) {
          mbar_wait_warp(&full[stage], phase);
          uint4* p = reinterpret_cast<uint4*>(sT + stage * T_STAGE) + lane * 4;  // 64 B per lane
          uint4 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = p[q];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t* w = reinterpret_cast<uint32_t*>(&v[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&w[e]);
              x = __hmul2(x, alpha2);
              w[e] = tanh_approx_bf16x2(*reinterpret_cast<uint32_t*>(&x));
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) p[q] = v[q];
          fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
          __syncwarp();
          if (lane == 0) mbar_arrive(&ready[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    // ---------------------------------------------------------------- epilogue (warps 2-5)
    const uint32_t q4 = warp & 3u;  // TMEM lane quarter this warp may access
    const int row = (int)(q4 * 32 + lane);
    named_bar_sync(1, 128);         // ssq_own written by the side warp
    mbar_wait_warp(tfull, 0);
    if (warp == 2 && lane == 0) TC_TRACE(2);
    tc_fence_after();
    uint32_t v[16];
    tmem_ld_32x32b_x16(tmem_base + ((q4 * 32u) << 16), v);
    tmem_wait_ld();
    float acc[TOK];
#pragma unroll
    for (int m = 0; m < TOK; ++m) acc[m] = __uint_as_float(v[m]);
    bool write_z = true;
    if (S > 1 && use_cluster) {
      // cluster mode: partials go straight into the leader's SMEM (DSMEM), one cluster barrier
      if (rank != 0) {
        const uint32_t dst = mapa_shared(recv + ((size_t)(rank - 1) * ROWS + row) * TOK, 0);
#pragma unroll
        for (int m = 0; m < TOK; m += 4)
          asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + m * 4), "f"(acc[m]),
                       "f"(acc[m + 1]), "f"(acc[m + 2]), "f"(acc[m + 3])
                       : "memory");
        if (MODE == MODE_RMS && warp == 2 && lane < TOK / 4) {
          const uint32_t sd = mapa_shared(recv_ssq + (rank - 1) * TOK + lane * 4, 0);
          asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sd), "f"(ssq_own[4 * lane]),
                       "f"(ssq_own[4 * lane + 1]), "f"(ssq_own[4 * lane + 2]), "f"(ssq_own[4 * lane + 3])
                       : "memory");
        }
      }
      cluster_sync_all();  // warps 0 and 1 join at the end of the kernel
      write_z = rank == 0;
      if (write_z) {
        for (int r = 1; r < S; ++r) {  // fixed rank order
          const float4* src = reinterpret_cast<const float4*>(recv + ((size_t)(r - 1) * ROWS + row) * TOK);
#pragma unroll
          for (int m4 = 0; m4 < TOK / 4; ++m4) {
            const float4 p = src[m4];
            acc[4 * m4] += p.x; acc[4 * m4 + 1] += p.y; acc[4 * m4 + 2] += p.z; acc[4 * m4 + 3] += p.w;
          }
        }
      }
    } else if (S > 1) {
      // publish this CTA's partial, then count arrivals on the tile; the last one reduces
      float4* mine = g_dtc_part[slot][blockIdx.x];
#pragma unroll
      for (int m4 = 0; m4 < TOK / 4; ++m4)
        __stcg(mine + row * (TOK / 4) + m4, make_float4(acc[4 * m4], acc[4 * m4 + 1], acc[4 * m4 + 2], acc[4 * m4 + 3]));
      if (MODE == MODE_RMS && warp == 2 && lane < TOK / 4)
        __stcg(&g_dtc_ssq[slot][blockIdx.x][lane], make_float4(ssq_own[4 * lane], ssq_own[4 * lane + 1],
                                                               ssq_own[4 * lane + 2], ssq_own[4 * lane + 3]));
      __threadfence();
      named_bar_sync(1, 128);
      if (warp == 2 && lane == 0) {
        const unsigned old = atomicAdd(&g_dtc_cnt[slot][tile], 1u);
        const int last = old == (unsigned)(S - 1);
        if (last) g_dtc_cnt[slot][tile] = 0u;  // nobody else touches it in this launch
        *last_flag = last;
      }
      named_bar_sync(1, 128);
      write_z = *last_flag != 0;
      if (write_z) {
        __threadfence();
        float tot[TOK];
#pragma unroll
        for (int m = 0; m < TOK; ++m) tot[m] = 0.f;
        for (int r = 0; r < S; ++r) {  // fixed rank order, own partial from registers
          if (r == rank) {
#pragma unroll
            for (int m = 0; m < TOK; ++m) tot[m] += acc[m];
          } else {
            const float4* src = g_dtc_part[slot][tile * S + r] + row * (TOK / 4);
#pragma unroll
            for (int m4 = 0; m4 < TOK / 4; ++m4) {
              const float4 p = __ldcg(src + m4);
              tot[4 * m4] += p.x; tot[4 * m4 + 1] += p.y; tot[4 * m4 + 2] += p.z; tot[4 * m4 + 3] += p.w;
            }
          }
        }
#pragma unroll
        for (int m = 0; m < TOK; ++m) acc[m] = tot[m];
      }
    }
    if (write_z) {
      float ssq[TOK];
#pragma unroll
      for (int m = 0; m < TOK; ++m) ssq[m] = 0.f;
      if (MODE == MODE_RMS) {
        if (S == 1 || use_cluster) {
#pragma unroll
          for (int m = 0; m < TOK; ++m) ssq[m] = ssq_own[m];
          for (int r = 1; r < S; ++r) {  // fixed rank order (cluster mode)
#pragma unroll
            for (int m = 0; m < TOK; ++m) ssq[m] += recv_ssq[(r - 1) * TOK + m];
          }
        } else {
          for (int r = 0; r < S; ++r) {  // fixed rank order
#pragma unroll
            for (int m4 = 0; m4 < TOK / 4; ++m4) {
              const float4 p = __ldcg(&g_dtc_ssq[slot][tile * S + r][m4]);
              ssq[4 * m4] += p.x; ssq[4 * m4 + 1] += p.y; ssq[4 * m4 + 2] += p.z; ssq[4 * m4 + 3] += p.w;
            }
          }
        }
      }
      const int n = n0 + row;
      if (n < N) {
        const float cb = cstar != nullptr ? __ldg(cstar + n) : 0.0f;
        const float invK = 1.0f / (float)K;
        pdl_wait_prior_grid();  // z may still be read by the previous kernel of the stream
#pragma unroll
        for (int m = 0; m < TOK; ++m) {
          if (m < M) {
            const float r = MODE == MODE_RMS ? rsqrtf(fmaf(ssq[m], invK, eps)) : 1.0f;
            z[(size_t)m * N + n] = __float2bfloat16_rn(fmaf(acc[m], r, cb));
          }
        }
      }
    }
  }
  if (S > 1 && use_cluster && warp < 2) cluster_sync_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
#ifdef FN_GEMV_TC_TRACE
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_tc_trace[trace_par][blockIdx.x < 160 ? blockIdx.x : 159][4] = smid;
    TC_TRACE(3);
  }
#endif
}

// ------------------------------------------------------------------ host side

namespace {
template <int MODE>
const void* dtc_kernel() {
  return (const void*)flashnorm_gemv_tc_kernel<MODE>;
}
const void* dtc_fptr(int mode) {
  return mode == MODE_RMS ? dtc_kernel<MODE_RMS>() : mode == MODE_DYT ? dtc_kernel<MODE_DYT>() : dtc_kernel<MODE_NONE>();
}
// can `clusters` clusters of S CTAs be resident at once?
bool cluster_fits(int mode, int S, int clusters) {
  if (dtc::smem_bytes(S, true) > dtc::SMEM_MAX) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * S);
  cfg.blockDim = dim3(dtc::THREADS);
  cfg.dynamicSmemBytes = dtc::smem_bytes(S, true);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  return cudaOccupancyMaxActiveClusters(&n, dtc_fptr(mode), &cfg) == cudaSuccess && n >= clusters;
}
}  // namespace

int gemv_tc_split(int K, int N, int num_sms) {
  using namespace dtc;
  const int tiles = (N + ROWS - 1) / ROWS;
  const int nkb = (K + BK - 1) / BK;
  int S = std::min(num_sms, MAX_CTAS) / tiles;
  S = std::min(S, MAX_S);
  S = std::min(S, nkb);
  return std::max(S, 1);
}

bool gemv_tc_supported(int M, int N, int num_sms) {
  return M >= 1 && M <= dtc::TOK && (N + dtc::ROWS - 1) / dtc::ROWS <= std::min(num_sms, dtc::MAX_CTAS);
}

cudaError_t launch_gemv_tc(const CUtensorMap& tw, const CUtensorMap& ta, const float* cstar, __nv_bfloat16* z,
                           int M, int K, int N, float eps, float alpha, int mode, int num_sms, cudaStream_t stream) {
  using namespace dtc;
  const void* fptr = dtc_fptr(mode);
  static bool attr_set[3] = {false, false, false};
  if (!attr_set[mode]) {
    cudaError_t e = cudaFuncSetAttribute(fptr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_MAX);
    if (e != cudaSuccess) return e;
    attr_set[mode] = true;
  }
  const int tiles = (N + ROWS - 1) / ROWS;
  int S = gemv_tc_split(K, N, num_sms);
  // Prefer a cluster (DSMEM reduction, ~1 us tail) of the largest size whose clusters are all
  // co-resident (GPC shapes cap clusters of 3 at 45 on this part); fall back to the global-
  // memory reduction with the full split when no cluster size > 1 fits.
  int use_cluster = 0;
  {
    static int ck[3][3] = {{-1, -1, -1}, {-1, -1, -1}, {-1, -1, -1}};
    if (ck[mode][0] == tiles && ck[mode][1] == S) {
      if (ck[mode][2] > 1) { S = ck[mode][2]; use_cluster = 1; }
    } else {
      int fit = 1;
      for (int c = S; c > 1; --c)
        if (cluster_fits(mode, c, tiles)) { fit = c; break; }
      ck[mode][0] = tiles; ck[mode][1] = S; ck[mode][2] = fit;
      if (fit > 1) { S = fit; use_cluster = 1; }
    }
  }
  // partial-buffer slot: launches in flight together (PDL overlap, graph replays) use
  // different slots; SLOTS consecutive launches cannot overlap (each waits for the previous)
  static std::atomic<unsigned> seq{0};
  int slot = (int)(seq.fetch_add(1u) % SLOTS);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles * S);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem_bytes(S, use_cluster != 0);
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = use_cluster ? S : 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  void* args[] = {(void*)&tw, (void*)&ta, (void*)&cstar, (void*)&z, (void*)&M, (void*)&K, (void*)&N,
                  (void*)&eps, (void*)&alpha, (void*)&S, (void*)&slot, (void*)&use_cluster};
  return cudaLaunchKernelExC(&cfg, fptr, args);
}

}  // namespace fn
