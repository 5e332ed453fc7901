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
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>

namespace fn {

namespace dtc {
constexpr int ROWS = 128;               // W* rows per MMA (M)
constexpr int TOK = 16;                 // token rows (MMA N; rows >= M are TMA zero-fill)
constexpr int BK = 64;                  // k per stage (one SW128 atom row of bf16)
constexpr int T_STAGE = TOK * BK * 2;   // 2 KiB
constexpr int THREADS = 192;
constexpr int TMEM_COLS = 32;           // D of MMA j in columns [16j, 16j+16), j < R <= 2 (R = 4: 64)
constexpr int BOX_ROWS_MAX = 256;       // TMA box rows (R = 4 tiles load two boxes per stage)
constexpr int TOK_GS = 8;               // resident tokens: stages per readiness group
constexpr int TOK_GROUPS = 8;           // resident tokens: at most 64 stages (128 KiB) ...
constexpr int TOK_MAX_BYTES = 64 * 1024;  // ... but the host keeps it <= 64 KiB
constexpr int MAX_S = 8;                // K splits per tile (portable cluster size)
constexpr int MAX_CTAS = 160;           // tiles * S <= #SMs (148)
constexpr int SLOTS = 4;                // global-mode partial buffers, round robin over launches
constexpr size_t SMEM_MAX = 232448;     // opt-in dynamic SMEM per CTA (ring sizes stay below it)
// tile = R x 128 W* rows (R MMAs per k step sharing the token operand)
// stage = KB consecutive 64-wide k blocks (KB = 2: one 3-D TMA box of 32 KiB for a 128-row tile —
// TMA streams near the HBM rate only with boxes this large, tools/micro/stream_bw.cu)
template <int R, int KB = 1> struct Cfg {
  static constexpr int W_STAGE = R * ROWS * BK * 2 * KB;             // 16 / 32 KiB
  static constexpr int TK_STAGE = T_STAGE * KB;                      // token bytes per stage
  static constexpr int STAGES = (R * KB) == 1 ? 12 : 6;              // default: ~204-216 KiB ring
  static size_t smem(int stages) { return 1024 + (size_t)stages * (W_STAGE + TK_STAGE) + 1024; }
};
}  // namespace dtc

// global-mode split-K partials: [slot][CTA = tile * S + rank][j][row][token]; counter per tile
__device__ float4 g_dtc_part[dtc::SLOTS][dtc::MAX_CTAS][2 * dtc::ROWS * dtc::TOK / 4];
__device__ float4 g_dtc_ssq[dtc::SLOTS][dtc::MAX_CTAS][dtc::TOK / 4];
__device__ unsigned g_dtc_cnt[dtc::SLOTS][dtc::MAX_CTAS];

FN_DEVICE float4 ld_cluster_v4(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}

#ifdef FN_GEMV_TC_TRACE  // tools/micro/gemv_tc_trace.cu: per-CTA timeline (globaltimer, ns)
__device__ unsigned long long g_tc_trace[2][160][16];
__device__ unsigned g_tc_launch;
FN_DEVICE unsigned long long tc_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TC_TRACE(ev) g_tc_trace[trace_par][blockIdx.x < 160 ? blockIdx.x : 159][(ev)] = tc_gtime()
// per-stage SM-clock stamps of CTA 0 (launch parity 1): [0] MMA saw full, [1] producer issued,
// [2] side warp released, [3] producer saw empty
__device__ long long g_tc_stage[4][64];
#define TC_STAGE(w, i) do { if (trace_par == 1 && blockIdx.x == 0 && (i) < 64) g_tc_stage[w][i] = clock64(); } while (0)
// epilogue SM-clock stamps of CTAs 0 (leader) and 1 (peer), launch parity 1, warp 2 lane 0
__device__ long long g_tc_epi[2][8];
#define TC_EPI(e) do { if (trace_par == 1 && blockIdx.x < 2 && warp == 2 && lane == 0) g_tc_epi[blockIdx.x][e] = clock64(); } while (0)
#else
#define TC_EPI(e)
#define TC_TRACE(ev)
#define TC_STAGE(w, i)
#endif

// resident-token slice size (stages) is carried in bits 8..15 of `flags`
FN_DEVICE int nkb_host_tokmax(int flags) { return (flags >> 8) & 0xFF; }

template <int MODE, int R, int KB>
__global__ void __launch_bounds__(dtc::THREADS, R == 4 ? 1 : 2)  // R < 4: <= 168 registers (two CTAs may share an SM)
    flashnorm_gemv_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_a,
                             const float* __restrict__ cstar, __nv_bfloat16* __restrict__ z, int M, int K, int N,
                             float eps, float alpha, int S, int slot, int use_cluster,
                             const float* __restrict__ row_scale, const RopeParams rope, int l2pf,
                             int stages, int flags, const __nv_bfloat16* __restrict__ wptr,
                             const __nv_bfloat16* __restrict__ aptr) {
  using namespace dtc;
  constexpr int W_STAGE = Cfg<R, KB>::W_STAGE;
  constexpr int T_STAGE = Cfg<R, KB>::TK_STAGE;  // shadows dtc::T_STAGE: KB token boxes per stage
  constexpr int KSUB = ROWS * BK * 2;             // bytes of one 128-row x 64-k W* sub-block
  const int STAGES = stages;  // ring depth (runtime: the host sizes it for 1 or 2 CTAs per SM)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // resident tokens (flags & 32, R = KB = 1): this CTA's whole token slice [my_kb][16 x 64] SW128 is staged
  // ONCE after the dependency wait by warps 2-5 (DyT: tanh applied then, once per element) and the ring
  // carries W* only; tokmax = the host's bound on my_kb (its size)
  const bool tokres = (flags & 32) != 0;
  const int tokmax = tokres ? (nkb_host_tokmax(flags)) : 0;
  uint8_t* sW = smem;                                  // [STAGES][R*128 x 64] SW128
  uint8_t* sT = sW + STAGES * W_STAGE;                 // [STAGES][16 x 64] SW128, or [tokmax][16 x 64] resident
  uint64_t* bars = reinterpret_cast<uint64_t*>(sT + (tokres ? tokmax * dtc::T_STAGE : STAGES * T_STAGE));
  uint64_t* full = bars;               // [STAGES] W* + tokens landed
  uint64_t* empty = bars + STAGES;     // [STAGES] stage consumed
  uint64_t* ready = bars + 2 * STAGES; // [STAGES] DyT: tokens transformed
  uint64_t* tfull = bars + 3 * STAGES; // accumulator complete
  uint64_t* tokready = tfull + 1;      // [TOK_GROUPS] resident tokens: group g of TOK_GS stages transformed
  uint64_t* tokland = tokready + dtc::TOK_GROUPS;  // [TOK_GROUPS] resident tokens: group g landed (TMA)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tokland + dtc::TOK_GROUPS);
  float* ssq_own = reinterpret_cast<float*>(tmem_holder + 4);  // [16] this CTA's partial ssq per token
  float* ssq_red = ssq_own + TOK;                              // [4 warps][16]
  int* last_flag = reinterpret_cast<int*>(ssq_red + 4 * TOK);
  uint64_t* recv_bar = reinterpret_cast<uint64_t*>(last_flag + 2);  // push mode: peers' partials landed
  // cluster mode: after the last MMA the ring is free; each CTA stages its partial there
  float* part = reinterpret_cast<float*>(smem);                // [R][128][16]
  // push mode: the leader's receive slots, one per peer rank, beside the ring (a peer may finish
  // before the leader's ring is drained): [S-1][R*128*16 + 16] fp32
  constexpr int RECV_STRIDE = R * ROWS * TOK + TOK;
  float* recv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 1024);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int rank = (int)(blockIdx.x % (unsigned)S);  // K-split rank within the tile
  // cluster mode: use_cluster = CTAs per cluster = T tiles x S splits; the tile's leader (rank 0) has
  // cluster rank `lead` (clusters are consecutive blockIdx.x ranges, tiles consecutive inside them)
  const uint32_t lead = use_cluster ? (uint32_t)((int)(blockIdx.x % (unsigned)use_cluster) - rank) : 0u;
  const int tile = (int)(blockIdx.x / (unsigned)S);
  const int n0 = tile * R * ROWS;
  constexpr int TCOLS = R * TOK > TMEM_COLS ? R * TOK : TMEM_COLS;  // TMEM columns (power of two >= 32)
  constexpr int NBOX = R * ROWS > BOX_ROWS_MAX ? R * ROWS / BOX_ROWS_MAX : 1;  // TMA boxes per W* stage
  const int nkb = (K + BK * KB - 1) / (BK * KB);  // stages of KB k blocks
  const int kb0 = (int)(((long long)rank * nkb) / S);
  const int kb1 = (int)(((long long)(rank + 1) * nkb) / S);
  const int my_kb = kb1 - kb0;  // >= 1 (S <= nkb)
  // stage i of this CTA: KB = 1 -> 2-D box at k = i * 64; KB = 2 -> 3-D box {64, rows, 2} at k block 2 i
  auto load_w = [&](void* dst, uint64_t* bar, int i) {
    if (KB == 1) {
#pragma unroll
      for (int b = 0; b < NBOX; ++b)
        tma_load_2d(static_cast<uint8_t*>(dst) + b * (W_STAGE / NBOX), &tmap_w, bar, i * BK,
                    n0 + b * (R * ROWS / NBOX), kEvictFirst);
    } else {
      tma_load_3d(dst, &tmap_w, bar, 0, n0, i * KB, kEvictFirst);
    }
  };
  auto load_t = [&](void* dst, uint64_t* bar, int i) {
    if (KB == 1) tma_load_2d(dst, &tmap_a, bar, i * BK, 0, kEvictLast);
    else tma_load_3d(dst, &tmap_a, bar, 0, 0, i * KB, kEvictLast);
  };
  auto prefetch_w = [&](int i, int nrow0) {
    if (KB == 1) {
#pragma unroll
      for (int b = 0; b < NBOX; ++b) tma_prefetch_l2_2d(&tmap_w, i * BK, nrow0 + b * (R * ROWS / NBOX));
    } else {
      tma_prefetch_l2_3d(&tmap_w, 0, nrow0, i * KB);
    }
  };

  // the next call's CTAs may queue for free SMs right away (flags & 64: only once this CTA's W* loads are
  // all issued — A/B knob FN_DECODE_PDL_LATE)
  if (!(flags & 64)) pdl_launch_dependents();
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
      mbar_init(&empty[s], 1);  // MMA commit
      mbar_init(&ready[s], 1);
    }
    mbar_init(tfull, 1);
    for (int g = 0; g < TOK_GROUPS; ++g) {
      mbar_init(&tokready[g], 1);
      mbar_init(&tokland[g], 1);
    }
    mbar_init(recv_bar, 1);  // push mode: the leader's expect_tx + each peer's bulk copy (complete_tx)
    fence_mbar_init();
    if (S > 1 && use_cluster && (flags & 1) && rank == 0)
      mbar_arrive_expect_tx(recv_bar, (uint32_t)((S - 1) * RECV_STRIDE * 4));
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, TCOLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const bool push = S > 1 && use_cluster && (flags & 1);
  if (push) cluster_arrive_relaxed();  // barrier inits published; the matching wait precedes any remote access

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const int pre = my_kb < STAGES ? my_kb : STAGES;
      // W* is constant: its first `pre` stages stream before the dependency wait
      const uint32_t stage_tx = W_STAGE + (tokres ? 0 : T_STAGE);
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], stage_tx);
        load_w(sW + i * W_STAGE, &full[i], kb0 + i);
      }
      // ... and the rest of this CTA's W* slice is pulled into L2 (up to l2pf boxes), so the
      // HBM stream keeps going while this call waits for the previous one; the ring refills
      // after the wait then hit L2
      for (int i = pre; i < my_kb && i < pre + l2pf; ++i)
        prefetch_w(kb0 + i, n0);  // the box is the whole R x 128-row tile
      if (flags & 2) {
        // ... and the whole slice of the CTA half a grid away: CTAs start in blockIdx order as
        // the previous call's CTAs leave, so the upper half typically starts late; its W* is
        // then already in L2 when it does
        const int pb = (int)((blockIdx.x + gridDim.x / 2) % gridDim.x);
        const int prank = pb % S, pn0 = (pb / S) * R * ROWS;
        const int pk0 = (int)(((long long)prank * nkb) / S), pk1 = (int)(((long long)(prank + 1) * nkb) / S);
        for (int i = pk0; i < pk1; ++i) prefetch_w(i, pn0);
      }
      pdl_wait_prior_grid();  // tokens may be the previous kernel's output
      TC_TRACE(1);
      if (!tokres) {
        for (int i = 0; i < pre; ++i) load_t(sT + i * T_STAGE, &full[i], kb0 + i);
      } else {
        // the whole token slice at once, one barrier per group of TOK_GS stages (ahead of every
        // post-wait W* load in the TMA queue)
        for (int g = 0; g * TOK_GS < my_kb; ++g) {
          const int i0 = g * TOK_GS, i1 = min(my_kb, i0 + TOK_GS);
          mbar_arrive_expect_tx(&tokland[g], (uint32_t)((i1 - i0) * dtc::T_STAGE));
          for (int i = i0; i < i1; ++i) load_t(sT + i * dtc::T_STAGE, &tokland[g], kb0 + i);
        }
      }
      int stage = pre == STAGES ? 0 : pre;
      uint32_t phase = pre == STAGES ? 1u : 0u;
      for (int i = 0; i < pre; ++i) TC_STAGE(1, i);
      for (int i = pre; i < my_kb; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        TC_STAGE(1, i);
        mbar_arrive_expect_tx(&full[stage], stage_tx);
        load_w(sW + stage * W_STAGE, &full[stage], kb0 + i);
        if (!tokres) load_t(sT + stage * T_STAGE, &full[stage], kb0 + i);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (flags & 64) pdl_launch_dependents();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(ROWS, TOK);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < my_kb; ++i) {
        if (tokres) {
          if (i % TOK_GS == 0) mbar_wait(MODE == MODE_DYT ? &tokready[i / TOK_GS] : &tokland[i / TOK_GS], 0);
          mbar_wait(&full[stage], phase);
        } else if (MODE == MODE_DYT) {
          mbar_wait(&ready[stage], phase);
        } else {
          mbar_wait(&full[stage], phase);
        }
#ifdef FN_GEMV_TC_TRACE
        TC_STAGE(0, i);
        if (i == 0) TC_TRACE(5);
        if (i == STAGES) TC_TRACE(6);
        if (i == my_kb - 1) TC_TRACE(7);
#endif
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {  // the stage's k blocks: [kb][rows][64] / [kb][16][64] in SMEM
          const uint64_t bdesc =
              make_sw128_desc(smem_u32(tokres ? sT + i * dtc::T_STAGE : sT + stage * T_STAGE + kk * dtc::T_STAGE));
#pragma unroll
          for (int j = 0; j < R; ++j) {  // rows [128j, 128j+128) of the tile: 16 KiB into the box
            const uint64_t adesc = make_sw128_desc(smem_u32(sW + stage * W_STAGE + (kk * R + j) * KSUB));
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16(tmem_base + j * TOK, adesc + 2 * k, bdesc + 2 * k, idesc, (i | kk | k) != 0);
          }
        }
        umma_commit(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      umma_commit(tfull);
    }
  } else {
    // ------------------------------------------------------------ side warp (warp 2), then epilogue
    if (tokres) {
      if (MODE == MODE_DYT) {
        // the token slice landed once (TMA, per group): tanh(alpha a) in place, once per element, exactly
        // as the in-ring transform (RN_bf16(tanh(RN_bf16(alpha) a))); rows >= M are zero fill
        const int t = (int)threadIdx.x - 64;  // 0..127
        const __nv_bfloat162 alpha2 = __floats2bfloat162_rn(alpha, alpha);
        for (int g = 0; g * TOK_GS < my_kb; ++g) {
          const int i0 = g * TOK_GS, i1 = min(my_kb, i0 + TOK_GS);
          mbar_wait_warp(&tokland[g], 0);
          for (int i = i0; i < i1; ++i) {
            uint4* p = reinterpret_cast<uint4*>(sT + i * dtc::T_STAGE) + t;
            uint4 v = *p;
            uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&w[e]);
              x = __hmul2(x, alpha2);
              w[e] = tanh_approx_bf16x2(*reinterpret_cast<uint32_t*>(&x));
            }
            *p = v;
          }
          fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
          named_bar_sync(2, 128);
          if (t == 0) mbar_arrive(&tokready[g]);
        }
      }
    } else if (MODE == MODE_DYT) {
      // tanh(alpha a) in place on each token stage before its MMA: warps 2-5, one 16-byte
      // chunk per thread (2 KiB per stage), so the transform keeps ahead of the W* stream
      const __nv_bfloat162 alpha2 = __floats2bfloat162_rn(alpha, alpha);
      const int t = (int)threadIdx.x - 64;  // 0..127
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < my_kb; ++i) {
        mbar_wait_warp(&full[stage], phase);
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          uint4* p = reinterpret_cast<uint4*>(sT + stage * T_STAGE + kk * dtc::T_STAGE) + t;
          uint4 v = *p;
          uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&w[e]);
            x = __hmul2(x, alpha2);
            w[e] = tanh_approx_bf16x2(*reinterpret_cast<uint32_t*>(&x));
          }
          *p = v;
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        named_bar_sync(2, 128);
        if (t == 0) mbar_arrive(&ready[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    if (warp >= 3 && wptr != nullptr && (flags & 12)) {
      // idle epilogue warps (3-5) pull W* lines beyond the ring into L2 with plain prefetches
      // (LSU path; the TMA queue stays free for the producer): own slice (flag 4) and/or the
      // slice of the CTA half a grid away (flag 8), one 128-byte line = one row x one k block
      const int t = (int)threadIdx.x - 96;  // 0..95
      const int rows = R * ROWS;
      auto pf = [&](int nbase, int ka, int kb) {
        const int nlines = (kb - ka) * rows;
        for (int l = t; l < nlines; l += 96) {
          const int n = nbase + l % rows, k = ka + l / rows;
          if (n < N) {
            if (flags & 16) asm volatile("prefetch.global.L2 [%0];" ::"l"(wptr + (size_t)n * K + (size_t)k * BK));
            else asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(wptr + (size_t)n * K + (size_t)k * BK));
          }
        }
      };
      const int pre = my_kb < STAGES ? my_kb : STAGES;
      const int nkb64 = (K + BK - 1) / BK;  // pf() works in 64-wide k blocks
      if (flags & 4) pf(n0, (kb0 + pre) * KB, min(kb1 * KB, nkb64));
      if (flags & 8) {
        const int pb = (int)((blockIdx.x + gridDim.x / 2) % gridDim.x);
        const int prank = pb % S, pn0 = (pb / S) * R * ROWS;
        pf(pn0, (int)(((long long)prank * nkb) / S) * KB, min((int)(((long long)(prank + 1) * nkb) / S) * KB, nkb64));
      }
    }
    if (MODE == MODE_RMS) {
      // per-token partial ssq over this CTA's K range, read by warps 2-5 straight from global
      // (L2) after the dependency wait: beside the contraction and OFF the
      // W* ring — a side warp squaring each ring stage gated its release and paced the whole
      // ring at ~400 cycles per stage (tools/micro/gemv_tc_trace.cu, per-stage clocks)
      pdl_wait_prior_grid();  // tokens may be the previous kernel's output
      const int t = (int)threadIdx.x - 64;  // 0..127
      const int k0 = kb0 * BK * KB;
      const int nch = (min(kb1 * BK * KB, K) - k0) / 8;  // 16-byte chunks (K % 8 == 0)
      constexpr int CPT = 2;                        // chunks per thread per token per round
      float sm[TOK];
#pragma unroll
      for (int m = 0; m < TOK; ++m) sm[m] = 0.f;
      for (int c0 = t; c0 < nch; c0 += 128 * CPT) {
        uint4 v[TOK][CPT];
#pragma unroll
        for (int m = 0; m < TOK; ++m)
#pragma unroll
          for (int u = 0; u < CPT; ++u) {
            const int c = c0 + u * 128;
            v[m][u] = (m < M && c < nch) ? __ldg(reinterpret_cast<const uint4*>(aptr + (size_t)m * K + k0) + c)
                                         : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
        for (int m = 0; m < TOK; ++m)
#pragma unroll
          for (int u = 0; u < CPT; ++u) {
            float x, s0 = 0.f, s1 = 0.f;
            x = bf16lo(v[m][u].x); s0 = fmaf(x, x, s0);
            x = bf16hi(v[m][u].x); s1 = fmaf(x, x, s1);
            x = bf16lo(v[m][u].y); s0 = fmaf(x, x, s0);
            x = bf16hi(v[m][u].y); s1 = fmaf(x, x, s1);
            x = bf16lo(v[m][u].z); s0 = fmaf(x, x, s0);
            x = bf16hi(v[m][u].z); s1 = fmaf(x, x, s1);
            x = bf16lo(v[m][u].w); s0 = fmaf(x, x, s0);
            x = bf16hi(v[m][u].w); s1 = fmaf(x, x, s1);
            sm[m] += s0 + s1;
          }
      }
#pragma unroll
      for (int m = 0; m < TOK; ++m) {
        float x = sm[m];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        sm[m] = x;
      }
      if (lane == 0)
#pragma unroll
        for (int m = 0; m < TOK; ++m) ssq_red[(warp - 2) * TOK + m] = sm[m];
      named_bar_sync(1, 128);
      if (t < TOK) ssq_own[t] = (ssq_red[t] + ssq_red[TOK + t]) + (ssq_red[2 * TOK + t] + ssq_red[3 * TOK + t]);
    }
    // ---------------------------------------------------------------- epilogue (warps 2-5)
    const uint32_t q4 = warp & 3u;  // TMEM lane quarter this warp may access
    const int row = (int)(q4 * 32 + lane);
    named_bar_sync(1, 128);         // ssq_own complete
    // RoPE: fetch this thread's cos/sin (per token) while the accumulator is still being built;
    // only block 0 of the tile (R = 1 covers it whole) is used below
    const bool rope_blk = R == 1 && MODE == MODE_RMS && rope.pos != nullptr && n0 < rope.n;
    float rc[TOK], rs[TOK];
    if (rope_blk) {
      const int n = n0 + row;
      const int hh = rope.h >> 1;
      const int i = (n % rope.h) >> 1;
#pragma unroll
      for (int m = 0; m < TOK; ++m) {
        rc[m] = 0.f;
        rs[m] = 0.f;
        if (m < M) {
          const int pos = __ldg(rope.pos + m);
          rc[m] = __ldg(rope.cos_tab + (size_t)pos * hh + i);
          rs[m] = __ldg(rope.sin_tab + (size_t)pos * hh + i);
        }
      }
    }
    // z (written below) may still be read by the previous kernel of the stream: wait for it here,
    // while the contraction runs (RMS mode already waited before reading the tokens)
    if (MODE != MODE_RMS) pdl_wait_prior_grid();
    mbar_wait_warp(tfull, 0);
    TC_EPI(0);
    if (warp == 2 && lane == 0) TC_TRACE(2);
    tc_fence_after();
    float acc[R][TOK];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      uint32_t v[16];
      tmem_ld_32x32b_x16(tmem_base + ((q4 * 32u) << 16) + j * TOK, v);
      tmem_wait_ld();
#pragma unroll
      for (int m = 0; m < TOK; ++m) acc[j][m] = __uint_as_float(v[m]);
    }
    TC_EPI(1);
    float ssq[TOK];
#pragma unroll
    for (int m = 0; m < TOK; ++m) ssq[m] = MODE == MODE_RMS ? ssq_own[m] : 0.f;
    bool write_z = true;
    if (push) {
      // push mode: each peer stores its partial straight into its receive slot in the leader
      // (DSMEM stores from registers), then every peer epilogue thread release-arrives on the
      // leader's recv barrier; the leader sums the slots in fixed rank order (deterministic).
      // No cluster-wide barrier: a peer leaves as soon as its stores are issued.
      if (rank != 0) {
        // stage the partial (+ ssq) in this CTA's own SMEM (the ring is free once tfull fired),
        // then ONE bulk copy moves it into the leader's receive slot and completes on the leader's
        // recv barrier (a release-arrive per thread after DSMEM stores measured ~1500 cycles)
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
          for (int m4 = 0; m4 < TOK / 4; ++m4)
            reinterpret_cast<float4*>(part)[(j * ROWS + row) * (TOK / 4) + m4] =
                make_float4(acc[j][4 * m4], acc[j][4 * m4 + 1], acc[j][4 * m4 + 2], acc[j][4 * m4 + 3]);
        if (MODE == MODE_RMS && warp == 2 && lane < TOK) part[R * ROWS * TOK + lane] = ssq_own[lane];
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the bulk-copy engine
        named_bar_sync(1, 128);
        TC_EPI(2);
        if (warp == 2) {
          cluster_wait();  // the leader's recv barrier is initialised (arrive at kernel start)
          if (lane == 0) {
            dsmem_bulk_copy(mapa_shared(recv + (rank - 1) * RECV_STRIDE, lead), part, RECV_STRIDE * 4,
                            mapa_shared(recv_bar, lead));
            bulk_commit_group();
            bulk_wait_read();  // the source (this CTA's SMEM) stays valid until read
          }
          __syncwarp();
        }
        TC_EPI(3);
        write_z = false;
      } else {
        TC_EPI(2);
        mbar_wait_warp_cluster(recv_bar, 0);
        TC_EPI(3);
        for (int r = 1; r < S; ++r) {  // fixed rank order
          const float* sl = recv + (r - 1) * RECV_STRIDE;
#pragma unroll
          for (int j = 0; j < R; ++j)
#pragma unroll
            for (int m4 = 0; m4 < TOK / 4; ++m4) {
              const float4 p = reinterpret_cast<const float4*>(sl + (j * ROWS + row) * TOK)[m4];
              acc[j][4 * m4] += p.x; acc[j][4 * m4 + 1] += p.y; acc[j][4 * m4 + 2] += p.z; acc[j][4 * m4 + 3] += p.w;
            }
          if (MODE == MODE_RMS)
#pragma unroll
            for (int m = 0; m < TOK; ++m) ssq[m] += sl[R * ROWS * TOK + m];
        }
      }
    } else if (S > 1 && use_cluster) {
      // cluster mode: every CTA parks its partial in its own (now free) ring SMEM; after one
      // cluster barrier the leader reads ranks 1..S-1 over DSMEM in fixed rank order; a
      // second barrier keeps the other CTAs' SMEM alive until the leader is done
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int m4 = 0; m4 < TOK / 4; ++m4)
          reinterpret_cast<float4*>(part)[(j * ROWS + row) * (TOK / 4) + m4] =
              make_float4(acc[j][4 * m4], acc[j][4 * m4 + 1], acc[j][4 * m4 + 2], acc[j][4 * m4 + 3]);
      if (MODE == MODE_RMS && warp == 2 && lane < TOK)
        part[R * ROWS * TOK + lane] = ssq_own[lane];
      if (warp == 2 && lane == 0) TC_TRACE(8);
      cluster_sync_all();  // (1) partials visible cluster-wide; warps 0 and 1 join below
      if (warp == 2 && lane == 0) TC_TRACE(9);
      write_z = rank == 0;
      if (write_z) {
        for (int r = 1; r < S; ++r) {  // fixed rank order
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const uint32_t src = mapa_shared(part + (j * ROWS + row) * TOK, lead + (uint32_t)r);
#pragma unroll
            for (int m4 = 0; m4 < TOK / 4; ++m4) {
              const float4 p = ld_cluster_v4(src + m4 * 16);
              acc[j][4 * m4] += p.x; acc[j][4 * m4 + 1] += p.y; acc[j][4 * m4 + 2] += p.z; acc[j][4 * m4 + 3] += p.w;
            }
          }
          if (MODE == MODE_RMS) {
            const uint32_t ss = mapa_shared(part + R * ROWS * TOK, lead + (uint32_t)r);
#pragma unroll
            for (int m4 = 0; m4 < TOK / 4; ++m4) {
              const float4 p = ld_cluster_v4(ss + m4 * 16);
              ssq[4 * m4] += p.x; ssq[4 * m4 + 1] += p.y; ssq[4 * m4 + 2] += p.z; ssq[4 * m4 + 3] += p.w;
            }
          }
        }
      }
      if (warp == 2 && lane == 0) TC_TRACE(10);
      cluster_sync_all();  // (2) the leader has read every remote partial
      if (warp == 2 && lane == 0) TC_TRACE(11);
    } else if (S > 1) {
      // global mode: publish this CTA's partial, count arrivals on the tile; the last reduces
      float4* mine = g_dtc_part[slot][blockIdx.x];
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int m4 = 0; m4 < TOK / 4; ++m4)
          __stcg(mine + (j * ROWS + row) * (TOK / 4) + m4,
                 make_float4(acc[j][4 * m4], acc[j][4 * m4 + 1], acc[j][4 * m4 + 2], acc[j][4 * m4 + 3]));
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
        float tot[R][TOK], st[TOK];
#pragma unroll
        for (int m = 0; m < TOK; ++m) {
          st[m] = 0.f;
#pragma unroll
          for (int j = 0; j < R; ++j) tot[j][m] = 0.f;
        }
        for (int r = 0; r < S; ++r) {  // fixed rank order, own partial from registers
          const float4* src = g_dtc_part[slot][tile * S + r];
#pragma unroll
          for (int j = 0; j < R; ++j)
#pragma unroll
            for (int m4 = 0; m4 < TOK / 4; ++m4) {
              const float4 p = r == rank ? make_float4(acc[j][4 * m4], acc[j][4 * m4 + 1], acc[j][4 * m4 + 2],
                                                       acc[j][4 * m4 + 3])
                                         : __ldcg(src + (j * ROWS + row) * (TOK / 4) + m4);
              tot[j][4 * m4] += p.x; tot[j][4 * m4 + 1] += p.y; tot[j][4 * m4 + 2] += p.z; tot[j][4 * m4 + 3] += p.w;
            }
          if (MODE == MODE_RMS) {
#pragma unroll
            for (int m4 = 0; m4 < TOK / 4; ++m4) {
              const float4 p = __ldcg(&g_dtc_ssq[slot][tile * S + r][m4]);
              st[4 * m4] += p.x; st[4 * m4 + 1] += p.y; st[4 * m4 + 2] += p.z; st[4 * m4 + 3] += p.w;
            }
          }
        }
#pragma unroll
        for (int m = 0; m < TOK; ++m) {
          ssq[m] = st[m];
#pragma unroll
          for (int j = 0; j < R; ++j) acc[j][m] = tot[j][m];
        }
      }
    }
    TC_EPI(7);
    if (write_z) {
      const float invK = 1.0f / (float)K;
      float rr[TOK];
#pragma unroll
      for (int m = 0; m < TOK; ++m)
        rr[m] = MODE == MODE_RMS ? rsqrtf(fmaf(ssq[m], invK, eps))
                                 : (MODE == MODE_NONE && row_scale != nullptr && m < M ? __ldg(row_scale + m) : 1.0f);
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int n = n0 + j * ROWS + row;
        if (R == 1 && rope_blk) {
          // RoPE (Fig 5(b)): the pair partner of W* row n is row n^1, held by lane^1; cos/sin are
          // scaled once per token by r * qk (shared by every head)
          float pv[TOK];
#pragma unroll
          for (int m = 0; m < TOK; ++m) pv[m] = __shfl_xor_sync(0xffffffffu, acc[j][m], 1);
          float sc[TOK];  // per-token scale of this row's head: r (Fig 5(b)) or the head's s_b (Fig 6(b))
#pragma unroll
          for (int m = 0; m < TOK; ++m) sc[m] = rr[m];
          float g_own = 1.0f, g_pair = 1.0f;
          if (rope.g_q != nullptr) {
            // QK-norm: MS of each token's head over the head's rows (h / 32 warps of this tile)
            float* red = reinterpret_cast<float*>(smem + 65536);  // [4 warps][TOK], ring is free here
#pragma unroll
            for (int m = 0; m < TOK; ++m) {
              float q = acc[j][m] * acc[j][m];
#pragma unroll
              for (int off = 16; off > 0; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
              if (lane == 0) red[q4 * TOK + m] = q;
            }
            named_bar_sync(3, 128);
            const int wph = rope.h / 32;                 // warps per head (h = 32, 64 or 128)
            const int w0 = (int)(q4 / (uint32_t)wph) * wph;
#pragma unroll
            for (int m = 0; m < TOK; ++m) {
              float ss = 0.f;
              for (int w = 0; w < wph; ++w) ss += red[(w0 + w) * TOK + m];
              sc[m] = rsqrtf(fmaf(rope.eps_qk, 1.0f / (rr[m] * rr[m]), ss / (float)rope.h));
            }
            if (n < rope.n) {
              const float* gsrc = n < rope.n_q ? rope.g_q : rope.g_k;
              g_own = __ldg(gsrc + n % rope.h);
              g_pair = __ldg(gsrc + (n ^ 1) % rope.h);
            }
          }
          if (n < N && n < rope.n) {
            const float sgn = (n & 1) ? 1.0f : -1.0f;  // y0 = x0 c g0 - x1 s g1, y1 = x1 c g1 + x0 s g0
#pragma unroll
            for (int m = 0; m < TOK; ++m) {
              if (m < M) {
                const float rq = sc[m] * rope.qk;
                z[(size_t)m * N + n] =
                    __float2bfloat16_rn(fmaf(acc[j][m], rc[m] * rq * g_own, sgn * pv[m] * (rs[m] * rq * g_pair)));
              }
            }
            continue;
          }
        } else if (R >= 2 && MODE == MODE_RMS && rope.pos != nullptr && rope.g_q == nullptr &&
                   n0 + j * ROWS < rope.n) {
          float pv[TOK];
#pragma unroll
          for (int m = 0; m < TOK; ++m) pv[m] = __shfl_xor_sync(0xffffffffu, acc[j][m], 1);
          if (n < N && n < rope.n) {
            const int hh = rope.h >> 1;
            const int i = (n % rope.h) >> 1;
            const float sgn = (n & 1) ? 1.0f : -1.0f;
#pragma unroll
            for (int m = 0; m < TOK; ++m) {
              if (m < M) {
                const int pos = __ldg(rope.pos + m);
                const float rq = rr[m] * rope.qk;
                const float c = __ldg(rope.cos_tab + (size_t)pos * hh + i) * rq;
                const float sn = __ldg(rope.sin_tab + (size_t)pos * hh + i) * rq;
                z[(size_t)m * N + n] = __float2bfloat16_rn(fmaf(acc[j][m], c, sgn * pv[m] * sn));
              }
            }
            continue;
          }
        }
        if (n < N) {
          const float cb = cstar != nullptr ? __ldg(cstar + n) : 0.0f;
#pragma unroll
          for (int m = 0; m < TOK; ++m)
            if (m < M) z[(size_t)m * N + n] = __float2bfloat16_rn(fmaf(acc[j][m], rr[m], cb));
        }
      }
    }
  }
  if (warp == 2 && lane == 0) TC_TRACE(12);
  TC_EPI(4);
  if (push) {
    if (rank == 0 || warp != 2) cluster_wait();  // pairs with the arrive at the start (peer warp 2 waited above)
  } else if (S > 1 && use_cluster && warp < 2) {
    cluster_sync_all();
    cluster_sync_all();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TC_TRACE(13);
  TC_EPI(5);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TCOLS);
  }
  TC_EPI(6);
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
template <int MODE, int R, int KB>
const void* dtc_kernel() {
  return (const void*)flashnorm_gemv_tc_kernel<MODE, R, KB>;
}
template <int R, int KB>
const void* dtc_fptr_rk(int mode) {
  return mode == MODE_RMS ? dtc_kernel<MODE_RMS, R, KB>() : mode == MODE_DYT ? dtc_kernel<MODE_DYT, R, KB>()
                                                                             : dtc_kernel<MODE_NONE, R, KB>();
}
const void* dtc_fptr(int mode, int R, int KB) {
  if (R == 1) return KB == 2 ? dtc_fptr_rk<1, 2>(mode) : dtc_fptr_rk<1, 1>(mode);
  return R == 2 ? dtc_fptr_rk<2, 1>(mode) : dtc_fptr_rk<4, 1>(mode);
}
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e != nullptr ? atoi(e) : dflt;
}
// A/B knobs (defaults = the measured best): FN_DECODE_STAGES ring depth cap, FN_DECODE_PUSH
// push-mode cluster reduction, FN_DECODE_PF2 partner-slice L2 prefetch
int dtc_flags() {
  // LSU prefetch of the whole own slice (FN_DECODE_LSUPF=1) measured 25 % below the HBM rate on long
  // streams (N = 18432: 5.05 vs 6.78 TB/s) and no better on config 2 than a bounded TMA prefetch
  // (FN_DECODE_L2PF stages beyond the ring): off by default
  static const int f = (env_int("FN_DECODE_PUSH", 1) ? 1 : 0) | (env_int("FN_DECODE_PF2", 0) ? 2 : 0) |
                       (env_int("FN_DECODE_LSUPF", 0) & 7) << 2 |  // bit 2 of LSUPF: evict_normal hint
                       (env_int("FN_DECODE_PDL_LATE", 0) ? 64 : 0);
  return f;
}
size_t dtc_recv_bytes(int R, int S) {
  return (dtc_flags() & 1) && S > 1 ? (size_t)(S - 1) * (R * dtc::ROWS * dtc::TOK + dtc::TOK) * 4 : 0;
}
// tok: resident-token stages (0 = tokens ride the ring)
size_t dtc_smem_for(int R, int KB, int stages, int S, int tok) {
  size_t ring;
  if (tok > 0) ring = 1024 + (size_t)stages * dtc::Cfg<1, 1>::W_STAGE + (size_t)tok * dtc::T_STAGE + 1024;
  else ring = R == 1 ? (KB == 2 ? dtc::Cfg<1, 2>::smem(stages) : dtc::Cfg<1, 1>::smem(stages))
                     : R == 2 ? dtc::Cfg<2, 1>::smem(stages) : dtc::Cfg<4, 1>::smem(stages);
  return ring + dtc_recv_bytes(R, S);
}
// deepest ring (<= the default depth) that fits the SMEM budget beside the receive slots
int dtc_stages(int R, int KB, int S, int tok) {
  static const int cap = env_int("FN_DECODE_STAGES", 0);
  int st = cap >= 2 ? cap : (tok > 0 ? 13 : ((R * KB) == 1 ? dtc::Cfg<1, 1>::STAGES : dtc::Cfg<2, 1>::STAGES));
  while (st > 2 && dtc_smem_for(R, KB, st, S, tok) > dtc::SMEM_MAX - 256) --st;
  return st;
}
size_t dtc_smem(int R, int KB, int S, int tok) { return dtc_smem_for(R, KB, dtc_stages(R, KB, S, tok), S, tok); }
cudaError_t dtc_set_attr(int mode, int R, int KB) {
  // budget less 256 B of static shared memory headroom (debug/trace builds add some)
  return ensure_smem_attr(dtc_fptr(mode, R, KB), (int)dtc::SMEM_MAX - 256);
}
// can `clusters` clusters of C CTAs each (tile height R x 128, K split S) be resident at once?
bool cluster_fits(int mode, int R, int KB, int S, int C, int clusters, int tok) {
  if (dtc_set_attr(mode, R, KB) != cudaSuccess) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * C);
  cfg.blockDim = dim3(dtc::THREADS);
  cfg.dynamicSmemBytes = dtc_smem(R, KB, S, tok);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  return cudaOccupancyMaxActiveClusters(&n, dtc_fptr(mode, R, KB), &cfg) == cudaSuccess && n >= clusters;
}
struct DtcPlan {
  int R, S, cluster, T;  // cluster: CTAs per cluster (T tiles x S splits), 0 = global-memory reduction
  int KB;                // 64-wide k blocks per ring stage (2: one 32 KiB 3-D TMA box, R = 1, K % 64 == 0)
  int tok;               // resident-token stages per CTA (0: tokens ride the ring)
};
// Tile height (R x 128 rows) and K split S, with the S CTAs of a tile in one co-resident
// cluster (DSMEM reduction).  R = 1 whenever its tiles fit the SMs; R = 2 extends the kernel
// to N <= 256 * #SMs.  (Config 2, N = 6144: R = 1 -> 48 tiles x clusters of 2 (3 do not fit:
// 45 max) = 96 CTAs, 10.2 us; R = 2 -> 24 tiles x clusters of 5 = 120 CTAs measured slower,
// 13.2 us: the 5-way DSMEM reduction and the shallower 32 KiB-stage ring cost more than the
// extra SMs bring.)
DtcPlan dtc_plan(int mode, int K, int N, int num_sms) {
  using namespace dtc;
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, DtcPlan> cache;
  const auto key = std::make_tuple(mode, K, N, num_sms);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const int nkb = (K + BK - 1) / BK;
  const int cap = std::min(num_sms, MAX_CTAS);
  static const int s_env = [] {
    const char* e = getenv("FN_DECODE_SMAX");  // A/B knob: cap on the K split
    return e != nullptr ? atoi(e) : MAX_S;
  }();
  static const int t_env = env_int("FN_DECODE_TMAX", 4);          // A/B knob: cap on tiles per cluster
  static const int force_global = env_int("FN_DECODE_GLOBAL", 0);  // A/B knob: global-memory split-K reduction
  // A/B knob: k blocks per stage.  2 = 32 KiB 3-D boxes (6-stage ring): config 2 9.79 vs 9.70 us for
  // 16 KiB boxes with the bounded prefetch, long streams equal; default 1
  static const int kb_env = env_int("FN_DECODE_KB", 1);
  static const int tokres_env = env_int("FN_DECODE_TOKRES", 1);  // A/B knob: resident token slice
  DtcPlan best{1, 1, 0, 1, 1, 0};
  int best_ctas = -1;
  for (int R = 1; R <= 4; R *= 2) {
    const int tiles = (N + R * ROWS - 1) / (R * ROWS);
    if (tiles > cap) continue;
    if (R > 1 && best_ctas > 0) break;  // taller tiles only when shorter ones do not fit the SMs
    const int KB = (R == 1 && K % BK == 0 && kb_env == 2) ? 2 : 1;
    const int nst = (nkb + KB - 1) / KB;  // ring stages of the whole K
    // R = 4 (N up to 512 x #SMs) runs unsplit: the split-K partial buffers hold R <= 2 tiles
    const int smax = R == 4 ? 1 : std::max(1, std::min(std::min(cap / tiles, std::min(MAX_S, s_env)), nst));
    // the most CTAs (tiles x S <= #SMs) whose clusters of T tiles x S splits are all co-resident;
    // T > 1 packs several tiles' split groups into one cluster, which lets S = 3 fit where
    // clusters of 3 do not (GPC shapes: 45 clusters of 3, but 24 of 6 on this part)
    // tokens resident when the per-CTA slice (ceil(stages / S) x 2 KiB) stays small
    auto tok_for = [&](int S) {
      const int tm = (nst + S - 1) / S;
      // measured (config 2): DyT 11.1 -> ~10 us (the transform leaves the per-stage path); RMS / none
      // slower with the shallower W* ring (9 vs 12 stages), so only DyT keeps its tokens resident
      return (tokres_env && mode == MODE_DYT && R == 1 && KB == 1 && tm * T_STAGE <= TOK_MAX_BYTES &&
              tm <= TOK_GS * TOK_GROUPS) ? tm : 0;
    };
    DtcPlan p{R, 1, 0, 1, KB, tok_for(1)};
    for (int S = smax; S > 1 && !force_global && p.S == 1; --S)
      for (int T = 1; T <= t_env && T * S <= MAX_S; T *= 2) {
        if (tiles % T) break;
        if (cluster_fits(mode, R, KB, S, T * S, tiles / T, tok_for(S))) {
          p = DtcPlan{R, S, T * S, T, KB, tok_for(S)};
          break;
        }
      }
    if (p.S == 1 && smax > 1) p = DtcPlan{R, smax, 0, 1, KB, tok_for(smax)};  // global-memory reduction
    const int ctas = tiles * p.S;
    if (ctas > best_ctas) { best = p; best_ctas = ctas; }
  }
  if (env_int("FN_DECODE_VERBOSE", 0))
    fprintf(stderr, "[flashnorm] decode plan K=%d N=%d: R=%d KB=%d S=%d T=%d cluster=%d tok=%d stages=%d smem=%zu\n",
            K, N, best.R, best.KB, best.S, best.T, best.cluster, best.tok, dtc_stages(best.R, best.KB, best.S, best.tok),
            dtc_smem(best.R, best.KB, best.S, best.tok));
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, best);
  return best;
}
}  // namespace

int gemv_tc_split(int K, int N, int num_sms) { return dtc_plan(MODE_RMS, K, N, num_sms).S; }

bool gemv_tc_supported(int M, int N, int num_sms) {
  return M >= 1 && M <= dtc::TOK && (N + 4 * dtc::ROWS - 1) / (4 * dtc::ROWS) <= std::min(num_sms, dtc::MAX_CTAS);
}

cudaError_t launch_gemv_tc(const CUtensorMap& tw, const CUtensorMap& ta, const float* cstar, __nv_bfloat16* z,
                           int M, int K, int N, float eps, float alpha, int mode, int num_sms, cudaStream_t stream,
                           const float* row_scale, RopeParams rope, const __nv_bfloat16* wptr,
                           const __nv_bfloat16* aptr) {
  using namespace dtc;
  const DtcPlan p = dtc_plan(mode, K, N, num_sms);
  if (cudaError_t e = dtc_set_attr(mode, p.R, p.KB); e != cudaSuccess) return e;
  const void* fptr = dtc_fptr(mode, p.R, p.KB);
  const int tiles = (N + p.R * ROWS - 1) / (p.R * ROWS);
  int S = p.S, use_cluster = p.cluster;  // CTAs per cluster (0: none)
  // global-mode partial-buffer slot: launches in flight together use different slots
  static std::atomic<unsigned> seq{0};
  int slot = (int)(seq.fetch_add(1u) % SLOTS);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles * S);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = dtc_smem(p.R, p.KB, S, p.tok);
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = use_cluster ? use_cluster : 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  static const int l2pf = [] {
    const char* e = getenv("FN_DECODE_L2PF");  // A/B knob: W* stages per CTA prefetched to L2 pre-wait
    // measured on config 2 (graph, 8 rotating W*): 0 / 4 / 8 / 12 stages -> 10.6 / 10.1 / 9.71 / 9.70 us
    return e != nullptr ? atoi(e) : 12;
  }();
  int stages = dtc_stages(p.R, p.KB, S, p.tok);
  int flags = dtc_flags() | (p.tok > 0 ? 32 | (p.tok << 8) : 0);
  void* args[] = {(void*)&tw, (void*)&ta, (void*)&cstar, (void*)&z, (void*)&M, (void*)&K, (void*)&N,
                  (void*)&eps, (void*)&alpha, (void*)&S, (void*)&slot, (void*)&use_cluster, (void*)&row_scale,
                  (void*)&rope, (void*)&l2pf, (void*)&stages, (void*)&flags, (void*)&wptr,
                  (void*)&aptr};
  return cudaLaunchKernelExC(&cfg, fptr, args);
}

int gemv_tc_tile_rows(int mode, int K, int N, int num_sms) { return dtc_plan(mode, K, N, num_sms).R * dtc::ROWS; }
int gemv_tc_kblocks(int mode, int K, int N, int num_sms) { return dtc_plan(mode, K, N, num_sms).KB; }

}  // namespace fn
