// gemm2_sm100.cu — K3 (CTA-pair variant): the prefill FlashNorm GEMM on 2-SM tcgen05.
//
//   z[m][j] = RN( fma( sum_k a[m][k] W*t[j][k],  rsqrt(ssq_m/K + eps),  c*_j ) )
//
// Same method as gemm_sm100.cu (deferred normalization; the RMS reduced by a warp
// group beside the tensor core, Fig 8(c)), but each 256x256 output tile is computed
// by a CTA PAIR with tcgen05.mma.cta_group::2: CTA r of the pair holds A rows
// [m0+128r, +128) and W* rows [n0+128r, +128) of every K-block, the leader's MMA
// reads both halves, and each CTA's TMEM receives its own 128 rows x 256 columns.
// Versus the 1-CTA kernel this halves the B operand traffic per SM (SMEM and L2),
// and 32 KiB stages allow a 6-deep ring.
//
// Roles per CTA (384 threads):  warp 0 TMA producer (both CTAs, signalling the
// leader's `full`), warp 1 MMA issuer (leader only), warp 2 TMEM allocator
// (cta_group::2), warps 4-7 ssq group, warps 8-11 epilogue.
//
// Stage flow (RMS): both CTAs' TMA complete on the leader's `full[s]`; the leader's
// MMA commit multicasts `mma_done[s]` to both CTAs; each CTA's ssq group squares
// its A half then (the tensor core has consumed the stage, so it has certainly
// landed in both CTAs — the peer CTA has no cheaper local "landed" signal: relaying
// `full` with a cluster-scope remote arrive was measured 2x slower), fences its
// loads (a store consuming them + bar.sync) and releases `empty[s]` for its own
// producer.  The ssq work of stage s overlaps the MMAs of stages s+1.. (Fig 8(c)).
// NONE mode: the commit releases `empty[s]` directly.  DyT stays on the 1-CTA kernel.
//
// ssq reuse: the tiles of one CTA pair revisit the same 256-row M blocks (the
// schedule walks M fastest so concurrent pairs share W* tiles in L2), so each CTA
// keeps the reduced ssq of its 128 rows in a small direct-mapped SMEM table keyed
// by M block.  A revisited block costs no SMEM reads; its stages are released by
// the MMA commit alone.  The MMA thread mirrors the table's tags to pick the
// commit target, so both sides take identical decisions without communicating.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <type_traits>

namespace fn {

namespace gemm2 {
constexpr int BM = 128;          // rows per CTA (pair tile = 256)
constexpr int BN = 256;          // pair tile columns (accumulator width per CTA)
constexpr int BNH = BN / 2;      // W* rows loaded per CTA
constexpr int BK = 64;
constexpr int STAGES = 6;
constexpr int A_STAGE = BM * BK * 2;   // 16 KiB
constexpr int B_STAGE = BNH * BK * 2;  // 16 KiB
constexpr int THREADS = 384;
constexpr int TMEM_COLS = 2 * BN;
constexpr int BAR_BYTES = 1024;
constexpr int SSQ_SLOTS = 16;          // per-CTA cache of reduced row ssq, by M block
static_assert(SSQ_SLOTS == PAIR_SSQ_SLOTS, "the host schedule mirrors this cache");
constexpr int SMEM_BYTES = 1024 + STAGES * (A_STAGE + B_STAGE) + BAR_BYTES + (4 + SSQ_SLOTS) * BM * 4 + 32 +
                             (2 + SSQ_SLOTS) * BM * 4 +  // + LayerNorm mean buffers
                             4 * 256 * 4;                // + the tile's c* per epilogue warp
// the pair tile width is a template parameter: 256 (default) or 224 (picked by the host when it
// evens out the last wave of tiles over the CTA pairs, gemm2_pick_bn); TMEM stays 2 x 256 columns
constexpr int smem_bytes(int bn) { return SMEM_BYTES - STAGES * (B_STAGE - (bn / 2) * BK * 2); }
}  // namespace gemm2

FN_DEVICE unsigned sk_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FN_DEVICE void sk_st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
FN_DEVICE uint64_t sk_gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifdef FN_SK_TRACE  // tools/micro/sk_trace.cu: per-CTA globaltimer stamps (ns) of the first 4 items
__device__ unsigned long long g_sk_trace[160][4][6];
#define SK_STAMP(li, e) do { if (lane == 0 && (li) < 4 && blockIdx.x < 160) g_sk_trace[blockIdx.x][li][e] = sk_gtime(); } while (0)
__device__ unsigned long long g_sk_chunk[160][4][4][8][2];  // [cta][item][epilogue warp][chunk][tmem ready, stored]
#define SK_CSTAMP(li, j, e) do { if (lane == 0 && (li) < 4 && blockIdx.x < 160 && (j) < 8) g_sk_chunk[blockIdx.x][li][ew][j][e] = sk_gtime(); } while (0)
#else
#define SK_STAMP(li, e)
#define SK_CSTAMP(li, j, e)
#endif

template <int MODE, int BN_ = gemm2::BN, bool TBL = true, bool SK = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm2::THREADS, 1)
    flashnorm_gemm2_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                           GemmParams p,
                           const __grid_constant__ std::conditional_t<TBL, PairSchedule, PairScheduleNone> sched) {
  using namespace gemm2;
  constexpr int BN = BN_;                // pair tile columns
  constexpr int BNH = BN / 2;            // W* rows loaded per CTA
  constexpr int B_STAGE = BNH * BK * 2;  // 16 / 14 KiB
  static_assert(BN % 32 == 0 && BN <= 256, "pair tile width");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* full = bars;                    // [STAGES] leader: both CTAs' TMA bytes landed
  uint64_t* empty = bars + STAGES;          // [STAGES] local: stage may be refilled
  uint64_t* mma_done = bars + 2 * STAGES;   // [STAGES] local: the MMA finished reading the stage (multicast commit)
  uint64_t* tfull = bars + 3 * STAGES;      // [2] local: accumulator ready (multicast commit)
  uint64_t* tempty = tfull + 2;             // [2] leader: both CTAs drained the accumulator
  uint64_t* sfull = tempty + 2;             // [2] local ssq handshake
  uint64_t* sempty = sfull + 2;             // [2]
  uint64_t* afull = sempty + 2;             // [STAGES] DyT: local raw-A landed
  uint64_t* ready = afull + STAGES;         // [STAGES] DyT (leader): both CTAs' prologue done
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ready + STAGES);
  float* ssq_buf = reinterpret_cast<float*>(smem + STAGES * (A_STAGE + B_STAGE) + BAR_BYTES);  // [2][BM]
  float* ssq_fence = ssq_buf + 2 * BM;
  float* epi_fence = ssq_fence + BM;
  float* ssq_cache = epi_fence + BM;  // [SSQ_SLOTS][BM]
  uint8_t* sig_dst = reinterpret_cast<uint8_t*>(ssq_cache + SSQ_SLOTS * BM);  // 16 B: DyT peer signal landing
  const uint8_t* sig_src = sig_dst + 16;                                      // 16 B: its (unused) source
  float* mu_buf = reinterpret_cast<float*>(sig_dst + 32);  // [2][BM] LayerNorm (ln_u): row means
  float* mu_cache = mu_buf + 2 * BM;                       // [SSQ_SLOTS][BM]
  float* cst_smem = mu_cache + SSQ_SLOTS * BM;             // [4 warps][256] the tile's c*
  const bool ln = MODE == MODE_RMS && p.ln_u != nullptr;   // exact deferred LayerNorm (reading c29)
  // RMS with LOCAL A completion (p.rms_local): each CTA's A half lands on its own `afull`, the
  // ssq group reads it there while the MMA runs (release `empty` = MMA commit + ssq group), and
  // warp 3 relays "A landed" to the leader's `ready` (the peer with a 16-byte DSMEM bulk copy)
  const bool la = MODE == MODE_RMS && p.rms_local != 0;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      // RMS: ssq group (la: + MMA commit);  NONE/DyT: MMA commit
      mbar_init(&empty[s], la ? 2 : 1);
      mbar_init(&mma_done[s], 1);
      mbar_init(&afull[s], 1);
      mbar_init(&ready[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2);
      mbar_init(&sfull[b], 1);
      mbar_init(&sempty[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_holder, TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync_all();  // barrier inits + TMEM allocation visible pair-wide
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int num_tiles = p.num_tiles;  // pair tiles: num_m_blocks (of 256) x num_n_blocks
  const int nkb = p.num_k_blocks;
  const int rot = pair_tile_rotation(p, nclusters);
  auto next_tile = [&](int& j) -> int {
    if constexpr (TBL) {
      if (sched.waves > 0) return next_sched_tile(j, sched, cluster, nclusters);
    }
    return next_pair_tile(j, cluster, nclusters, rot, num_tiles);
  };
  // every role walks the same item sequence: whole tiles (k blocks [0, nkb)) or, with the
  // stream-K tail (SK), the pair's whole-tile waves and then its stream-K items (kernels.h)
  auto next_item = [&](int& j, PairItem& it) -> bool {
    if constexpr (SK) {
      if (j < p.sk_dp_waves) {
        it = PairItem{cluster + j * nclusters, 0, nkb, 0, -1};
        ++j;
        return true;
      }
      if (!sk_item(p, cluster, nclusters, j - p.sk_dp_waves, it)) return false;
      ++j;
      return true;
    } else {
      const int t = next_tile(j);
      if (t < 0) return false;
      it = PairItem{t, 0, nkb, 0, -1};
      return true;
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one()) {
      const uint32_t full0 = mapa_shared(&full[0], 0);  // leader's barrier array
      int stage = 0;
      uint32_t phase = 0;
      PairItem it;
      for (int jw = 0; next_item(jw, it);) {
        int m_blk, n_blk;
        tile_coords(it.tile, p, m_blk, n_blk);
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = full0 + stage * 8;
          if (MODE == MODE_DYT || la) {
            // raw A lands on a LOCAL barrier (DyT: this CTA's prologue warps transform it;
            // la: the ssq group reads it and warp 3 relays its arrival to the leader);
            // B still completes on the leader's `full`
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * B_STAGE);
            mbar_arrive_expect_tx(&afull[stage], A_STAGE);
            tma_load_2d(sA + stage * A_STAGE, &tmap_a, &afull[stage], kb * BK, m_blk * 2 * BM + rank * BM, kEvictLast);
          } else {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (A_STAGE + B_STAGE));
            tma_load_2d_pair(sA + stage * A_STAGE, &tmap_a, fb, kb * BK, m_blk * 2 * BM + rank * BM, kEvictLast);
          }
          tma_load_2d_pair(sB + stage * B_STAGE, &tmap_b, fb, kb * BK, n_blk * BN + rank * BNH, kEvictNormal);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader && elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(2 * BM, BN);
      int tag[SSQ_SLOTS];  // mirrors the ssq group's cache decisions (same sequence, same updates)
#pragma unroll
      for (int i = 0; i < SSQ_SLOTS; ++i) tag[i] = -1;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      PairItem it;
      for (int jw = 0; next_item(jw, it); ++local) {
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        int m_blk, n_blk_unused;
        tile_coords(it.tile, p, m_blk, n_blk_unused);
        const int slot = m_blk % SSQ_SLOTS;
        bool cached = false;
        if (it.kb0 == 0 && it.kb1 == nkb) {  // partial K ranges (stream-K) neither use nor fill the ssq cache
#pragma unroll
          for (int i = 0; i < SSQ_SLOTS; ++i)
            if (i == slot) { cached = tag[i] == m_blk; tag[i] = m_blk; }
        }
        uint64_t* release = (MODE == MODE_RMS && !cached && !la) ? mma_done : empty;
        mbar_wait(&tempty[as], aphase ^ 1);
        SK_STAMP(local, 0);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          if (MODE == MODE_DYT || la) mbar_wait(&ready[stage], phase);  // both CTAs' A ready (DyT: transformed)
          tc_fence_after();
          const uint64_t adesc = make_sw128_desc(smem_u32(sA + stage * A_STAGE));
          const uint64_t bdesc = make_sw128_desc(smem_u32(sB + stage * B_STAGE));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != it.kb0 || k != 0) ? 1u : 0u);
          umma_commit_pair_mc(&release[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair_mc(&tfull[as], 0x3);
        SK_STAMP(local, 1);
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ la relay (both CTAs)
    if (la && elect_one()) {
      const uint32_t ready0 = mapa_shared(&ready[0], 0);
      const uint32_t sig0 = mapa_shared(sig_dst, 0);  // 16-byte landing slot in the leader
      int stage = 0;
      uint32_t phase = 0;
      PairItem it;
      for (int jw = 0; next_item(jw, it);) {
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          mbar_wait(&afull[stage], phase);
          if (leader) mbar_arrive_expect_tx(&ready[stage], 16);  // + the peer's 16-byte signal
          else dsmem_signal16(sig0, sig_src, ready0 + stage * 8);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ ssq group (both CTAs)
    if (MODE == MODE_RMS) {
      const int t = threadIdx.x - 128;
      int tag[SSQ_SLOTS];
#pragma unroll
      for (int i = 0; i < SSQ_SLOTS; ++i) tag[i] = -1;
      uint32_t md_phase = 0;  // per-stage parity of mma_done (uncached tiles) / afull (la: every tile)
      // the barrier that says "this stage's A may be read": mma_done (consumed by the MMA, so it
      // has landed in both CTAs) or, with la, this CTA's own afull (landed; read beside the MMA)
      auto wait_a = [&](int st) {
        mbar_wait_warp(la ? &afull[st] : &mma_done[st], (md_phase >> st) & 1u);
        md_phase ^= 1u << st;
      };
      int stage = 0;
      int local = 0;
      PairItem it;
      for (int jw = 0; next_item(jw, it); ++local) {
        int m_blk, n_blk_unused;
        tile_coords(it.tile, p, m_blk, n_blk_unused);
        const int slot = m_blk % SSQ_SLOTS;
        bool cached = false;
        if (it.kb0 == 0 && it.kb1 == nkb) {  // mirrors the MMA thread: partial K ranges bypass the cache
#pragma unroll
          for (int i = 0; i < SSQ_SLOTS; ++i)
            if (i == slot) { cached = tag[i] == m_blk; tag[i] = m_blk; }
        }
        const int nk_it = it.kb1 - it.kb0;
        float ssq, mu = 0.f;
        if (cached) {
          // this CTA already reduced these 128 rows for an earlier N tile: the ring
          // stages of this tile are released by the MMA commit alone (la: plus this group's
          // arrival, after the stage landed, which keeps the group within one ring phase)
          if (la) {
            for (int kb = 0; kb < nkb; ++kb) {
              wait_a(stage);
              if (t == 0) mbar_arrive(&empty[stage]);
              if (++stage == STAGES) stage = 0;
            }
          } else {
            stage = (stage + nkb) % STAGES;
          }
          ssq = ssq_cache[slot * BM + t];
          if (ln) mu = mu_cache[slot * BM + t];
        } else if (ln) {
          // LayerNorm: sum(a - a0) and sum((a - a0)^2) with the shift a0 = a[m][0] (logical chunk 0
          // of stage kb = 0), so var = S2/K - (S1/K)^2 does not cancel for rows with a large mean;
          // ssq := K var (the epilogue's rsqrt(ssq/K + eps) is then LayerNorm's 1/sqrt(var + eps))
          // (s0, s1) and (q0, q1) as packed pairs {lo, hi}: lo elements -> s0 / q0, hi -> s1 / q1
          uint64_t S = 0, Q = 0, Sb = 0, Qb = 0, A0 = 0;  // two chains each (words x,y / z,w)
          float a0 = 0.f;
          for (int kb = 0; kb < nkb; ++kb) {
            wait_a(stage);
            const uint4* row = reinterpret_cast<const uint4*>(sA + stage * A_STAGE + t * 128);
            if (kb == 0) {
              a0 = bf16lo(row[t & 7].x);
              A0 = f2_pack(a0, a0);
            }
            // the last K block's columns >= K are TMA zero fill: they would add -a0 to S1 and
            // a0^2 to S2, so only the cmax logical 8-column chunks inside K are summed
            const int cmax = min(8, (p.K - kb * 64) >> 3);
            // all 8 loads in flight first (a guarded load per chunk serialised LDS -> use), then
            // the chunks inside K; the masked tail chunks are TMA zero fill, read but not summed
            uint4 v8[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) v8[c] = row[c ^ (t & 7)];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              if (cmax < 8 && c >= cmax) break;
              const uint4 v = v8[c];
              uint64_t D;
              D = f2_sub(f2_bf16x2(v.x), A0); S = f2_add(S, D); Q = f2_fma(D, D, Q);
              D = f2_sub(f2_bf16x2(v.y), A0); S = f2_add(S, D); Q = f2_fma(D, D, Q);
              D = f2_sub(f2_bf16x2(v.z), A0); Sb = f2_add(Sb, D); Qb = f2_fma(D, D, Qb);
              D = f2_sub(f2_bf16x2(v.w), A0); Sb = f2_add(Sb, D); Qb = f2_fma(D, D, Qb);
            }
            // the fence store issues only after every LDS above returned; the 128-thread barrier
            // drains it before the release (a per-warp release after __syncwarp raced in the batched
            // decode kernel's analogous ssq reads)
            ssq_fence[t] = (f2_lo(S) + f2_hi(S)) + (f2_lo(Q) + f2_hi(Q)) + (f2_lo(Sb) + f2_lo(Qb));
            named_bar_sync(1, 128);
            if (t == 0) mbar_arrive(&empty[stage]);
            if (++stage == STAGES) stage = 0;
          }
          const float S1 = (f2_lo(S) + f2_hi(S)) + (f2_lo(Sb) + f2_hi(Sb));
          const float S2 = (f2_lo(Q) + f2_hi(Q)) + (f2_lo(Qb) + f2_hi(Qb)), invK = 1.0f / (float)p.K;
          ssq = fmaxf(S2 - S1 * (S1 * invK), 0.0f);
          mu = fmaf(S1, invK, a0);
          ssq_cache[slot * BM + t] = ssq;
          mu_cache[slot * BM + t] = mu;
        } else {
          // (a stream-K item: the partial ssq of its k blocks; the finisher adds the contributor's)
          // packed pairs: P01 = (s0, s1) <- lo / hi of words x and z, P23 = (s2, s3) <- y and w
          uint64_t P01 = 0, P23 = 0;
          for (int kb = 0; kb < nk_it; ++kb) {
            wait_a(stage);
            const uint4* row = reinterpret_cast<const uint4*>(sA + stage * A_STAGE + t * 128);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint4 v = row[c ^ (t & 7)];
              uint64_t X;
              X = f2_bf16x2(v.x); P01 = f2_fma(X, X, P01);
              X = f2_bf16x2(v.y); P23 = f2_fma(X, X, P23);
              X = f2_bf16x2(v.z); P01 = f2_fma(X, X, P01);
              X = f2_bf16x2(v.w); P23 = f2_fma(X, X, P23);
            }
            ssq_fence[t] = (f2_lo(P01) + f2_hi(P01)) + (f2_lo(P23) + f2_hi(P23));  // issues only after every LDS above returned
            named_bar_sync(1, 128);                 // drains the 128 stores
            if (t == 0) mbar_arrive(&empty[stage]);
            if (++stage == STAGES) stage = 0;
          }
          ssq = (f2_lo(P01) + f2_hi(P01)) + (f2_lo(P23) + f2_hi(P23));
          if (it.kb0 == 0 && it.kb1 == nkb) ssq_cache[slot * BM + t] = ssq;
        }
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait_warp(&sempty[as], aphase ^ 1);
        ssq_buf[as * BM + t] = ssq;
        if (ln) mu_buf[as * BM + t] = mu;
        named_bar_sync(1, 128);
        if (t == 0) mbar_arrive(&sfull[as]);
      }
    }
    if (MODE == MODE_DYT) {
      // prologue: rewrite this CTA's A half with tanh(alpha a) (bf16x2 multiply + MUFU tanh),
      // make the generic writes visible to the tensor core, and report to the leader
      const int t = threadIdx.x - 128;
      const __nv_bfloat162 alpha2 = __floats2bfloat162_rn(p.alpha, p.alpha);
      const uint32_t ready0 = mapa_shared(&ready[0], 0);
      const uint32_t sig0 = mapa_shared(sig_dst, 0);  // 16-byte landing slot in the leader
      int stage = 0;
      uint32_t phase = 0;
      PairItem it;
      for (int jw = 0; next_item(jw, it);) {
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          mbar_wait_warp(&afull[stage], phase);
          uint4* row = reinterpret_cast<uint4*>(sA + stage * A_STAGE + t * 128);
          uint4 v[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = row[c ^ (t & 7)];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint32_t* w = reinterpret_cast<uint32_t*>(&v[c]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&w[q]);
              x = __hmul2(x, alpha2);
              w[q] = tanh_approx_bf16x2(*reinterpret_cast<uint32_t*>(&x));
            }
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) row[c ^ (t & 7)] = v[c];
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (t == 0) {
            if (leader) mbar_arrive_expect_tx(&ready[stage], 16);  // + the peer's 16-byte signal
            else dsmem_signal16(sig0, sig_src, ready0 + stage * 8);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const uint32_t ew = warp - 8;
    const uint32_t tempty0 = mapa_shared(&tempty[0], 0);
    int local = 0;
    const float invK = 1.0f / static_cast<float>(p.K);
    PairItem it;
    for (int jw = 0; next_item(jw, it); ++local) {
      int m_blk, n_blk;
      tile_coords(it.tile, p, m_blk, n_blk);
      const int as = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      const int rl = ew * 32 + lane;  // this thread's row within the CTA's 128
      if (ew == 0) SK_STAMP(local, 2);
      float r = 1.0f, mu = 0.f, ssq = 0.f, ssq_part = 0.f;
      // stream-K (kernels.h): the partial of the other pair's k range lives in sk_part
      float* skp = nullptr;
      float* sks = nullptr;
      unsigned* skf = nullptr;
      if (SK && it.fix != 0) {
        // [32-column chunk j][float4 q][row]: a warp's 32 rows of one float4 are 512 contiguous bytes
        skp = p.sk_part + ((size_t)it.sk * 2 + rank) * (BM * 256) + (size_t)rl * 4;
        sks = p.sk_part + (size_t)p.sk_tiles * 2 * BM * 256 + ((size_t)it.sk * 2 + rank) * BM + rl;
        skf = p.sk_flag + it.sk * 2 + rank;
      }
      const bool fin = SK && (it.fix == 1 || it.fix == 3);
      if (fin) {  // finisher: wait for the contributor's partial (acquire), before this item's ssq
        if (ew == 0 && lane == 0) {
          const uint64_t t0 = sk_gtime();
          while (sk_ld_acquire(skf) == 0u) {
            __nanosleep(64);
            if (sk_gtime() - t0 > 2000000000ull) __trap();  // a lost partial: fail loudly, never hang
          }
        }
        named_bar_sync(2, 128);
        if (ew == 0) SK_STAMP(local, 3);
        if (MODE == MODE_RMS) ssq_part = __ldcg(sks);
        // fix 3: the partial into the OTHER accumulator buffer while this item's MMA still runs:
        // the finisher is its pair's last item, so that buffer is drained (this warp group's
        // previous epilogue) and never written again; the chunk loop then reads both from TMEM
        const uint32_t pbuf = tmem_base + ((ew * 32u) << 16) + (as ^ 1) * BN;
#pragma unroll 1
        for (int j = 0; j < (it.fix == 3 ? BN / 32 : 0); ++j) {
          const float4* src = reinterpret_cast<const float4*>(skp) + j * 8 * BM;
          uint32_t pv[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 c4 = __ldcg(src + q * BM);
            pv[4 * q] = __float_as_uint(c4.x); pv[4 * q + 1] = __float_as_uint(c4.y);
            pv[4 * q + 2] = __float_as_uint(c4.z); pv[4 * q + 3] = __float_as_uint(c4.w);
          }
          tmem_st_32x32b_x32(pbuf + j * 32, pv);
        }
        tmem_wait_st();
      }
      if (MODE == MODE_RMS) {
        mbar_wait_warp(&sfull[as], aphase);
        ssq = ssq_buf[as * BM + rl];
        if (ln) mu = mu_buf[as * BM + rl];
        epi_fence[rl] = ssq + mu;  // consumes both loads before the buffer is released
        named_bar_sync(2, 128);
        if (ew == 0 && lane == 0) mbar_arrive(&sempty[as]);
        if (fin) ssq = ssq_part + ssq;  // fixed order: earlier k blocks first
      }
      if (MODE == MODE_RMS) r = rsqrtf(fmaf(ssq, invK, p.eps));
      // the tile's c* slice to this warp's SMEM while the accumulator is still being produced (its
      // L2 round trip off the per-chunk chain below)
      float* cst_w = cst_smem + ew * 256;
      if (p.cstar != nullptr) {
        __syncwarp();  // the previous tile's reads of cst_w are done
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = n_blk * BN + lane * 8 + h * 4;
          float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (cc < p.N) cv = __ldg(reinterpret_cast<const float4*>(p.cstar + cc));
          reinterpret_cast<float4*>(cst_w)[lane * 2 + h] = cv;
        }
        __syncwarp();
      }
      mbar_wait_warp(&tfull[as], aphase);
      if (ew == 0) SK_STAMP(local, 4);
      tc_fence_after();
      const int row = m_blk * 2 * BM + rank * BM + rl;
      const uint32_t taddr = tmem_base + ((ew * 32u) << 16) + as * BN;
      if (SK && it.fix == 2) {
        // contributor: the fp32 accumulator (and the partial ssq) to sk_part, then release the flag
#pragma unroll 1
        for (int j = 0; j < BN / 32; ++j) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + j * 32, v);
          tmem_wait_ld();
          float4* dst = reinterpret_cast<float4*>(skp) + j * 8 * BM;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            __stcg(dst + q * BM, make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                        __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
        }
        if (MODE == MODE_RMS) __stcg(sks, ssq);
        tc_fence_before();
        named_bar_sync(2, 128);  // all 128 rows stored; TMEM reads of this buffer completed
        if (ew == 0 && lane == 0) {
          mbar_arrive_cluster(tempty0 + as * 8);
          __threadfence();
          sk_st_release(skf, 1u);
        }
        if (ew == 0) SK_STAMP(local, 5);
        continue;
      }
      if (MODE == MODE_RMS && p.glu_act >= 0 && p.glu_act != RELU_FFN) {
        // GLU epilogue: TMEM columns [0,128) = gate block n_blk, [128,256) = up block n_blk
        const int F = p.N / 2;
        const float s_row = p.glu_act == GLU_SILU ? r : r * r;  // output scale (reading c25)
        if (n_blk == 0 && row < p.M && p.s_out != nullptr) p.s_out[row] = s_row;
        __nv_bfloat16* hrow = p.z + static_cast<size_t>(row) * F + n_blk * (BN / 2);
#pragma unroll 1
        for (int j = 0; j < BN / 64; ++j) {
          uint32_t vg[32], vu[32];
          tmem_ld_32x32b_x32(taddr + j * 32, vg);
          tmem_ld_32x32b_x32(taddr + BN / 2 + j * 32, vu);
          tmem_wait_ld();
          uint32_t packed[16];
#pragma unroll
          for (int q = 0; q < 16; ++q)
            packed[q] = pack_bf16(glu_apply(p.glu_act, __uint_as_float(vg[2 * q]), __uint_as_float(vu[2 * q]), r),
                                  glu_apply(p.glu_act, __uint_as_float(vg[2 * q + 1]), __uint_as_float(vu[2 * q + 1]), r));
          if (row < p.M) {
            uint4* dst = reinterpret_cast<uint4*>(hrow + j * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              dst[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
          }
        }
        tc_fence_before();
        named_bar_sync(2, 128);
        if (ew == 0 && lane == 0) mbar_arrive_cluster(tempty0 + as * 8);
        continue;
      }
      if (MODE == MODE_NONE && p.row_scale != nullptr) r = row < p.M ? __ldg(p.row_scale + row) : 1.0f;
      const bool relu_ffn = MODE == MODE_RMS && p.glu_act == RELU_FFN;  // Fig 2(b): relu(acc), s = r
      if (relu_ffn) {
        if (n_blk == 0 && row < p.M && p.s_out != nullptr) p.s_out[row] = r;
      }
      const int n_base = n_blk * BN;
      __nv_bfloat16* zrow = p.z + static_cast<size_t>(row) * p.N + n_base;
      float head_sb = 1.0f;  // QK-norm: 1/RMS of the current Q/K head of this row (reading c28)
#pragma unroll 1
      for (int j = 0; j < BN / 32; ++j) {
        if (n_base + j * 32 >= p.N) break;  // warp-uniform
        uint32_t v[32];
        if (SK && it.fix == 1) {  // + the contributor's partial (earlier k blocks) from L2
          const float4* src = reinterpret_cast<const float4*>(skp) + j * 8 * BM;
          float4 pc[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) pc[q] = __ldcg(src + q * BM);  // in flight with the TMEM load
          tmem_ld_32x32b_x32(taddr + j * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            v[4 * q] = __float_as_uint(pc[q].x + __uint_as_float(v[4 * q]));
            v[4 * q + 1] = __float_as_uint(pc[q].y + __uint_as_float(v[4 * q + 1]));
            v[4 * q + 2] = __float_as_uint(pc[q].z + __uint_as_float(v[4 * q + 2]));
            v[4 * q + 3] = __float_as_uint(pc[q].w + __uint_as_float(v[4 * q + 3]));
          }
        } else if (SK && it.fix == 3) {  // + the partial staged in the other TMEM buffer
          uint32_t pv[32];
          tmem_ld_32x32b_x32(taddr + j * 32, v);
          tmem_ld_32x32b_x32(taddr + ((as ^ 1) - as) * BN + j * 32, pv);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = __float_as_uint(__uint_as_float(pv[q]) + __uint_as_float(v[q]));
        } else {
          tmem_ld_32x32b_x32(taddr + j * 32, v);
          tmem_wait_ld();
        }
        SK_CSTAMP(local, j, 0);
        float cb[32];
        if (p.cstar != nullptr) {
          const float4* c4 = reinterpret_cast<const float4*>(cst_w + j * 32);  // zero past N
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 cv = c4[q];
            cb[4 * q + 0] = cv.x; cb[4 * q + 1] = cv.y; cb[4 * q + 2] = cv.z; cb[4 * q + 3] = cv.w;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) cb[q] = 0.f;
        }
        uint32_t packed[16];
        if (MODE == MODE_RMS && p.rope.pos != nullptr && n_base + j * 32 < p.rope.n) {
          // Fig 5(b): cos/sin scaled once per token by r (and sqrt(1/sqrt h)), shared by all heads
          const int pos = row < p.M ? __ldg(p.rope.pos + row) : 0;
          const int hh = p.rope.h >> 1;
          const int col0 = n_base + j * 32;
          const bool qkn = p.rope.g_q != nullptr;
          if (qkn && col0 % p.rope.h == 0) {
            // Fig 6(b): the head's own RMS from the unscaled accumulator (s_a cancels); the head's
            // h / 32 chunks are read from TMEM once more for the sum of squares
            float ss = 0.f;
            for (int u = 0; u < p.rope.h / 32; ++u) {
              uint32_t w[32];
              tmem_ld_32x32b_x32(taddr + (j + u) * 32, w);
              tmem_wait_ld();
#pragma unroll
              for (int q = 0; q < 32; ++q) ss = fmaf(__uint_as_float(w[q]), __uint_as_float(w[q]), ss);
            }
            head_sb = rsqrtf(fmaf(p.rope.eps_qk, 1.0f / (r * r), ss / (float)p.rope.h));
          }
          const float rq = (qkn ? head_sb : r) * p.rope.qk;
          float gm[32];  // QK-norm weights of these 32 head dimensions (Fig 7(b)), else 1
          if (qkn) {
            const float* gsrc = (col0 < p.rope.n_q ? p.rope.g_q : p.rope.g_k) + (col0 % p.rope.h);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 g4 = __ldg(reinterpret_cast<const float4*>(gsrc) + q);
              gm[4 * q] = g4.x; gm[4 * q + 1] = g4.y; gm[4 * q + 2] = g4.z; gm[4 * q + 3] = g4.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) gm[q] = 1.0f;
          }
          const int i0 = ((n_base + j * 32) % p.rope.h) >> 1;  // 16 consecutive pair indices
          float cs[16], sn[16];
          if ((hh & 3) == 0 && i0 + 16 <= hh) {  // one head, 16-byte aligned: 4 x float4 each
            const float4* c4 = reinterpret_cast<const float4*>(p.rope.cos_tab + (size_t)pos * hh + i0);
            const float4* s4 = reinterpret_cast<const float4*>(p.rope.sin_tab + (size_t)pos * hh + i0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 c = __ldg(c4 + q), sv = __ldg(s4 + q);
              cs[4 * q] = c.x; cs[4 * q + 1] = c.y; cs[4 * q + 2] = c.z; cs[4 * q + 3] = c.w;
              sn[4 * q] = sv.x; sn[4 * q + 1] = sv.y; sn[4 * q + 2] = sv.z; sn[4 * q + 3] = sv.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const int i = ((n_base + j * 32 + 2 * q) % p.rope.h) >> 1;
              cs[q] = __ldg(p.rope.cos_tab + (size_t)pos * hh + i);
              sn[q] = __ldg(p.rope.sin_tab + (size_t)pos * hh + i);
            }
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            // y0 = x0 cos g0 - x1 sin g1, y1 = x1 cos g1 + x0 sin g0 (permuteg)
            const float c = cs[q] * rq, s = sn[q] * rq;
            const float x0 = __uint_as_float(v[2 * q]), x1 = __uint_as_float(v[2 * q + 1]);
            const float g0 = gm[2 * q], g1 = gm[2 * q + 1];
            packed[q] = pack_bf16(fmaf(x0, c * g0, -x1 * (s * g1)), fmaf(x1, c * g1, x0 * (s * g0)));
          }
        } else if (relu_ffn) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            packed[q] = pack_bf16(fmaxf(__uint_as_float(v[2 * q]), 0.0f), fmaxf(__uint_as_float(v[2 * q + 1]), 0.0f));
        } else if (ln) {
          // z = (acc - mu u_j) r + c*_j: the mean moved through the contraction (reading c29)
          float uu[32];
          const float4* u4 = reinterpret_cast<const float4*>(p.ln_u + n_base + j * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (n_base + j * 32 + q * 4 < p.N) x = __ldg(u4 + q);
            uu[4 * q + 0] = x.x; uu[4 * q + 1] = x.y; uu[4 * q + 2] = x.z; uu[4 * q + 3] = x.w;
          }
#pragma unroll
          for (int q = 0; q < 16; ++q)
            packed[q] = pack_bf16(fmaf(fmaf(-mu, uu[2 * q], __uint_as_float(v[2 * q])), r, cb[2 * q]),
                                  fmaf(fmaf(-mu, uu[2 * q + 1], __uint_as_float(v[2 * q + 1])), r, cb[2 * q + 1]));
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            packed[q] = pack_bf16(fmaf(__uint_as_float(v[2 * q]), r, cb[2 * q]),
                                  fmaf(__uint_as_float(v[2 * q + 1]), r, cb[2 * q + 1]));
        }
#ifdef FN_SK_TRACE
        if (p.stg == 2) {  // trace experiment: no output stores
          if (packed[0] == 0x12345678u && packed[15] == 0x9abcdef0u) p.z[0] = __float2bfloat16(1.f);
        } else
#endif
        if (row < p.M) {
          if (p.ndst == 0) {
            uint4* dst = reinterpret_cast<uint4*>(zrow + j * 32);
            if (p.stg == 1 && n_base + j * 32 + 32 <= p.N && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
              // two full 32-byte sectors per lane (256-bit stores)
              st_global_v8(dst, make_uint4(packed[0], packed[1], packed[2], packed[3]),
                           make_uint4(packed[4], packed[5], packed[6], packed[7]));
              st_global_v8(dst + 2, make_uint4(packed[8], packed[9], packed[10], packed[11]),
                           make_uint4(packed[12], packed[13], packed[14], packed[15]));
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (n_base + j * 32 + q * 8 < p.N)
                  dst[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
            }
          } else {
            // fused gather: the same 64-byte row segment to every destination (st.global to a
            // peer-mapped address is an NVLink store), overlapped with the next tile's mainloop
            const size_t off = static_cast<size_t>(row) * p.ldz + p.col0 + n_base + j * 32;
#pragma unroll 1
            for (int d = 0; d < p.ndst; ++d) {
              uint4* dst = reinterpret_cast<uint4*>(p.zdst[d] + off);
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (n_base + j * 32 + q * 8 < p.N) {
                  const uint4 v4 = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
                  if (p.mc) multimem_st_v4(dst + q, v4);  // NVLS: one store, every rank's buffer
                  else dst[q] = v4;
                }
            }
          }
        }
        SK_CSTAMP(local, j, 1);
      }
      tc_fence_before();
      named_bar_sync(2, 128);  // all 4 warps' TMEM loads of this buffer completed
      if (ew == 0 && lane == 0) {
        mbar_arrive_cluster(tempty0 + as * 8);  // one arrival per CTA, at the leader
        if (fin) *skf = 0u;                     // consumed: zero for the next call
      }
      if (ew == 0) SK_STAMP(local, 5);
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer must be done with the leader's barriers / TMEM
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

int gemm2_smem_bytes() { return gemm2::SMEM_BYTES; }

// stream-K tail plan (kernels.h GemmParams::sk_*): with C pairs and T tiles, T % C != 0 and at
// least one whole wave, the last (T % C) + C tiles are split into equal K ranges (U / C >= nkb
// k blocks per pair: every split tile has one contributor and one finisher); sk_dp_waves whole
// waves go first.  Returns the scratch bytes (0: no stream-K).
int64_t gemm2_sk_plan(int num_tiles, int nkb, int num_sms, int* sk_tiles, int* sk_dp_waves) {
  *sk_tiles = 0;
  *sk_dp_waves = 0;
  const int C = num_sms / 2;
  if (C <= 0 || num_tiles < C || num_tiles % C == 0 || nkb < 2) return 0;
  const int waves = num_tiles / C;  // whole waves
  if (waves > 3) return 0;          // the ragged last wave costs < 1/4 of the run: not worth the fixup
  *sk_tiles = num_tiles % C + C;
  *sk_dp_waves = waves - 1;
  return (int64_t)(*sk_tiles) * 2 * gemm2::BM * (256 + 1) * 4 + (int64_t)(*sk_tiles) * 2 * 4 + 64;
}

// Pair tile width for an M x N problem: the one with the shorter makespan, counted as
// ceil(tiles / pairs) rounds of bn columns (the last N block counted whole), 224 discounted by
// its lower per-tile rate.  Config 3 keeps 256 (25 x 256 vs 28 x 224: 2 % shorter, not enough);
// its 8-rank shard (N = 3584) takes 224 (4 x 256 vs 4 x 224); config 4 keeps 256.
int gemm2_pick_bn(int M, int N, int num_sms, bool allow_224) {
  static const int force = [] {
    const char* e = getenv("FN_GEMM2_BN");  // A/B knob: 256 or 224
    return e != nullptr ? atoi(e) : 0;
  }();
  if (!allow_224) return 256;
  if (force == 256 || force == 224) return force;
  const long long pairs = num_sms / 2 > 0 ? num_sms / 2 : 1;
  const long long mb = (M + 255) / 256;
  auto span = [&](int bn) {
    const long long tiles = mb * ((N + bn - 1) / bn);
    return ((tiles + pairs - 1) / pairs) * bn;
  };
  // a 224-wide tile runs ~2.5 % below a 256-wide one (tools/ab_bn.py: config 3 1484 vs 1478
  // TFLOP/s although its span is 2 % shorter); 160-wide tiles measured 7-17 % slower everywhere
  return span(224) * 40 < span(256) * 39 ? 224 : 256;
}

// host cache of matched schedules (tile_rot == 2), keyed by the tile grid and the pair count;
// any other case gets the empty table (waves = 0: the kernel computes its order itself)
static const PairSchedule* pair_schedule(const GemmParams& p, int pairs) {
  static const PairSchedule none = {};
  if (p.tile_rot != 2) return &none;
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, std::unique_ptr<PairSchedule>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(p.num_m_blocks, p.num_n_blocks, p.group_m, pairs);
  auto it = cache.find(key);
  if (it == cache.end()) {
    // bounded (16 KiB per entry); entries are never freed, so a returned table stays valid while
    // other threads launch — past the bound new shapes take the closed-form rotation instead
    if (cache.size() >= 512) return &none;
    std::unique_ptr<PairSchedule> s(new PairSchedule());
    if (!build_pair_schedule(p, pairs, *s)) s->waves = 0;
    it = cache.emplace(key, std::move(s)).first;
  }
  return it->second.get();
}

template <int MODE, int BN, bool TBL, bool SK = false>
static cudaError_t launch_gemm2_k(const CUtensorMap& ta, const CUtensorMap& tb_half, const GemmParams& p, int pairs,
                                  const void* sched, cudaStream_t stream) {
  using namespace gemm2;
  const void* fptr = (const void*)flashnorm_gemm2_kernel<MODE, BN, TBL, SK>;
  const int smem = smem_bytes(BN);
  if (cudaError_t e = ensure_smem_attr(fptr, smem); e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = nullptr;
  cfg.numAttrs = 0;  // cluster shape comes from __cluster_dims__
  void* args[] = {(void*)&ta, (void*)&tb_half, (void*)&p, const_cast<void*>(sched)};
  return cudaLaunchKernelExC(&cfg, fptr, args);
}

template <int MODE, int BN>
static cudaError_t launch_gemm2_t(const CUtensorMap& ta, const CUtensorMap& tb_half, const GemmParams& p,
                                  int num_sms, cudaStream_t stream) {
  int pairs = num_sms / 2;
  if (p.num_tiles < pairs) pairs = p.num_tiles;
  if (p.sk_tiles > 0) {  // stream-K tail: whole-tile waves in grid-stride order, then the K-split items
    static const PairScheduleNone none_sk = {0};
    if constexpr (MODE == MODE_RMS || MODE == MODE_NONE)
      return launch_gemm2_k<MODE, BN, false, true>(ta, tb_half, p, pairs, &none_sk, stream);
    return cudaErrorInvalidValue;
  }
  // one wave or less: the order cannot matter, and the table-free instance skips the 16 KiB
  // parameter upload (measured ~0.4 us per call on small shapes)
  const PairSchedule* sched = p.num_tiles > pairs ? pair_schedule(p, pairs) : nullptr;
  if (sched != nullptr && sched->waves > 0) return launch_gemm2_k<MODE, BN, true>(ta, tb_half, p, pairs, sched, stream);
  static const PairScheduleNone none = {0};
  return launch_gemm2_k<MODE, BN, false>(ta, tb_half, p, pairs, &none, stream);
}

cudaError_t launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb_half, const GemmParams& p, int mode,
                         int num_sms, cudaStream_t stream) {
  if (p.bn == 224) {  // DyT, GLU and RoPE run 256-wide tiles (the host never asks)
    if (mode == MODE_RMS) return launch_gemm2_t<MODE_RMS, 224>(ta, tb_half, p, num_sms, stream);
    if (mode == MODE_NONE) return launch_gemm2_t<MODE_NONE, 224>(ta, tb_half, p, num_sms, stream);
    return cudaErrorInvalidValue;
  }
  if (mode == MODE_RMS) return launch_gemm2_t<MODE_RMS, 256>(ta, tb_half, p, num_sms, stream);
  if (mode == MODE_DYT) return launch_gemm2_t<MODE_DYT, 256>(ta, tb_half, p, num_sms, stream);
  return launch_gemm2_t<MODE_NONE, 256>(ta, tb_half, p, num_sms, stream);
}

}  // namespace fn
