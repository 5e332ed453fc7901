// gemm_sm100.cu — K3: the prefill FlashNorm GEMM for sm_100a (tcgen05 + TMEM + TMA).
//
//   z[m][j] = RN( fma( sum_k a[m][k] W*t[j][k],  r_m,  c*_j ) )
//   r_m     = rsqrt( ssq_m / K + eps ),  ssq_m = sum_k a[m][k]^2
//
// PAPER.md:17 (Fig 1(c), deferred normalization, scale before bias) and
// PAPER.md:20/154 (Fig 8(c)): the matrix unit runs the contraction while a
// separate "vector unit" computes the RMS.  On B200 the matrix unit is the
// tcgen05 tensor core fed by TMA, and the vector unit is a warp group that
// squares the SAME shared-memory A tiles the MMA is consuming; the epilogue
// applies the deferred scale while the tensor core already accumulates the
// next tile into the other TMEM buffer ("scaling in parallel to the matrix
// unit").
//
// Persistent, warp-specialized, one CTA per SM (384 threads):
//   warp 0      TMA producer (one elected lane): A[128x64] + B[256x64] per stage
//   warp 1      MMA issuer  (one elected lane): 4 x tcgen05.mma 128x256x16 per stage
//   warp 2      TMEM allocator (512 columns = 2 accumulator buffers of 256)
//   warp 3      idle
//   warps 4-7   side group: MODE_RMS  -> per-row sum of squares from the A stage
//                           MODE_DYT  -> in-place tanh(alpha a) of the A stage (prologue)
//                           MODE_NONE -> nothing
//   warps 8-11  epilogue: TMEM -> regs -> *r + c* -> bf16 -> global
#include "common.cuh"
#include "kernels.h"

namespace fn {

namespace gemm {
constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;  // 128 bytes of bf16 = one SW128 atom row
constexpr int STAGES = 4;
constexpr int A_STAGE = BM * BK * 2;  // 16 KiB
constexpr int B_STAGE = BN * BK * 2;  // 32 KiB
constexpr int THREADS = 384;
constexpr int TMEM_COLS = 2 * BN;  // double-buffered fp32 accumulator
constexpr int BAR_BYTES = 1024;
constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * (A_STAGE + B_STAGE) + BAR_BYTES + 6 * BM * 4;
}  // namespace gemm

template <int MODE>
__global__ void __launch_bounds__(gemm::THREADS, 1)
    flashnorm_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                          GemmParams p) {
  using namespace gemm;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* full = bars;                 // TMA landed            [STAGES]
  uint64_t* empty = bars + STAGES;       // stage free            [STAGES]
  uint64_t* ready = bars + 2 * STAGES;   // DyT: A transformed    [STAGES]
  uint64_t* tfull = bars + 3 * STAGES;   // accumulator ready     [2]
  uint64_t* tempty = tfull + 2;          // accumulator drained   [2]
  uint64_t* sfull = tempty + 2;          // ssq ready             [2]
  uint64_t* sempty = sfull + 2;          // ssq consumed          [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + 2);
  float* ssq_buf = reinterpret_cast<float*>(smem + STAGES * (A_STAGE + B_STAGE) + BAR_BYTES);  // [2][BM]
  float* ssq_fence = ssq_buf + 2 * BM;  // [BM] scratch: load-completion fence of the side group
  float* epi_fence = ssq_fence + BM;    // [BM] scratch: load-completion fence of the epilogue
  float* mu_buf = epi_fence + BM;       // [2][BM] LayerNorm (ln_u): row means
  const bool ln = MODE == MODE_RMS && p.ln_u != nullptr;  // exact deferred LayerNorm (reading c29)

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MODE == MODE_RMS ? 2 : 1);  // MMA commit (+ ssq group)
      mbar_init(&ready[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
      mbar_init(&sfull[b], 1);
      mbar_init(&sempty[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_holder, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int num_tiles = p.num_tiles;
  const int nkb = p.num_k_blocks;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int m_blk, n_blk;
        tile_coords(tile, p, m_blk, n_blk);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], A_STAGE + B_STAGE);
          tma_load_2d(sA + stage * A_STAGE, &tmap_a, &full[stage], kb * BK, m_blk * BM, kEvictLast);
          tma_load_2d(sB + stage * B_STAGE, &tmap_b, &full[stage], kb * BK, n_blk * BN, kEvictNormal);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          if (MODE == MODE_DYT) mbar_wait(&ready[stage], phase);  // tanh prologue applied
          else mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = make_sw128_desc(smem_u32(sA + stage * A_STAGE));
          const uint64_t bdesc = make_sw128_desc(smem_u32(sB + stage * B_STAGE));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // +32 bytes per K=16 step inside the 128-byte swizzle atom (encoded >> 4)
            umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[as]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ side group
    const int t = threadIdx.x - 128;  // row of the A tile owned by this thread
    if (MODE == MODE_RMS) {
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        // packed pairs (sm_100 FADD2 / FFMA2, common.cuh): A01 = (s0, s1), A23 = (s2, s3)
        uint64_t A01 = 0, A23 = 0, A0 = 0;
        float a0 = 0.f;  // LayerNorm: shift a[m][0] (see gemm2_sm100.cu)
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait_warp(&full[stage], phase);
          const uint4* row = reinterpret_cast<const uint4*>(sA + stage * A_STAGE + t * 128);
          if (ln) {
            // s0, s1: sum(a - a0);  s2, s3: sum((a - a0)^2)
            if (kb == 0) {
              a0 = bf16lo(row[t & 7].x);
              A0 = f2_pack(a0, a0);
            }
            // columns >= K of the last K block are TMA zero fill: not summed (see gemm2_sm100.cu)
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
              D = f2_sub(f2_bf16x2(v.x), A0); A01 = f2_add(A01, D); A23 = f2_fma(D, D, A23);
              D = f2_sub(f2_bf16x2(v.y), A0); A01 = f2_add(A01, D); A23 = f2_fma(D, D, A23);
              D = f2_sub(f2_bf16x2(v.z), A0); A01 = f2_add(A01, D); A23 = f2_fma(D, D, A23);
              D = f2_sub(f2_bf16x2(v.w), A0); A01 = f2_add(A01, D); A23 = f2_fma(D, D, A23);
            }
            ssq_fence[t] = (f2_lo(A01) + f2_hi(A01)) + (f2_lo(A23) + f2_hi(A23));
            named_bar_sync(1, 128);
            if (t == 0) mbar_arrive(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = row[c ^ (t & 7)];  // swizzled order: conflict-free, sum is order-free
            uint64_t X;
            X = f2_bf16x2(v.x); A01 = f2_fma(X, X, A01);
            X = f2_bf16x2(v.y); A23 = f2_fma(X, X, A23);
            X = f2_bf16x2(v.z); A01 = f2_fma(X, X, A01);
            X = f2_bf16x2(v.w); A23 = f2_fma(X, X, A23);
          }
          // WAR hazard on the A stage: LDS results can still be in flight when a later
          // barrier/arrive issues (neither waits on the LDS scoreboard; under full
          // tensor-core SMEM load they were seen to return after the TMA refill,
          // giving non-deterministic ssq on B200).  The store below cannot issue
          // until every load of this stage has RETURNED (it consumes all four
          // accumulators); bar.sync then drains the stores of all 128 threads, and
          // only then does the group release the stage (2nd arrival on `empty`,
          // next to the MMA commit).  The MMA itself never waits for this group:
          // the RMS runs beside the contraction, not in front of it (Fig 8(c)).
          ssq_fence[t] = (f2_lo(A01) + f2_hi(A01)) + (f2_lo(A23) + f2_hi(A23));
          named_bar_sync(1, 128);
          if (t == 0) mbar_arrive(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait_warp(&sempty[as], aphase ^ 1);
        const float s0 = f2_lo(A01), s1 = f2_hi(A01), s2 = f2_lo(A23), s3 = f2_hi(A23);
        if (ln) {
          const float S1 = s0 + s1, S2 = s2 + s3, invK = 1.0f / (float)p.K;
          ssq_buf[as * BM + t] = fmaxf(S2 - S1 * (S1 * invK), 0.0f);  // K var
          mu_buf[as * BM + t] = fmaf(S1, invK, a0);
        } else {
          ssq_buf[as * BM + t] = (s0 + s1) + (s2 + s3);
        }
        named_bar_sync(1, 128);  // all 128 ssq values written (bar.sync drains the STS)
        if (t == 0) mbar_arrive(&sfull[as]);
      }
    } else if (MODE == MODE_DYT) {
      // alpha*a as one bf16x2 multiply (alpha rounded to bf16; exact for the synthetic
      // alpha = 0.5), then the bf16x2 MUFU tanh: 2 instructions per pair keep the
      // prologue ahead of the tensor core (reading c14).
      const __nv_bfloat162 alpha2 = __floats2bfloat162_rn(p.alpha, p.alpha);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait_warp(&full[stage], phase);
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
          fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
          named_bar_sync(1, 128);
          if (t == 0) mbar_arrive(&ready[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue
    const uint32_t ew = warp - 8;  // == warp % 4: TMEM lane quarter this warp may access
    int local = 0;
    const float invK = 1.0f / static_cast<float>(p.K);
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      int m_blk, n_blk;
      tile_coords(tile, p, m_blk, n_blk);
      const int as = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      float r = 1.0f, mu = 0.f;
      if (MODE == MODE_RMS) {
        mbar_wait_warp(&sfull[as], aphase);
        const float ssq = ssq_buf[as * BM + ew * 32 + lane];
        if (ln) mu = mu_buf[as * BM + ew * 32 + lane];
        epi_fence[ew * 32 + lane] = ssq + mu;  // issues only once the LDS above have returned
        named_bar_sync(2, 128);           // ... and bar.sync drains it: ssq_buf[as] is free
        if (ew == 0 && lane == 0) mbar_arrive(&sempty[as]);
        r = rsqrtf(fmaf(ssq, invK, p.eps));
      }
      mbar_wait_warp(&tfull[as], aphase);
      tc_fence_after();
      const int row = m_blk * BM + ew * 32 + lane;
      const uint32_t taddr = tmem_base + ((ew * 32u) << 16) + as * BN;
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
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[as]);
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
        tmem_ld_32x32b_x32(taddr + j * 32, v);
        tmem_wait_ld();
        float cb[32];
        if (p.cstar != nullptr) {
          const float4* c4 = reinterpret_cast<const float4*>(p.cstar + n_base + j * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (n_base + j * 32 + q * 4 < p.N) cv = __ldg(c4 + q);
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
        if (row < p.M) {
          if (p.ndst == 0) {
            uint4* dst = reinterpret_cast<uint4*>(zrow + j * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (n_base + j * 32 + q * 8 < p.N)
                dst[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
            }
          } else {
            // fused gather (see gemm2_sm100.cu): every destination gets the row segment
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
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

int gemm_smem_bytes() { return gemm::SMEM_BYTES; }

cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int mode,
                        int num_sms, cudaStream_t stream) {
  using namespace gemm;
  const void* fptr = mode == MODE_RMS ? (const void*)flashnorm_gemm_kernel<MODE_RMS>
                     : mode == MODE_DYT ? (const void*)flashnorm_gemm_kernel<MODE_DYT>
                                        : (const void*)flashnorm_gemm_kernel<MODE_NONE>;
  if (cudaError_t e = ensure_smem_attr(fptr, SMEM_BYTES); e != cudaSuccess) return e;
  const int grid = p.num_tiles < num_sms ? p.num_tiles : num_sms;
  void* args[] = {(void*)&ta, (void*)&tb, (void*)&p};
  return cudaLaunchKernel(fptr, dim3(grid), dim3(THREADS), args, SMEM_BYTES, stream);
}

}  // namespace fn
