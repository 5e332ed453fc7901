// gemv_wide.cu — K4w: batched-decode FlashNorm linear for 17 <= M <= 128 tokens on tcgen05.
//
//   z[m][j] = RN( fma( sum_k a[m][k] W*t[j][k], r_m, c*_j ) ),  r_m = rsqrt(ssq_m/K + eps)
//   (Fig 1(c); the RMS reduced beside the contraction, Fig 8(c))
//
// Past 16 tokens the library used to fall to the GEMM kernels, whose 128 x 256 tiles give config 2's
// N = 6144 only 24 CTAs: ~30 us per call (0.26 of HBM) for any M in 17..128, three times the
// 16-token decode (tools/bench_midm.py).  This kernel is K4's swap-AB contraction (gemv_tc.cu) with
// the token count as the MMA N:
//
//   D[128 W* rows x T tokens] (TMEM, fp32) += W*[128 x 16k] . a^T[16k x T],   T = 32 / 64 / 128 >= M
//
// tcgen05 takes 45.5 / 48 / 64 cycles per 16-k step for N = 32 / 64 / 128 against 45.5 for N = 16
// (tools/micro/mma_rate.cu), so up to 64 tokens stream W* at the 16-token rate.  Work split as K4:
// tile = 128 W* rows, its K range split over the S CTAs of one thread-block cluster, the peers'
// fp32 partials (and partial ssq) pushed into the leader's shared memory with one bulk copy each and
// summed in fixed rank order (deterministic).  Per CTA (192 threads): warp 0 TMA producer (W* 16 KiB
// + tokens T x 128 B per stage), warp 1 TMEM allocator + MMA issuer, warps 2-5 the per-token
// partial ssq (RMS, from global after the dependency wait, off the ring) and then the epilogue, 16
// tokens at a time.  Modes: rmsnorm / layernorm (pre-centered input) and none (optionally with a
// per-row output scale), RoPE on the Q/K columns (rmsnorm, NEXT-2) with or without QK-norm (NEXT-4,
// h | 128); DyT runs as the K8 tanh pre-pass + none; GLU keeps its kernels.  W* streams before the PDL dependency wait (a constant
// operand, as in K4: include/flashnorm.h states the precondition); tokens are loaded after it.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

namespace fn {

namespace dw {
constexpr int ROWS = 128;              // W* rows per tile (MMA M)
constexpr int BK = 64;                 // k per stage (one SW128 atom row of bf16)
constexpr int THREADS = 192;
constexpr int W_STAGE = ROWS * BK * 2;  // 16 KiB
constexpr int MAX_S = 8;               // K splits per tile (portable cluster size)
constexpr int MAX_STAGES = 12;
constexpr int CTRL = 4096;             // barriers + ssq scratch after the ring (bytes)
constexpr size_t SMEM_MAX = 232448;
}  // namespace dw

template <int MODE, int T>
__global__ void __launch_bounds__(dw::THREADS, 1)
    flashnorm_gemv_wide_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_a,
                               const float* __restrict__ cstar, __nv_bfloat16* __restrict__ z, int M, int K, int N,
                               float eps, int S, int stages, int l2pf, const __nv_bfloat16* __restrict__ aptr,
                               const float* __restrict__ row_scale, const RopeParams rope) {
  using namespace dw;
  constexpr int T_STAGE = T * BK * 2;      // token bytes per stage
  constexpr int RECV = ROWS * T + T;       // floats per peer slot: partial D + partial ssq
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;                                  // [stages][128 x 64] SW128
  uint8_t* sT = sW + (size_t)stages * W_STAGE;         // [stages][T x 64] SW128
  uint64_t* bars = reinterpret_cast<uint64_t*>(sT + (size_t)stages * T_STAGE);
  uint64_t* full = bars;                 // [stages] W* + tokens landed
  uint64_t* empty = bars + stages;       // [stages] stage consumed (MMA commit)
  uint64_t* tfull = bars + 2 * stages;   // accumulator complete
  uint64_t* recv_bar = tfull + 1;        // leader: the peers' partials landed
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(recv_bar + 1);
  float* ssq_own = reinterpret_cast<float*>(tmem_holder + 4);  // [T] this CTA's partial ssq per token
  float* recv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + CTRL);  // [S-1][RECV]
  float* part = reinterpret_cast<float*>(smem);  // a peer's staged partial (the ring is free after the MMAs)

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int rank = (int)(blockIdx.x % (unsigned)S);  // K-split rank = cluster rank (one tile per cluster)
  const int tile = (int)(blockIdx.x / (unsigned)S);
  const int n0 = tile * ROWS;
  const int nkb = (K + BK - 1) / BK;
  const int kb0 = (int)(((long long)rank * nkb) / S);
  const int kb1 = (int)(((long long)(rank + 1) * nkb) / S);
  const int my_kb = kb1 - kb0;  // >= 1 (S <= nkb)
  const bool push = S > 1;

  pdl_launch_dependents();  // the next call's CTAs may queue for free SMs right away
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_w);
    prefetch_tmap(&tmap_a);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);  // MMA commit
    }
    mbar_init(tfull, 1);
    mbar_init(recv_bar, 1);  // the leader's expect_tx + each peer's bulk copy (complete_tx)
    fence_mbar_init();
    if (push && rank == 0) mbar_arrive_expect_tx(recv_bar, (uint32_t)((S - 1) * RECV * 4));
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, T);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (push) cluster_arrive_relaxed();  // barrier inits published; the matching wait precedes any remote access

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const int pre = my_kb < stages ? my_kb : stages;
      for (int i = 0; i < pre; ++i) {  // W* is constant: its first stages stream before the wait
        mbar_arrive_expect_tx(&full[i], (uint32_t)(W_STAGE + T_STAGE));
        tma_load_2d(sW + (size_t)i * W_STAGE, &tmap_w, &full[i], (kb0 + i) * BK, n0, kEvictFirst);
      }
      for (int i = pre; i < my_kb && i < pre + l2pf; ++i) tma_prefetch_l2_2d(&tmap_w, (kb0 + i) * BK, n0);
      pdl_wait_prior_grid();  // tokens may be the previous kernel's output
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sT + (size_t)i * T_STAGE, &tmap_a, &full[i], (kb0 + i) * BK, 0, kEvictLast);
      int stage = pre == stages ? 0 : pre;
      uint32_t phase = pre == stages ? 1u : 0u;
      for (int i = pre; i < my_kb; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], (uint32_t)(W_STAGE + T_STAGE));
        tma_load_2d(sW + (size_t)stage * W_STAGE, &tmap_w, &full[stage], (kb0 + i) * BK, n0, kEvictFirst);
        tma_load_2d(sT + (size_t)stage * T_STAGE, &tmap_a, &full[stage], (kb0 + i) * BK, 0, kEvictLast);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(ROWS, T);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < my_kb; ++i) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t adesc = make_sw128_desc(smem_u32(sW + (size_t)stage * W_STAGE));
        const uint64_t bdesc = make_sw128_desc(smem_u32(sT + (size_t)stage * T_STAGE));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) umma_bf16(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, (i | k) != 0);
        umma_commit(&empty[stage]);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
      umma_commit(tfull);
    }
  } else {
    // ------------------------------------------------------------ warps 2-5: ssq, then the epilogue
    const int t = (int)threadIdx.x - 64;  // 0..127
    pdl_wait_prior_grid();  // tokens (RMS) are read below; z is written below
    if (MODE == MODE_RMS) {
      // per-token partial ssq over this CTA's K range, straight from global (L2), 16 tokens at a time,
      // beside the contraction and off the W* ring (as K4).  (Reading the SMEM token stages instead,
      // each warp releasing a stage after its reads, measured 2-5 % faster at 64-128 tokens but gave
      // run-to-run differences in the ssq of the highest token rows at 128 tokens: not adopted.)
      float* ssq_red = ssq_own + T;  // [4 warps][T]
      const int k0 = kb0 * BK;
      const int nch = (min(kb1 * BK, K) - k0) / 8;  // 16-byte chunks (K % 8 == 0)
      for (int mc = 0; mc * 16 < T; ++mc) {
        float sm[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) sm[m] = 0.f;
        if (mc * 16 < M) {
          for (int c = t; c < nch; c += 128) {
            uint4 v[16];
#pragma unroll
            for (int m = 0; m < 16; ++m) {
              const int tok = mc * 16 + m;
              v[m] = tok < M ? __ldg(reinterpret_cast<const uint4*>(aptr + (size_t)tok * K + k0) + c)
                             : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int m = 0; m < 16; ++m) {
              float x, s0 = 0.f, s1 = 0.f;
              x = bf16lo(v[m].x); s0 = fmaf(x, x, s0);
              x = bf16hi(v[m].x); s1 = fmaf(x, x, s1);
              x = bf16lo(v[m].y); s0 = fmaf(x, x, s0);
              x = bf16hi(v[m].y); s1 = fmaf(x, x, s1);
              x = bf16lo(v[m].z); s0 = fmaf(x, x, s0);
              x = bf16hi(v[m].z); s1 = fmaf(x, x, s1);
              x = bf16lo(v[m].w); s0 = fmaf(x, x, s0);
              x = bf16hi(v[m].w); s1 = fmaf(x, x, s1);
              sm[m] += s0 + s1;
            }
          }
        }
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          float x = sm[m];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
          if (lane == 0) ssq_red[(warp - 2) * T + mc * 16 + m] = x;
        }
      }
      named_bar_sync(1, 128);
      if (t < T) ssq_own[t] = (ssq_red[t] + ssq_red[T + t]) + (ssq_red[2 * T + t] + ssq_red[3 * T + t]);
      named_bar_sync(1, 128);  // ssq_own complete
    }
    const uint32_t q4 = warp & 3u;  // TMEM lane quarter this warp may access
    const int row = (int)(q4 * 32 + lane);
    mbar_wait_warp(tfull, 0);
    tc_fence_after();
    if (push && rank != 0) {
      // peer: TMEM -> its own (now free) ring SMEM, 16 tokens at a time, + the partial ssq; then ONE
      // bulk copy into its slot of the leader's receive buffer, completing on the leader's recv_bar
      for (int c = 0; c < T / 16; ++c) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_base + ((q4 * 32u) << 16) + c * 16, v);
        tmem_wait_ld();
        float4* dst = reinterpret_cast<float4*>(part + row * T + c * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                               __uint_as_float(v[4 * q + 3]));
      }
      if (t < T) part[ROWS * T + t] = MODE == MODE_RMS ? ssq_own[t] : 0.f;
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the bulk-copy engine
      named_bar_sync(1, 128);
      if (warp == 2) {
        cluster_wait();  // the leader's recv_bar is initialised (arrive at kernel start)
        if (lane == 0) {
          dsmem_bulk_copy(mapa_shared(recv + (size_t)(rank - 1) * RECV, 0u), part, (uint32_t)(RECV * 4),
                          mapa_shared(recv_bar, 0u));
          bulk_commit_group();
          bulk_wait_read();  // the source (this CTA's SMEM) stays valid until read
        }
        __syncwarp();
      }
    } else {
      if (push) mbar_wait_warp_cluster(recv_bar, 0);  // every peer's partial landed
      const float invK = 1.0f / (float)K;
      const int n = n0 + row;
      const float cb = (n < N && cstar != nullptr) ? __ldg(cstar + n) : 0.0f;
      for (int c = 0; c < T / 16 && c * 16 < M; ++c) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_base + ((q4 * 32u) << 16) + c * 16, v);
        tmem_wait_ld();
        float acc[16], ssq[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          acc[m] = __uint_as_float(v[m]);
          ssq[m] = MODE == MODE_RMS ? ssq_own[c * 16 + m] : 0.f;
        }
        for (int r = 1; r < S; ++r) {  // fixed rank order
          const float* sl = recv + (size_t)(r - 1) * RECV;
          const float4* src = reinterpret_cast<const float4*>(sl + row * T + c * 16);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 p = src[q];
            acc[4 * q] += p.x; acc[4 * q + 1] += p.y; acc[4 * q + 2] += p.z; acc[4 * q + 3] += p.w;
          }
          if (MODE == MODE_RMS)
#pragma unroll
            for (int m = 0; m < 16; ++m) ssq[m] += sl[ROWS * T + c * 16 + m];
        }
        // RoPE on the Q/K columns [0, rope.n) (NEXT-2, Fig 5(b), as K4): the pair partner of W* row n
        // is row n ^ 1, held by lane ^ 1; cos/sin scaled once per token by r * qk
        const bool rope_row = MODE == MODE_RMS && rope.pos != nullptr && n0 < rope.n;  // warp-uniform per tile
        float pv[16];
        if (rope_row) {
#pragma unroll
          for (int m = 0; m < 16; ++m) pv[m] = __shfl_xor_sync(0xffffffffu, acc[m], 1);
        }
        // QK-norm (NEXT-4, Figs 6(b)/7(b), as K4): per Q/K head and token s_b = rsqrt(MS(head) +
        // eps_qk MSe(a)) replaces r (s_a cancels); the head's rows (h | 128) are h / 32 warps of this
        // tile: warp shuffles, then a [4 warps][16 tokens] exchange in the (free) ring
        float sb[16];
        float g_own = 1.0f, g_pair = 1.0f;
        const bool qkn = MODE == MODE_RMS && rope_row && rope.g_q != nullptr;  // warp-uniform
        if (qkn) {
          float* red = reinterpret_cast<float*>(smem);
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            float q = acc[m] * acc[m];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
            if (lane == 0) red[q4 * 16 + m] = q;
          }
          named_bar_sync(3, 128);
          const int wph = rope.h / 32;  // warps per head (h = 32, 64 or 128)
          const int w0 = (int)(q4 / (uint32_t)wph) * wph;
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            float ss = 0.f;
            for (int w = 0; w < wph; ++w) ss += red[(w0 + w) * 16 + m];
            const float rr = rsqrtf(fmaf(ssq[m], invK, eps));
            sb[m] = rsqrtf(fmaf(rope.eps_qk, 1.0f / (rr * rr), ss / (float)rope.h));
          }
          named_bar_sync(3, 128);  // red is rewritten by the next chunk
          if (n < rope.n) {
            const float* gsrc = n < rope.n_q ? rope.g_q : rope.g_k;
            g_own = __ldg(gsrc + n % rope.h);
            g_pair = __ldg(gsrc + (n ^ 1) % rope.h);
          }
        }
        if (n < N) {
          const bool rot = rope_row && n < rope.n;
          const int hh = rope.h >> 1;
          const int ri = rot ? (n % rope.h) >> 1 : 0;
          const float sgn = (n & 1) ? 1.0f : -1.0f;  // y0 = x0 c - x1 s, y1 = x1 c + x0 s
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            const int tok = c * 16 + m;
            if (tok < M) {
              // rmsnorm / layernorm: the deferred 1/RMS; none: 1 or the given per-row scale (the
              // down projection of a GLU / ReLU FFN, flashnorm_linear_scaled)
              const float rr = MODE == MODE_RMS ? rsqrtf(fmaf(ssq[m], invK, eps))
                                                : (row_scale != nullptr ? __ldg(row_scale + tok) : 1.0f);
              if (rot) {
                const int pos = __ldg(rope.pos + tok);
                const float rq = (qkn ? sb[m] : rr) * rope.qk;
                const float cc = __ldg(rope.cos_tab + (size_t)pos * hh + ri) * rq * g_own;
                const float sn = __ldg(rope.sin_tab + (size_t)pos * hh + ri) * rq * g_pair;
                z[(size_t)tok * N + n] = __float2bfloat16_rn(fmaf(acc[m], cc, sgn * pv[m] * sn));
              } else {
                z[(size_t)tok * N + n] = __float2bfloat16_rn(fmaf(acc[m], rr, cb));
              }
            }
          }
        }
      }
    }
  }
  if (push) {
    if (rank == 0 || warp != 2) cluster_wait();  // pairs with the arrive at the start (peer warp 2 waited above)
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, T);
  }
}

namespace {
template <int MODE, int T>
const void* dwk() {
  return (const void*)flashnorm_gemv_wide_kernel<MODE, T>;
}
const void* dw_fptr(int mode, int T) {
  if (mode == MODE_RMS) return T == 32 ? dwk<MODE_RMS, 32>() : T == 64 ? dwk<MODE_RMS, 64>() : dwk<MODE_RMS, 128>();
  return T == 32 ? dwk<MODE_NONE, 32>() : T == 64 ? dwk<MODE_NONE, 64>() : dwk<MODE_NONE, 128>();
}
int dw_tokens(int M) { return M <= 32 ? 32 : M <= 64 ? 64 : 128; }
size_t dw_recv_bytes(int T, int S) { return S > 1 ? (size_t)(S - 1) * (dw::ROWS * T + T) * 4 : 0; }
int dw_stages(int T, int S) {
  const size_t fixed = 1024 + dw::CTRL + dw_recv_bytes(T, S) + 256;
  const size_t per = dw::W_STAGE + (size_t)T * dw::BK * 2;
  if (dw::SMEM_MAX < fixed + 2 * per) return 0;
  return (int)std::min<size_t>(dw::MAX_STAGES, (dw::SMEM_MAX - fixed) / per);
}
size_t dw_smem(int T, int S, int stages) {
  return 1024 + (size_t)stages * (dw::W_STAGE + (size_t)T * dw::BK * 2) + dw::CTRL + dw_recv_bytes(T, S);
}
struct DwPlan {
  int T = 0, S = 0, stages = 0;
};
// the largest K split whose clusters (one tile, S CTAs) are all co-resident, tiles x S <= #SMs
DwPlan dw_plan(int mode, int M, int K, int N, int num_sms) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int>, DwPlan> cache;
  const int T = dw_tokens(M);
  const auto key = std::make_tuple(mode, T, K, N, num_sms);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  DwPlan best;
  const int tiles = (N + dw::ROWS - 1) / dw::ROWS;
  const int nkb = (K + dw::BK - 1) / dw::BK;
  if (tiles <= num_sms) {
    const void* f = dw_fptr(mode, T);
    for (int S = std::min(std::min(dw::MAX_S, num_sms / tiles), nkb); S >= 1; --S) {
      const int st = dw_stages(T, S);
      if (st < 2) continue;
      const size_t smem = dw_smem(T, S, st);
      if (ensure_smem_attr(f, (int)smem) != cudaSuccess) continue;
      if (S == 1) {
        best = DwPlan{T, 1, st};
        break;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(tiles * S);
      cfg.blockDim = dim3(dw::THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = S;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, f, &cfg) == cudaSuccess && n >= tiles) {
        best = DwPlan{T, S, st};
        break;
      }
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, best);
  return best;
}
}  // namespace

int gemv_wide_tokens(int M) { return dw_tokens(M); }

bool gemv_wide_supported(int mode, int M, int K, int N, int num_sms) {
  if (M <= 16 || M > 128 || (mode != MODE_RMS && mode != MODE_NONE) || K % 8 != 0) return false;
  return dw_plan(mode, M, K, N, num_sms).S > 0;
}

cudaError_t launch_gemv_wide(const CUtensorMap& tw, const CUtensorMap& ta, const float* cstar, __nv_bfloat16* z,
                             int M, int K, int N, float eps, int mode, int num_sms, cudaStream_t stream,
                             const __nv_bfloat16* aptr, const float* row_scale, RopeParams rope) {
  const DwPlan p = dw_plan(mode, M, K, N, num_sms);
  if (p.S <= 0) return cudaErrorInvalidConfiguration;
  const void* fptr = dw_fptr(mode, p.T);
  const size_t smem = dw_smem(p.T, p.S, p.stages);
  if (cudaError_t e = ensure_smem_attr(fptr, (int)smem); e != cudaSuccess) return e;
  const int tiles = (N + dw::ROWS - 1) / dw::ROWS;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles * p.S);
  cfg.blockDim = dim3(dw::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = p.S;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  const int l2pf = 12;  // W* stages per CTA prefetched to L2 before the dependency wait (as K4)
  int S = p.S, stages = p.stages;
  void* args[] = {(void*)&tw, (void*)&ta, (void*)&cstar, (void*)&z, (void*)&M, (void*)&K, (void*)&N,
                  (void*)&eps, (void*)&S, (void*)&stages, (void*)&l2pf, (void*)&aptr, (void*)&row_scale,
                  (void*)&rope};
  return cudaLaunchKernelExC(&cfg, fptr, args);
}

}  // namespace fn
