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

#include <atomic>

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

// predicated 16-byte streaming load; returns zeros when !pred (no branch)
FN_DEVICE uint4 ldg_stream_pred(const void* p, bool pred) {
  uint4 r;
  asm volatile(
      "{\n\t.reg .pred q;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0; mov.b32 %1, 0; mov.b32 %2, 0; mov.b32 %3, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "r"((uint32_t)pred));
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

static size_t gemv_regs_smem_bytes(int M, int K) {
  const size_t a_bytes = ((size_t)M * (K + 32) * 2 + 15) / 16 * 16;
  return a_bytes + (size_t)gv::SEG * gv::WARPS * 128 * 4 + 16 * 4;
}

template <int MODE>
__global__ void __launch_bounds__(gv::THREADS, 1)
    flashnorm_gemv_regs_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ Wt,
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

  // Per-warp load stream of the current segment: groups of CH chunks, one group
  // never spans two tiles, so group -> (tile, qb) is tracked incrementally
  // (no integer division on the load path) and every load is a predicated
  // 16-byte LDG (no branches between the loads in flight).
  const int nqb = (cpw + CH - 1) / CH;  // chunk-groups per tile for this warp
  auto load_group = [&](int tile, int qb, bool live, uint4 (&w)[CH]) {
    const int n = (t0 + tile) * 8 + g;
    const bool nvalid = live && n >= r0 && n < r1;
    const __nv_bfloat16* rowp = Wt + (size_t)(nvalid ? n : r0) * K;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int q = qb * CH + i;
      const int k = (warp + WARPS * q) * 32 + kq * 8;
      w[i] = ldg_stream_pred(rowp + (k < K ? k : 0), nvalid && q < cpw && k < K);
    }
  };

  uint4 wb0[CH], wb1[CH];
  const int seg0_tiles = ntiles < SEG ? ntiles : SEG;
  load_group(0, 0, seg0_tiles > 0 && nqb > 0, wb0);  // the W* stream starts before the RMS (Fig 8(c))

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
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  auto compute_group = [&](int tile, int qb, const uint4 (&w)[CH]) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int q = qb * CH + i;
      if (q < cpw) {  // warp-uniform: mma.sync needs the converged warp
        const int k = (warp + WARPS * q) * 32 + kq * 8;
        uint4 ra = make_uint4(0u, 0u, 0u, 0u), rb = make_uint4(0u, 0u, 0u, 0u);
        if (row_lo && k < K) ra = *reinterpret_cast<const uint4*>(a_s + (size_t)g * lda + k);
        if (row_hi && k < K) rb = *reinterpret_cast<const uint4*>(a_s + (size_t)(g + 8) * lda + k);
        mma_bf16_16816(acc, ra.x, rb.x, ra.y, rb.y, w[i].x, w[i].y);
        mma_bf16_16816(acc, ra.z, rb.z, ra.w, rb.w, w[i].z, w[i].w);
      }
    }
    if (qb == nqb - 1) {  // last group of this warp for the tile: park the partial tile
      *reinterpret_cast<float4*>(part + ((size_t)(tile % SEG) * WARPS + warp) * 128 + lane * 4) =
          make_float4(acc[0], acc[1], acc[2], acc[3]);
      acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
    }
  };

  for (int seg_t0 = 0; seg_t0 < ntiles; seg_t0 += SEG) {
    const int seg_tiles = (ntiles - seg_t0) < SEG ? (ntiles - seg_t0) : SEG;
    const int ngroups = seg_tiles * nqb;
    if (seg_t0 > 0) load_group(seg_t0, 0, nqb > 0, wb0);
    // (tile, qb) of the group held in each buffer / to be loaded next
    int ct = seg_t0, cq = 0;                     // group in wb0
    int lt = seg_t0, lq = 0;                     // last loaded group
    auto next = [&](int& t, int& q) { if (++q == nqb) { q = 0; ++t; } };
    for (int gi = 0; gi < ngroups; gi += 2) {
      next(lt, lq);
      load_group(lt, lq, gi + 1 < ngroups, wb1);
      compute_group(ct, cq, wb0);
      next(ct, cq);
      next(lt, lq);
      load_group(lt, lq, gi + 2 < ngroups, wb0);
      if (gi + 1 < ngroups) compute_group(ct, cq, wb1);
      next(ct, cq);
    }
    if (nqb == 0) {  // warp without K chunks (K < 16*32): contributes zero partials
      for (int tile = seg_t0; tile < seg_t0 + seg_tiles; ++tile)
        *reinterpret_cast<float4*>(part + ((size_t)(tile % SEG) * WARPS + warp) * 128 + lane * 4) =
            make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    // fixed-order reduction over the 16 warps, deferred scale, bias, bf16 store
    for (int e = tid; e < seg_tiles * 128; e += THREADS) {
      const int tile = seg_t0 + (e >> 7), slot = e & 127;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) s += part[((size_t)(tile % SEG) * WARPS + w) * 128 + slot];
      const int ln = slot >> 2, i = slot & 3;
      const int row = (ln >> 2) + (i >= 2 ? 8 : 0);
      const int col = (ln & 3) * 2 + (i & 1);
      const int n = (t0 + tile) * 8 + col;
      if (row < M && n >= r0 && n < r1) {
        const float r = MODE == MODE_RMS ? r_s[row] : 1.0f;
        const float cb = cstar != nullptr ? __ldg(cstar + n) : 0.0f;
        z[(size_t)row * N + n] = __float2bfloat16_rn(fmaf(s, r, cb));
      }
    }
    __syncthreads();
  }
}

static cudaError_t launch_gemv_regs(const __nv_bfloat16* a, const __nv_bfloat16* Wt, const float* cstar, __nv_bfloat16* z,
                        int M, int K, int N, float eps, float alpha, int mode, int num_sms, cudaStream_t stream) {
  const size_t smem = gemv_regs_smem_bytes(M, K);
  const void* fptr = mode == MODE_RMS ? (const void*)flashnorm_gemv_regs_kernel<MODE_RMS>
                     : mode == MODE_DYT ? (const void*)flashnorm_gemv_regs_kernel<MODE_DYT>
                                        : (const void*)flashnorm_gemv_regs_kernel<MODE_NONE>;
  if (smem > 48 * 1024)
    if (cudaError_t e = ensure_smem_attr(fptr, (int)smem); e != cudaSuccess) return e;
  // one CTA per SM, but never fewer than ~8 output rows per CTA
  int grid = (N + 7) / 8;
  if (grid > num_sms) grid = num_sms;
  void* args[] = {(void*)&a, (void*)&Wt, (void*)&cstar, (void*)&z, (void*)&M, (void*)&K, (void*)&N, (void*)&eps,
                  (void*)&alpha};
  return cudaLaunchKernel(fptr, dim3(grid), dim3(gv::THREADS), args, smem, stream);
}

// ============================================================================
// Main decode kernel: W* streamed by the bulk-copy engine (cp.async.bulk) into
// a shared-memory ring, tokens held in registers, tiles scheduled dynamically.
//
//  * warp 15 is the producer (one lane): it owns the ring and the tile schedule;
//    warps 0..14 compute.  (16 warps keep 4 per SM sub-partition, i.e. 128
//    registers per thread for the token fragments.)
//  * work unit = one 8-row mma tile of W*t, full K (64 KiB at K = 4096), copied as
//    8 row copies into padded smem rows (conflict-free B-fragment loads).  The
//    first S tiles of every CTA are static (b, b+G, ...), the rest are taken from
//    a global atomic counter, so SMs that start late or stream slower take fewer
//    tiles (the kernel ends within ~1 tile of perfect balance).  The counter
//    lives in one of gt::SLOTS launch slots; the CTA whose fetch is the launch's
//    last (the total number of fetches is known) stores 0 back — no end-of-kernel
//    atomics or fences, and graph replays find it reset.
//  * compute warp w owns a fixed K range; its A fragments (the M <= 16 tokens,
//    DyT-transformed once) live in registers, and its per-row partial ssq comes
//    from the same registers while the first tiles stream in — the RMS no longer
//    sits in front of the matrix unit (Fig 8(c)).
//  * per tile every warp parks its 16x8 partial in smem and releases the stage;
//    warp (seq % 15) reduces the tile in a fixed order and applies * r + c*,
//    overlapped with the stream.
// ============================================================================
#ifdef FN_GEMV_TRACE  // tools/micro/gemv_trace.cu: per-CTA timeline (globaltimer, ns)
__device__ unsigned long long g_gemv_trace[2][148 * 8];  // [launch slot parity]
FN_DEVICE unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_gemv_ttrace[2][16][6];  // block 0: per seq event times
#define FN_TTRACE(seq, ev) \
  if (blockIdx.x == 0 && (seq) < 16) g_gemv_ttrace[slot_id & 1][(seq)][(ev)] = gtime()
#define FN_TRACE(slot) \
  if ((threadIdx.x & 31) == 0 && (slot != 1 || threadIdx.x == 0) && blockIdx.x < 148) \
    g_gemv_trace[slot_id & 1][blockIdx.x * 8 + (slot)] = gtime()
#else
#define FN_TRACE(slot)
#define FN_TTRACE(seq, ev)
#endif

namespace gt {
constexpr int CWARPS = 15;                 // compute warps
constexpr int PWARP = CWARPS;              // producer warp index
constexpr int THREADS = (CWARPS + 1) * 32;
constexpr int CPW_MAX = 9;                 // K <= 15 * 9 * 32 = 4320
constexpr int K_MAX = 4096;                // K handled by this kernel (stage = 8 rows x K)
constexpr int SEG = 4;                     // partial-tile slots
constexpr int RPU = 8;                     // W* rows per work unit / ring stage (mma n = 8: rows >= RPU are zero)
constexpr int MAX_STAGES = 4;              // ring depth: as many 8-row stages as fit (3 at K = 4096)
constexpr int SLOTS = 64;                  // launch slots of the dynamic tile counter
// Dynamic SMEM budget of the one CTA per SM (227 KiB opt-in).  The ring is sized to fill
// it: W* prefetched before griddepcontrol.wait keeps HBM busy across the dependency on
// the previous kernel of the stream (PDL), which a 2-stage ring could not.
constexpr size_t SMEM_BUDGET = 232448;
}  // namespace gt

__device__ unsigned int g_gemv_sched[gt::SLOTS];  // [slot] = next dynamic tile (0 between launches)

static size_t gemv_fixed_smem_bytes() {
  return (size_t)gt::SEG * gt::CWARPS * 128 * 4 + 16 * 16 * 4 + gt::CWARPS * 32 * 4 + 16 +
         (2 * gt::MAX_STAGES + 2 * gt::SEG) * 8;
}
static int gemv_stages(int K) {
  const size_t per = (size_t)gt::RPU * (K * 2 + 64);
  size_t n = (gt::SMEM_BUDGET - gemv_fixed_smem_bytes()) / per;
  if (n > (size_t)gt::MAX_STAGES) n = gt::MAX_STAGES;
  return n < 2 ? 2 : (int)n;
}
static size_t gemv_tma_smem_bytes(int K) {
  return (size_t)gemv_stages(K) * gt::RPU * (K * 2 + 64) + gemv_fixed_smem_bytes();
}

template <int MODE, bool M_HI>
__global__ void __launch_bounds__(gt::THREADS, 1)
    flashnorm_gemv_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ Wt,
                          const float* __restrict__ cstar, __nv_bfloat16* __restrict__ z, int M, int K, int N,
                          float eps, float alpha, int slot_id, int STAGES) {
  using namespace gt;
  extern __shared__ __align__(128) uint8_t smem[];
  const int ldb = K * 2 + 64;  // padded smem row stride (bytes)
  uint8_t* ring = smem;
  float* part = reinterpret_cast<float*>(smem + (size_t)STAGES * RPU * ldb);  // [SEG][CWARPS][128]
  float* ssq_part = part + SEG * CWARPS * 128;                               // [16 warps][16 rows]
  float* part_fence = ssq_part + 16 * 16;                                    // [CWARPS*32] scratch
  int* stage_tile = reinterpret_cast<int*>(part_fence + CWARPS * 32);        // [MAX_STAGES]
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_tile + 4);              // [STAGES]
  uint64_t* empty = full + MAX_STAGES;                                       // [STAGES]
  uint64_t* part_full = empty + MAX_STAGES;                                  // [SEG]
  uint64_t* part_empty = part_full + SEG;                                    // [SEG]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ntiles = (N + RPU - 1) / RPU;  // work units of RPU rows
  const int G = gridDim.x;

  FN_TRACE(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CWARPS);
    }
    for (int s = 0; s < SEG; ++s) {
      mbar_init(&part_full[s], CWARPS);
      mbar_init(&part_empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == PWARP) {
    // -------------------------------------------------------------- producer
    pdl_launch_dependents();  // let the next call's CTAs queue for this SM right away
    if (elect_one()) {
      unsigned int* sched = &g_gemv_sched[slot_id];
      // fetches this launch makes: every dynamic tile once, plus one failing fetch by each
      // CTA whose static tiles are all valid; the fetch returning total-1 is the last one
      const int n_dyn_tiles = ntiles > STAGES * G ? ntiles - STAGES * G : 0;
      int n_dyn_ctas = ntiles - (STAGES - 1) * G;
      n_dyn_ctas = n_dyn_ctas < 0 ? 0 : (n_dyn_ctas > G ? G : n_dyn_ctas);
      const unsigned total_fetches = (unsigned)(n_dyn_tiles + n_dyn_ctas);
      int stage = 0;
      uint32_t phase = 0;
      for (int k = 0;; ++k) {
        int t;
        if (k < STAGES) t = blockIdx.x + k * G;                                    // static prologue
        else {                                                                      // dynamic
          const unsigned f = atomicAdd(sched, 1u);
          if (f == total_fetches - 1u) *sched = 0u;  // last fetch of this launch: reset the slot
          t = STAGES * G + (int)f;
        }
        if (k >= STAGES) mbar_wait(&empty[stage], phase ^ 1);
        if (t >= ntiles) {  // no more work: an empty stage carrying tile -1 ends the consumers
#ifdef FN_GEMV_TRACE
          g_gemv_trace[slot_id & 1][blockIdx.x * 8 + 6] = gtime();
          g_gemv_trace[slot_id & 1][blockIdx.x * 8 + 7] = (unsigned long long)k;
#endif
          stage_tile[stage] = -1;
          mbar_arrive(&full[stage]);
          break;
        }
        stage_tile[stage] = t;
        FN_TTRACE(k, 0);
        const int n0 = t * RPU;
        const int hi = n0 + RPU < N ? n0 + RPU : N;
        mbar_arrive_expect_tx(&full[stage], (uint32_t)(hi - n0) * K * 2);
        for (int n = n0; n < hi; ++n)
          bulk_g2s(ring + ((size_t)stage * RPU + (n - n0)) * ldb, Wt + (size_t)n * K, K * 2, &full[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    // W* is a constant operand and streamed above before any dependency wait; the
    // producer never touches a or z.
  } else {
    // -------------------------------------------------------------- compute warps
    // a (possibly the previous kernel's output) is read, and z written, only after
    // the programmatic dependency resolved
    pdl_wait_prior_grid();
    pdl_launch_dependents();
    if (warp == 0) FN_TRACE(2);
    const int g = lane >> 2;
    const int kq = lane & 3;
    const int kchunks = (K + 31) >> 5;
    const int kbase = (warp * kchunks) / CWARPS;
    const int cpw = ((warp + 1) * kchunks) / CWARPS - kbase;  // <= CPW_MAX

    uint4 fa[CPW_MAX], fb[CPW_MAX];
    float s_lo = 0.f, s_hi = 0.f;
#pragma unroll
    for (int j = 0; j < CPW_MAX; ++j) {
      fa[j] = make_uint4(0u, 0u, 0u, 0u);
      fb[j] = make_uint4(0u, 0u, 0u, 0u);
      const int k = (kbase + j) * 32 + kq * 8;
      if (j < cpw && k < K) {
        if (g < M) fa[j] = *reinterpret_cast<const uint4*>(a + (size_t)g * K + k);
        if (M_HI && g + 8 < M) fb[j] = *reinterpret_cast<const uint4*>(a + (size_t)(g + 8) * K + k);
      }
      if (MODE == MODE_RMS) {
        const uint32_t* wa = reinterpret_cast<const uint32_t*>(&fa[j]);
        const uint32_t* wb = reinterpret_cast<const uint32_t*>(&fb[j]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float x;
          x = bf16lo(wa[q]); s_lo = fmaf(x, x, s_lo);
          x = bf16hi(wa[q]); s_lo = fmaf(x, x, s_lo);
          if (M_HI) {
            x = bf16lo(wb[q]); s_hi = fmaf(x, x, s_hi);
            x = bf16hi(wb[q]); s_hi = fmaf(x, x, s_hi);
          }
        }
      }
      if (MODE == MODE_DYT) {
        uint32_t* wa = reinterpret_cast<uint32_t*>(&fa[j]);
        uint32_t* wb = reinterpret_cast<uint32_t*>(&fb[j]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          wa[q] = tanh_approx_bf16x2(pack_bf16(bf16lo(wa[q]) * alpha, bf16hi(wa[q]) * alpha));
          if (M_HI) wb[q] = tanh_approx_bf16x2(pack_bf16(bf16lo(wb[q]) * alpha, bf16hi(wb[q]) * alpha));
        }
      }
    }
    if (MODE == MODE_RMS) {  // partial ssq of rows g, g+8 over this warp's K range
      s_lo += __shfl_xor_sync(0xffffffffu, s_lo, 1);
      s_lo += __shfl_xor_sync(0xffffffffu, s_lo, 2);
      s_hi += __shfl_xor_sync(0xffffffffu, s_hi, 1);
      s_hi += __shfl_xor_sync(0xffffffffu, s_hi, 2);
      if (kq == 0) {
        ssq_part[warp * 16 + g] = s_lo;
        ssq_part[warp * 16 + g + 8] = s_hi;
      }
    }

    // r_m is formed lazily by each reducing warp from the 15 partial ssq; part_full
    // of its first tile orders those writes.
    bool have_r = false;
    float r_row = 1.0f;  // lanes 0..15: r for row = lane
    const bool row_lo = g < M;
    const bool row_hi = g + 8 < M;
    int stage = 0;
    uint32_t phase = 0;
    for (int seq = 0;; ++seq) {
      mbar_wait_warp(&full[stage], phase);
      const int t = stage_tile[stage];
      if (seq == 0) FN_TRACE(1);
      if (warp == 0 && lane == 0) FN_TTRACE(seq, 1);
      if (t < 0) break;  // producer signalled the end (warp-uniform)
      const uint8_t* rowp = ring + ((size_t)stage * RPU + (g < RPU ? g : 0)) * ldb;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < CPW_MAX; ++j) {
        const int k = (kbase + j) * 32 + kq * 8;
        if (j < cpw) {  // warp-uniform
          uint4 w = make_uint4(0u, 0u, 0u, 0u);
          if (k < K && g < RPU) w = *reinterpret_cast<const uint4*>(rowp + (size_t)k * 2);
          mma_bf16_16816(acc, fa[j].x, fb[j].x, fa[j].y, fb[j].y, w.x, w.y);
          mma_bf16_16816(acc, fa[j].z, fb[j].z, fa[j].w, fb[j].w, w.z, w.w);
        }
      }
      const int slot = seq % SEG;
      const uint32_t sphase = (uint32_t)(seq / SEG) & 1u;
      if (seq >= SEG) mbar_wait_warp(&part_empty[slot], sphase ^ 1u);  // reducer of seq-SEG done
      // the partial store consumes the MMA results (hence the LDS above): the stage is
      // released only after this warp's shared-memory reads have returned
      *reinterpret_cast<float4*>(part + ((size_t)slot * CWARPS + warp) * 128 + lane * 4) =
          make_float4(acc[0], acc[1], acc[2], acc[3]);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[stage]);
        mbar_arrive(&part_full[slot]);
        if (warp == 0) FN_TTRACE(seq, 2);
        if (warp == CWARPS - 1) FN_TTRACE(seq, 4);
      }
      if (++stage == STAGES) { stage = 0; phase ^= 1; }

      if (warp == seq % CWARPS) {
        // reduce tile t: fixed-order sum over the 15 warps, deferred scale, bias, bf16 store
        mbar_wait_warp(&part_full[slot], sphase);
        if (MODE == MODE_RMS && !have_r) {
          float ss = 0.f;
#pragma unroll
          for (int w = 0; w < CWARPS; ++w) ss += ssq_part[w * 16 + (lane & 15)];
          r_row = rsqrtf(fmaf(ss, 1.0f / (float)K, eps));
          have_r = true;
        }
        const float* P = part + (size_t)slot * CWARPS * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = q * 32 + lane;
          float sum = 0.f;
#pragma unroll
          for (int w = 0; w < CWARPS; ++w) sum += P[w * 128 + e];
          const int ln = e >> 2, i = e & 3;
          const int row = (ln >> 2) + (i >= 2 ? 8 : 0);
          const int col = (ln & 3) * 2 + (i & 1);
          const int n = t * RPU + col;
          const float r = __shfl_sync(0xffffffffu, r_row, row);
          if (row < M && col < RPU && n < N) {
            const float cb = cstar != nullptr ? __ldg(cstar + n) : 0.0f;
            z[(size_t)row * N + n] = __float2bfloat16_rn(fmaf(sum, MODE == MODE_RMS ? r : 1.0f, cb));
          }
          part_fence[warp * 32 + lane] = sum;  // issues after every LDS of this tile returned
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&part_empty[slot]);
        if (lane == 0) FN_TTRACE(seq, 3);
      }
    }
  }
#ifdef FN_GEMV_TRACE
  __syncthreads();
  if (threadIdx.x == 0) {
    FN_TRACE(3);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_gemv_trace[slot_id & 1][blockIdx.x * 8 + 4] = smid;
    FN_TRACE(5);
  }
#endif
}

size_t gemv_smem_bytes(int M, int K) {
  if (K <= gt::K_MAX) return gemv_tma_smem_bytes(K);
  return gemv_regs_smem_bytes(M, K);
}

bool gemv_supported(int M, int K) {
  if (M < 1 || M > GEMV_MAX_M) return false;
  if (K <= gt::K_MAX) return true;                       // ring kernel: always fits (>= 2 stages)
  return gemv_regs_smem_bytes(M, K) <= 200 * 1024;       // register-streaming kernel
}

cudaError_t launch_gemv(const __nv_bfloat16* a, const __nv_bfloat16* Wt, const float* cstar, __nv_bfloat16* z,
                        int M, int K, int N, float eps, float alpha, int mode, int num_sms, cudaStream_t stream) {
  if (K > gt::K_MAX) return launch_gemv_regs(a, Wt, cstar, z, M, K, N, eps, alpha, mode, num_sms, stream);
  const size_t smem = gemv_tma_smem_bytes(K);
  const bool hi = M > 8;
  const void* fptr;
  if (mode == MODE_RMS) fptr = hi ? (const void*)flashnorm_gemv_kernel<MODE_RMS, true> : (const void*)flashnorm_gemv_kernel<MODE_RMS, false>;
  else if (mode == MODE_DYT) fptr = hi ? (const void*)flashnorm_gemv_kernel<MODE_DYT, true> : (const void*)flashnorm_gemv_kernel<MODE_DYT, false>;
  else fptr = hi ? (const void*)flashnorm_gemv_kernel<MODE_NONE, true> : (const void*)flashnorm_gemv_kernel<MODE_NONE, false>;
  if (cudaError_t e = ensure_smem_attr(fptr, (int)smem); e != cudaSuccess) return e;
  // one launch slot of the dynamic tile counter per call (64 slots, round robin): calls
  // in flight at the same time (PDL overlap, other streams) use distinct counters
  static std::atomic<unsigned> seq{0};
  int slot_id = (int)(seq.fetch_add(1u) % gt::SLOTS);
  int grid = (N + gt::RPU - 1) / gt::RPU;
  if (grid > num_sms) grid = num_sms;
  int nst = gemv_stages(K);
  void* args[] = {(void*)&a, (void*)&Wt, (void*)&cstar, (void*)&z, (void*)&M, (void*)&K, (void*)&N, (void*)&eps,
                  (void*)&alpha, (void*)&slot_id, (void*)&nst};
  // programmatic dependent launch: the W* stream of this call may start while the
  // previous kernel of the stream drains (the kernel waits before touching a / z)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gt::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fptr, args);
}

}  // namespace fn
