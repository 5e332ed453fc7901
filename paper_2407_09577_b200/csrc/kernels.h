// kernels.h — internal launcher declarations (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda.h>
#include <stdint.h>

namespace fn {

// per-device, thread-safe (api.cu): SM count of the current device; set the kernel's opt-in
// dynamic shared memory on the current device once (cached per (device, kernel))
int device_sms();
cudaError_t ensure_smem_attr(const void* fptr, int bytes);
// plain row-major TMA map (api.cu; false on failure)
bool encode_plain_tmap(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int elem_bytes, int box_cols,
                       int box_rows);
// debug (FN_DEBUG_LAYERNORM): max over rows of |mean(a_m)| / rms(a_m); synchronizes `stream`
cudaError_t layernorm_center_check(const void* a, int64_t M, int64_t K, int dtype, cudaStream_t stream,
                                   float* max_ratio);

enum KernelMode { MODE_RMS = 0, MODE_DYT = 1, MODE_NONE = 2 };

// RoPE epilogue (NEXT-2, Fig 5(b), readings c26-c27): output columns [0, n) are
// Q/K heads of h columns; for token m at position pos[m], adjacent pairs (2i, 2i+1) of a head
// rotate with cos'/sin' = table[pos][i] * r_m * qk (the 1/RMS and sqrt(1/sqrt h) folded into
// cos/sin once per token); the V columns >= n keep acc * r_m.  pos == nullptr: off.
struct RopeParams {
  const int* pos;
  const float* cos_tab;  // [max_pos][h/2]
  const float* sin_tab;
  int n, h;
  float qk;
  // QK-norm (NEXT-4, reading c28): g_q != nullptr -> each Q head (columns
  // [0, n_q)) / K head ([n_q, n)) of acc is RMS-normalized on its own, s_b = rsqrt(MS(head) +
  // eps_qk * MSe(a)) (no 1/RMS(a): it cancels), and g_q / g_k are fused into cos / sin.
  const float* g_q;
  const float* g_k;
  int n_q;
  float eps_qk;
};

struct GemmParams {
  int M, N, K;
  int num_m_blocks, num_n_blocks, num_tiles, num_k_blocks;
  float eps, alpha;
  const float* cstar;
  __nv_bfloat16* z;
  const __nv_bfloat16* a;  // activations (the DyT prologue of the pair kernel reads them directly)
  int group_m;  // M blocks per tile group (L2 locality: A of a group stays resident while W* streams)
  // GLU epilogue (MODE_RMS only, NEXT-1, reading c25): -1 = off, else GLU_SILU/GLU_RELU/GLU_BILINEAR.
  // W* rows are gate/up interleaved in 128-row blocks; z is [M][N/2] and s_out[M] the output scale.
  int glu_act;
  float* s_out;
  // MODE_NONE: optional per-row output scale z = RN(acc * row_scale[m] + c*) (the GLU down projection)
  const float* row_scale;
  RopeParams rope;
  // MODE_RMS: exact LayerNorm deferred past the contraction (NEXT-4, reading c29) when non-null:
  // u = 1^T W* [N]; the side group reduces sum(a - a0) and sum((a - a0)^2) per row (shift a0 =
  // a[m][0]) and the epilogue writes z = RN(fma(fma(-mu, u_j, acc), rsqrt(var + eps), c*_j))
  const float* ln_u;
  // fused column gather (NEXT-3): ndst > 0 -> the epilogue stores each output row
  // segment of this rank's N-column shard to ndst destinations (local or peer-mapped [M x ldz]
  // buffers, e.g. every rank's gathered z), at columns [col0, col0 + N); ndst = 0 -> z [M x N]
  int ndst, ldz, col0;
  __nv_bfloat16* zdst[8];
  // mc = 1 (ndst == 1): zdst[0] is an NVLS multicast address; the epilogue stores with multimem.st,
  // so the switch replicates each 16-byte segment to every rank's buffer (one NVLink write per
  // rank instead of P - 1)
  int mc;
  int stg;  // pair kernel epilogue: 1 = 32-byte (256-bit) row-segment stores, 0 = 16-byte (A/B knob)
  int bn;  // pair kernel tile width (256 or 224, gemm2_pick_bn); num_n_blocks = ceil(N / bn)
  int rms_local;  // pair kernel, RMS: A completes on each CTA's own barrier (see gemm2_sm100.cu)
  int tile_rot;   // pair kernel wave order: 0 plain grid stride, 1 rotated (pair_tile_rotation), 2 matched table
  // stream-K tail (pair kernel, sk_tiles > 0): the first sk_dp_waves waves are whole tiles
  // (cluster + w * C), the last sk_tiles tiles are cut into K ranges of U / C k blocks per pair
  // (U = sk_tiles x num_k_blocks); a tile split over two pairs is finished by the pair holding
  // its last k block, which adds the other pair's fp32 partial (sk_part, flag sk_flag) in a
  // fixed order before the usual epilogue.  sk_part: [sk_tiles][2 CTAs][128 rows][256] fp32 +
  // [sk_tiles][2][128] partial ssq; sk_flag: [sk_tiles][2] (zero between calls).
  int sk_tiles, sk_dp_waves;
  float* sk_part;
  unsigned* sk_flag;
};

// one unit of a pair's work: tile `tile`, k blocks [kb0, kb1); fix 0 = whole tile (or a stream-K
// tile this pair owns entirely), 1 = stream-K finisher (adds the contributor's partial, read from
// L2 in its epilogue), 3 = a finisher that is its pair's LAST item (the partial is staged into the
// idle TMEM accumulator buffer while its MMA runs), 2 = stream-K contributor (writes its partial,
// no output); sk >= 0: index of the stream-K tile
struct PairItem {
  int tile, kb0, kb1, fix, sk;
};
// the pair's stream-K items over its K range [u0, u1) = tiles a..c: the contributor part (head of
// tile c) first — it never waits, so every partial gets written — then the finisher part (tail of
// tile a, which waits for the partial of the pair before), then the whole tiles c-1 .. a+1, whose
// MMA hides the finisher's epilogue (a finisher last would leave its partial reads as the tail).
// s = 0, 1, 2...; false when done.
__host__ __device__ inline bool sk_item(const GemmParams& p, int cluster, int C, int s, PairItem& it) {
  const long long nkb = p.num_k_blocks;
  const long long U = (long long)p.sk_tiles * nkb;
  const long long u0 = (long long)cluster * U / C, u1 = (long long)(cluster + 1) * U / C;
  if (u1 <= u0) return false;
  const long long a = u0 / nkb, c = (u1 - 1) / nkb;
  if (s > c - a) return false;
  const long long tt = s == 0 ? c : (s == 1 ? a : c - (s - 1));
  it.kb0 = (int)((u0 > tt * nkb ? u0 : tt * nkb) - tt * nkb);
  it.kb1 = (int)((u1 < (tt + 1) * nkb ? u1 : (tt + 1) * nkb) - tt * nkb);
  it.fix = it.kb1 < nkb ? 2 : (it.kb0 > 0 ? (s == c - a ? 3 : 1) : 0);
  it.sk = (int)tt;
  it.tile = p.sk_dp_waves * C + (int)tt;
  return true;
}
constexpr int MAX_GATHER_DST = 8;
enum GluAct { GLU_SILU = 0, GLU_RELU = 1, GLU_BILINEAR = 2 };
// Fig 2(b) (ReLU FFN, not gated): z = RN(relu(acc)) unscaled, s_out = r — the scale is deferred
// to the FFN output (ReLU(s a) = s ReLU(a), s >= 0)
constexpr int RELU_FFN = 3;

// the GLU epilogue's element op (reading c25): SwiGLU scales the gate before the activation,
// ReGLU / bilinear leave both scales to the output (s = r^2)
static __device__ __forceinline__ float glu_apply(int act, float gate, float up, float r) {
  if (act == GLU_SILU) {
    const float x = gate * r;
    return __fdividef(x, 1.0f + __expf(-x)) * up;
  }
  if (act == GLU_RELU) return fmaxf(gate, 0.0f) * up;
  return gate * up;
}

// Persistent tile order: groups of `group_m` M blocks, M fastest inside a group, so the
// tiles in flight at any time share a few W* column blocks (each streamed from HBM
// once per group) while the group's A rows stay in L2.
__host__ __device__ inline void tile_coords(int tile, const GemmParams& p, int& m_blk, int& n_blk) {
  const int G = p.group_m;
  const int per_group = G * p.num_n_blocks;
  const int grp = tile / per_group;
  const int idx = tile - grp * per_group;
  const int m0 = grp * G;
  const int gm = (p.num_m_blocks - m0) < G ? (p.num_m_blocks - m0) : G;
  m_blk = m0 + idx % gm;
  n_blk = idx / gm;
}

// Pair kernel wave order (DESIGN.md §12 item 1).  Wave j holds tiles [C j, C j + C) of the
// order above, exactly as a plain grid stride would (same W* column blocks in flight), but pair
// `cluster` takes tile C j + (cluster + rot j) mod C.  With s = C mod gm, rot = gm - s (or C - s,
// whichever moves the M block more slowly) keeps m_blk = cluster mod gm for ~C / min(s, gm - s)
// waves, so a pair meets ~3 M blocks instead of gm / gcd(s, gm) (config 3: 8) and the RMS side
// group computes far fewer uncached ssq blocks.  rot = 0 is the plain grid stride.
__host__ __device__ inline int pair_tile_rotation(const GemmParams& p, int C) {
  if (!p.tile_rot) return 0;
  const int gm = p.group_m < p.num_m_blocks ? p.group_m : p.num_m_blocks;
  const int s = C % gm;
  if (s == 0) return 0;
  return (gm - s <= s) ? gm - s : C - s;
}
// the pair's next tile (-1 when done); j counts waves and is advanced past the returned tile
__host__ __device__ inline int next_pair_tile(int& j, int cluster, int C, int rot, int num_tiles) {
  for (;;) {
    const int base = C * j;
    if (base >= num_tiles) return -1;
    const int t = base + (cluster + rot * j) % C;
    ++j;
    if (t < num_tiles) return t;
  }
}

// Matched wave order (tile_rot = 2): the same per-wave tile sets, but the host assigns each
// wave's tiles to pairs so that a pair whose ssq cache already holds a tile's M block takes it
// (a per-wave greedy matching), which brings config 3 from 218 uncached tiles (rotation) to
// near the one-per-pair floor.  The table rides in the kernel's parameter space (<= 16 KiB).
constexpr int PAIR_SSQ_SLOTS = 16;  // mirrors the pair kernel's per-CTA ssq cache (slot = m % 16)
constexpr int SCHED_MAX = 8192;
constexpr int SCHED_MAX_PAIRS = 160;
struct PairSchedule {
  int waves;                // 0: no table (rotation / plain stride)
  uint16_t t[SCHED_MAX];    // [waves][C]: tile of pair c in wave j, 0xFFFF = idle
};
// launches with at most one wave use this parameter instead (no 16 KiB parameter upload)
struct PairScheduleNone {
  int waves;
};
__host__ __device__ inline int next_sched_tile(int& j, const PairSchedule& s, int cluster, int C) {
  while (j < s.waves) {
    const int t = s.t[j * C + cluster];
    ++j;
    if (t != 0xFFFF) return t;
  }
  return -1;
}
// greedy per-wave matching (a pair on the same M block, then one holding it in its ssq cache,
// then any); false when the table does not fit (the caller keeps the rotation)
inline bool build_pair_schedule(const GemmParams& p, int C, PairSchedule& s) {
  const int nt = p.num_tiles;
  s.waves = 0;
  if (C <= 0 || C > SCHED_MAX_PAIRS || nt <= 0 || nt >= 0xFFFF) return false;
  const int waves = (nt + C - 1) / C;
  if ((long long)waves * C > SCHED_MAX) return false;
  int tag[PAIR_SSQ_SLOTS * SCHED_MAX_PAIRS];
  int cur[SCHED_MAX_PAIRS];
  for (int i = 0; i < C * PAIR_SSQ_SLOTS; ++i) tag[i] = -1;
  for (int c = 0; c < C; ++c) cur[c] = -1;
  for (int j = 0; j < waves; ++j) {
    const int t0 = j * C, n = (nt - t0) < C ? (nt - t0) : C;
    bool used[SCHED_MAX_PAIRS] = {};
    bool done[SCHED_MAX_PAIRS] = {};
    for (int c = 0; c < C; ++c) s.t[t0 + c] = 0xFFFF;
    for (int pass = 0; pass < 3; ++pass) {
      for (int i = 0; i < n; ++i) {
        if (done[i]) continue;
        int m, nb;
        tile_coords(t0 + i, p, m, nb);
        for (int c = 0; c < C; ++c) {
          if (used[c]) continue;
          const bool ok = pass == 0   ? cur[c] == m
                          : pass == 1 ? tag[c * PAIR_SSQ_SLOTS + m % PAIR_SSQ_SLOTS] == m
                                      : true;
          if (!ok) continue;
          used[c] = done[i] = true;
          s.t[t0 + c] = (uint16_t)(t0 + i);
          cur[c] = m;
          tag[c * PAIR_SSQ_SLOTS + m % PAIR_SSQ_SLOTS] = m;
          break;
        }
      }
    }
  }
  s.waves = waves;
  return true;
}

// K3: tcgen05 prefill GEMM (gemm_sm100.cu)
int gemm_smem_bytes();
int gemm2_pick_bn(int M, int N, int num_sms, bool allow_224);
// stream-K tail plan of the pair kernel (gemm2_sm100.cu): scratch bytes, 0 = none
int64_t gemm2_sk_plan(int num_tiles, int nkb, int num_sms, int* sk_tiles, int* sk_dp_waves);
cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int mode, int num_sms,
                        cudaStream_t stream);

// K3 pair variant: cta_group::2, 256x256 tiles (gemm2_sm100.cu); RMS / NONE modes
int gemm2_smem_bytes();
cudaError_t launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb_half, const GemmParams& p, int mode,
                         int num_sms, cudaStream_t stream);

// K4: decode GEMV, M <= 16 (gemv.cu)
constexpr int GEMV_MAX_M = 16;
bool gemv_supported(int M, int K);  // decode kernel handles this (M, K)
// K4 on tcgen05 (gemv_tc.cu): tw = W* map (box 64 x 128), ta = token map (box 64 x 16)
bool gemv_tc_supported(int M, int N, int num_sms);
// K4w (gemv_wide.cu): batched decode, 17 <= M <= 128 tokens, rmsnorm / layernorm / none; the token
// tensor map's box has gemv_wide_tokens(M) rows (32 / 64 / 128)
int gemv_wide_tokens(int M);
bool gemv_wide_supported(int mode, int M, int K, int N, int num_sms);
cudaError_t launch_gemv_wide(const CUtensorMap& tw, const CUtensorMap& ta, const float* cstar, __nv_bfloat16* z,
                             int M, int K, int N, float eps, int mode, int num_sms, cudaStream_t stream,
                             const __nv_bfloat16* aptr, const float* row_scale = nullptr,
                             RopeParams rope = RopeParams{nullptr, nullptr, nullptr, 0, 0, 1.f, nullptr, nullptr, 0, 0.f});
int gemv_tc_split(int K, int N, int num_sms);      // K splits per tile
int gemv_tc_tile_rows(int mode, int K, int N, int num_sms);  // W* rows per tile (128 or 256; the TMA box)
// 64-wide k blocks per decode ring stage: 1 -> 2-D maps (box 64 x rows); 2 -> 3-D maps
// {64, rows, K/64} with strides {row, 128 B}, box {64, rows, 2} (W*) / {64, 16, 2} (tokens)
int gemv_tc_kblocks(int mode, int K, int N, int num_sms);
cudaError_t launch_gemv_tc(const CUtensorMap& tw, const CUtensorMap& ta, const float* cstar, __nv_bfloat16* z,
                           int M, int K, int N, float eps, float alpha, int mode, int num_sms, cudaStream_t stream,
                           const float* row_scale = nullptr,
                           RopeParams rope = RopeParams{nullptr, nullptr, nullptr, 0, 0, 1.f, nullptr, nullptr, 0, 0.f},
                           const __nv_bfloat16* wptr = nullptr,   // W* base (L2 prefetch hints only)
                           const __nv_bfloat16* aptr = nullptr);  // tokens [M x K] (RMS: ssq read from global)
size_t gemv_smem_bytes(int M, int K);
cudaError_t launch_gemv(const __nv_bfloat16* a, const __nv_bfloat16* Wt, const float* cstar, __nv_bfloat16* z,
                        int M, int K, int N, float eps, float alpha, int mode, int num_sms, cudaStream_t stream);

// K5: fp32 SIMT path (simt_f32.cu)
cudaError_t launch_linear_f32(const float* a, const float* Wt, const float* cstar, float* z, int M, int K, int N,
                              float eps, float alpha, int mode, cudaStream_t stream, const float* u = nullptr);

// K1/K2: folds (fold.cu).  dtype: 0 = bf16, 1 = f32
// glu_half: -1 = rows as given; 0 / 1 = write row j to (j/128)*256 + glu_half*128 + j%128 (the
// gate / up half of the 128-row-block interleave of flashnorm_fold_glu_weights)
cudaError_t launch_fold_colsum(const void* Wt_star, int64_t N, int64_t K, int dtype, float* u, cudaStream_t stream);
cudaError_t launch_fold_weights(const void* Wt, int64_t N, int64_t K, int dtype, const float* g, const float* b,
                                const float* c, void* Wt_star, float* c_star, cudaStream_t stream, int glu_half = -1);
int64_t fold_mean_center_workspace(int64_t n_out, int64_t d_in);
// tm_v3: plain 2-D map of Vt, box 512 B x 32 rows (three-launch K2); tm_v / tm_vs: maps of Vt / Vt_star,
// box FOLD_BOX_BYTES wide x FOLD_BOX_ROWS rows (cluster K2).  workspace: fold_mean_center_workspace bytes.
constexpr int FOLD_BOX_BYTES = 256;
constexpr int FOLD_BOX_ROWS = 128;  // K2 box: 256 B x 128 rows = 32 KiB
// Vt: the input again (the one-launch persistent K2 encodes its own maps of Vt / Vt_star)
cudaError_t launch_fold_mean_center(const CUtensorMap& tm_v3, const CUtensorMap& tm_v, const CUtensorMap& tm_vs,
                                    const void* Vt, int64_t n_out, int64_t d_in, int dtype, const float* b_prev,
                                    void* Vt_star, float* b_prev_star, void* workspace, cudaStream_t stream,
                                    int* launches);

// K6/K7: baseline norm + gather permute (aux.cu)
// K8: y = RN_bf16(tanh(alpha a)) over n elements (n % 8 == 0), bit-identical to the GEMM prologue.
cudaError_t launch_dyt_prepass(const __nv_bfloat16* a, __nv_bfloat16* y, int64_t n, float alpha, int num_sms,
                               cudaStream_t stream);
cudaError_t launch_baseline_norm(const void* a, const float* g, const float* b, int64_t M, int64_t K, float eps,
                                 int norm_kind /*0 rms,1 ln,2 dyt*/, float alpha, int dtype, void* y,
                                 cudaStream_t stream);
cudaError_t launch_gather_columns(const void* parts, int64_t P, int64_t M, int64_t Nl, int elem_bytes, void* z,
                                  cudaStream_t stream);

}  // namespace fn
