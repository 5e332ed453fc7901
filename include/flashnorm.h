/*
 * flashnorm.h — C ABI of the B200-native FlashNorm hot path (libflashnorm.so).
 *
 * FlashNorm (arXiv 2407.09577, /root/reference/PAPER.md) computes RMSNorm /
 * LayerNorm / DyT followed by a linear layer as
 *
 *        z = (a · W*) · 1/RMSe(a) + c*                      (Fig 1(c))
 *
 * with the normalization weights folded into W* (Fig 1(b)), the
 * norm bias folded into c* = c + b·W (Fig A) and LayerNorm's mean
 * centering folded into the preceding layer V* (Fig B).  The
 * per-token sum of squares is reduced IN PARALLEL with the contraction
 * (Fig 8(c)).
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Every tensor pointer is a DEVICE pointer owned by the caller (except the
 *    *_from_host entry point, which says so).  The library allocates no device
 *    memory; it keeps only host-side caches (TMA descriptors).
 *  - Matrices are dense row-major.  Weights use the nn.Linear storage layout
 *    Wt[N][K] (K contiguous): the paper's W (K x N, y = x W) is
 *    W[i][j] = Wt[j][i].  Activations a[M][K], outputs z[M][N].
 *  - fn_dtype selects the storage type of the matrices (a, Wt, Wt*, V, V*, z).
 *    Vectors g, b, c, c*, b_prev, b_prev* are always float32.
 *  - Alignment: every matrix pointer 16-byte aligned; K % 8 == 0 and
 *    N % 8 == 0 (bf16) / K % 4 == 0 and N % 4 == 0 (f32), else FN_ERR_ALIGN.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is asynchronous on that stream and never synchronizes, except
 *    flashnorm_linear_from_host (documented below).
 *  - Errors are status codes; no exception crosses the ABI.  On error,
 *    flashnorm_last_error() returns thread-local text naming the offending
 *    shapes/values.  Shapes are never broadcast.
 *  - Outputs never alias inputs.
 */
#ifndef FLASHNORM_H_
#define FLASHNORM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FN_OK = 0,
    FN_ERR_NULL = 1,         /* required pointer is NULL                          */
    FN_ERR_SHAPE = 2,        /* non-positive or inconsistent size                 */
    FN_ERR_DTYPE = 3,        /* unknown fn_dtype                                  */
    FN_ERR_ALIGN = 4,        /* pointer not 16-B aligned / K, N not multiple of 8 */
    FN_ERR_VALUE = 5,        /* eps < 0, non-finite eps/alpha, bad mode           */
    FN_ERR_UNSUPPORTED = 6,  /* valid request this build does not implement       */
    FN_ERR_CUDA = 7,         /* CUDA runtime/driver failure (text has the reason) */
    FN_ERR_NCCL = 8          /* NCCL missing or failed (text has the reason)       */
} fn_status;

typedef enum {
    FN_RMSNORM = 0,    /* z = (a W*) * rsqrt(ssq/K + eps) + c*         PAPER.md:14,17,177 */
    FN_LAYERNORM = 1,  /* same kernel math on an input already mean-centered by a
                          V* folded with flashnorm_fold_mean_center     */
    FN_DYT = 2,        /* z = tanh(alpha a) W* + c* (no deferral: tanh is not scale-
                          commutative); reading c10 of DESIGN.md                          */
    FN_NONE = 3        /* z = a W* + c* — plain linear layer: the upstream V* layer of
                          config 4 and the GEMM half of the unfused baseline             */
} fn_mode;

typedef enum { FN_BF16 = 0, FN_F32 = 1 } fn_dtype;

typedef enum {
    FN_PATH_AUTO = 0,    /* M <= 16: decode kernel; 17 <= M <= 128 (rmsnorm / layernorm /
                            none, DyT with a workspace): the batched-decode kernel when its
                            cluster plan fits; else tcgen05 GEMM                              */
    FN_PATH_GEMM = 1,    /* force the tcgen05/TMEM/TMA kernel (bf16 only)                   */
    FN_PATH_GEMV = 2,    /* force the decode kernel (bf16, M <= 16): the tcgen05 split-K
                            kernel when ceil(N/128) <= #SMs, else the mma.sync kernel;
                            17 <= M <= 128: the batched-decode kernel where supported        */
    FN_PATH_SIMT = 3,    /* the fp32 FFMA kernel (the only path for FN_F32)                 */
    FN_PATH_GEMM1 = 4,   /* force the 1-CTA tcgen05 kernel (FN_PATH_GEMM picks the CTA-pair
                            cta_group::2 kernel when M > 128)                               */
    FN_PATH_GEMV_MMA = 5 /* force the mma.sync decode kernel (comparison / fallback)        */
} fn_path;

/* --------------------------------------------------------------------------
 * flashnorm_fold_weights — offline fold of g and b into W*, c*.
 *   PAPER.md:25 (Fig A): c* = c + b·W with the ORIGINAL W, then
 *   PAPER.md:16 (Fig 1(b)): W*_{i,j} = g_i · W_{i,j}.
 *
 *   Wt      [N][K] storage dtype, input.
 *   g       [K] float32 or NULL (= ones);  b [K] float32 or NULL (= zeros);
 *   c       [N] float32 or NULL (= zeros).
 *   Wt_star [N][K] storage dtype, output.
 *   c_star  [N] float32 output; may be NULL only if b == NULL and c == NULL.
 *
 *   fold_weights numerics (the contract the CPU mirror reproduces bit-exactly):
 *     Wt_star[j][i] = RN_dtype( RN_f32( g_i * Wt[j][i] ) )
 *     c_star[j]     = RN_f32( (double)c_j + S_j ), S_j = fp64 sum of the exact
 *                     products b_i*Wt[j][i]: lane l (0..31) of row j's warp sums
 *                     its 16-byte chunks q = l, l+32, ... ascending (elements
 *                     ascending inside a chunk), then the 32 lane sums are
 *                     combined by an xor butterfly 16,8,4,2,1.
 * -------------------------------------------------------------------------- */
fn_status flashnorm_fold_weights(const void* Wt, int64_t N, int64_t K, fn_dtype dtype,
                                 const float* g, const float* b, const float* c,
                                 void* Wt_star, float* c_star, void* stream);

/* --------------------------------------------------------------------------
 * flashnorm_fold_mean_center — offline fold of LayerNorm's mean centering into
 * the preceding linear layer V.  PAPER.md:42-49 (§1.2, Fig B):
 *   s_i = sum_j v_{i,j},  v*_{i,j} = v_{i,j} - s_i / n.
 *   Paper V is d_in x n_out; storage Vt[n_out][d_in].  n = n_out (the width of
 *   the LayerNorm that follows).  V's own bias: b_prev* = b_prev - mean(b_prev)
 *   (paper silent; reading c7).
 *
 *   Vt          [n_out][d_in] storage dtype, input.
 *   b_prev      [n_out] float32 or NULL;  b_prev_star [n_out] float32 output or
 *               NULL (must be non-NULL iff b_prev is non-NULL).
 *   Vt_star     [n_out][d_in] storage dtype, output.
 *   workspace   device scratch of flashnorm_fold_mean_center_workspace_bytes()
 *               bytes, 16-B aligned (fp64 partial column sums, then s_i / n); no
 *               initialization needed, contents unspecified on return.
 *   One cooperative launch when V fits the SMs' shared memory (ceil(n_out/64) x
 *   ceil(row_bytes/512) tiles of 32 KiB, at most 7 per SM: the 4096 x 4096 bf16 V of
 *   config 4 does): every CTA holds its tiles from the HBM read to the V* store, with
 *   two grid-wide barriers (partials -> s_i -> centering).  Otherwise three launches
 *   (partials, s_i + b_prev*, centering; PDL-chained).  FN_K2_VARIANT=3 forces the
 *   three launches; FN_K2_VARIANT=1 a one-launch cluster kernel that computes the
 *   same bits with no workspace (clusters of 8 CTAs own a 256-byte column slab, the
 *   lane sums meet over DSMEM); both measured slower (A/B references, DESIGN.md §6 K2).

 *   fold_mean_center numerics (mirrored bit-exactly on the CPU):
 *     partial[c][i] = fp64 sum of Vt[j][i], j in [32c, 32c+32) ascending
 *     s_i           = fp64: lane l (0..31) sums partial[c][i] for c = l, l+32, ...
 *                     ascending, then the 32 lane sums are combined by an xor
 *                     butterfly 16,8,4,2,1
 *     mu_i          = RN_f32( s_i / (double)n_out )       (fp64 quotient, one rounding)
 *     Vt_star[j][i] = RN_dtype( fsub_rn( Vt[j][i], mu_i ) ) (one f32 subtraction; IEEE: inf/NaN
 *                     propagate)
 *     b_prev_star_j = RN_f32( (double)b_prev_j - T / n_out ), T: 256 threads,
 *                     thread t sums j = t, t+256, ... ascending (fp64), xor
 *                     butterfly 16,8,4,2,1 per warp, then the 8 warp totals
 *                     added in ascending order.
 * -------------------------------------------------------------------------- */
int64_t flashnorm_fold_mean_center_workspace_bytes(int64_t n_out, int64_t d_in);
fn_status flashnorm_fold_mean_center(const void* Vt, int64_t n_out, int64_t d_in, fn_dtype dtype,
                                     const float* b_prev, void* Vt_star, float* b_prev_star,
                                     void* workspace, void* stream);

/* --------------------------------------------------------------------------
 * flashnorm_linear — the per-token hot path.  PAPER.md:17 (Fig 1(c)), with the
 * RMS reduced in parallel with the contraction (Fig 8(c)):
 *
 *   rmsnorm / layernorm:  z[m][j] = RN( fma(acc[m][j], r_m, c*_j) ),
 *                         acc = sum_k a[m][k] W*t[j][k]  (fp32 accumulate),
 *                         r_m = rsqrt( ssq_m / K + eps ),  ssq_m = sum_k a[m][k]^2
 *                         (eps inside the sqrt; scale BEFORE the
 *                         bias).
 *   dyt:                  z = RN( sum_k RN_dtype(tanh(alpha a[m][k])) W*t[j][k] + c*_j )
 *   none:                 z = RN( sum_k a[m][k] W*t[j][k] + c*_j )
 *
 *   a       [M][K] storage dtype;  Wt_star [N][K];  c_star [N] float32 or NULL;
 *   z       [M][N] storage dtype, output (must not alias a).
 *   eps     >= 0 and finite (ignored for dyt/none);  alpha finite (dyt only).
 *   M == 0 is a no-op returning FN_OK.  A row with ssq == 0 and eps == 0 yields
 *   IEEE inf/NaN in that row (documented; not reported per row).
 *   bf16: tcgen05 GEMM (prefill), batched decode (17..128 tokens) or decode GEMV (<= 16),
 *         chosen by M (FN_PATH_AUTO);
 *   f32:  FFMA SIMT kernel (no TF32).
 *   FN_LAYERNORM trusts that `a` was mean-centered upstream: release builds do
 *   not check it.  With the environment variable FN_DEBUG_LAYERNORM=1 the call first
 *   measures max_m |mean(a_m)| / rms(a_m) on the device (one extra kernel and a stream
 *   synchronization) and returns FN_ERR_VALUE, naming the value, if it exceeds 1e-2.
 *
 *   Programmatic dependent launch (decode paths, M <= 128): the decode kernels are launched
 *   with programmatic stream serialization and start streaming Wt_star (and c_star) into
 *   shared memory BEFORE waiting for the preceding kernel on `stream`; `a` is read only
 *   after that wait and `z` written only after it.  Precondition: Wt_star and c_star are not
 *   written by a kernel that is still running on `stream` when this call is enqueued
 *   (weights are written once, offline: the fold kernels of this library, torch copies and
 *   cuBLAS all complete and flush before a dependent launch may start, because none of them
 *   triggers early).  The only kernels of this library that trigger early
 *   (griddepcontrol.launch_dependents) are the decode kernels themselves, which write z; a
 *   decode call whose Wt_star is the z of the immediately preceding decode call must put an
 *   event or a plain kernel between them.
 * -------------------------------------------------------------------------- */
fn_status flashnorm_linear(const void* a, const void* Wt_star, const float* c_star,
                           int64_t M, int64_t K, int64_t N, float eps, float alpha,
                           fn_mode mode, fn_dtype dtype, void* z, void* stream);

/* Same as flashnorm_linear with an explicit kernel choice (tests, benchmarks). */
fn_status flashnorm_linear_ex(const void* a, const void* Wt_star, const float* c_star,
                              int64_t M, int64_t K, int64_t N, float eps, float alpha,
                              fn_mode mode, fn_dtype dtype, void* z, fn_path path, void* stream);

/* flashnorm_linear_ws — flashnorm_linear_ex with caller-owned device scratch, used for two things:
 *  (1) mode == FN_DYT on a bf16 GEMM path (M > 16 or an explicit GEMM path): the library computes
 *      RN_bf16(tanh(alpha a)) ONCE per element (kernel K8, an HBM-bound pre-pass; DyT is named at
 *      PAPER.md:5 and its bias at PAPER.md:25, the elementwise formula is reading c10) and then runs
 *      the GEMM in mode FN_NONE on it, instead of recomputing tanh in the A-tile prologue of every N
 *      tile (MUFU tanh: ~16 values/clk/SM on sm_100a, the rate at which the tensor core consumes A at
 *      BN = 256, DESIGN.md §6 K8).  z is bit-identical to the prologue path.  Two launches.
 *  (2) the stream-K tail of the CTA-pair GEMM (plain epilogue): when the pair-tile count T is not
 *      a multiple of the 74 CTA pairs and T < 4 x 74, the last (T mod 74) + 74 tiles are split
 *      into equal K ranges, and a tile split over two pairs is finished by the pair holding its
 *      last k block, which adds the other's fp32 partial in a fixed order
 *      (deterministic, but not bit-identical to the unsplit tile).  Which kernels use it is the
 *      environment variable FN_GEMM2_SK, read at every call: 0 none, 1 the mode-none kernel
 *      (FN_NONE, DyT after its pre-pass), 2 also rmsnorm / layernorm; unset (default): the
 *      mode-none kernel when K >= 8192 (+2.7 % on the FFN down projection, no gain at K = 4096,
 *      DESIGN.md §6); flashnorm_linear_workspace_bytes follows the policy.
 *  Layout: [4 KiB stream-K flags][stream-K fp32 partials][DyT buffer of M*K*2].  The FIRST 4 KiB
 *  MUST BE ZERO before a call (zero-fill the buffer once); every call leaves them zero, so one
 *  workspace serves any sequence of calls on one stream (and CUDA graph replays).  The rest is
 *  scratch, contents unspecified on return.
 *   workspace        16-B aligned device scratch, or NULL (then workspace_bytes must be 0 and the
 *                    call is exactly flashnorm_linear_ex); must not alias a, Wt_star or z;
 *                    ownership stays with the caller.
 *   workspace_bytes  its size; a DyT GEMM that needs more returns FN_ERR_VALUE; a workspace too
 *                    small for the stream-K scratch runs whole tiles.
 * Other modes / paths ignore the workspace.
 * flashnorm_linear_workspace_bytes returns the size a call with the same
 * arguments would use (0 = none needed). */
int64_t flashnorm_linear_workspace_bytes(int64_t M, int64_t K, int64_t N, fn_mode mode, fn_dtype dtype,
                                         fn_path path);
fn_status flashnorm_linear_ws(const void* a, const void* Wt_star, const float* c_star,
                              int64_t M, int64_t K, int64_t N, float eps, float alpha,
                              fn_mode mode, fn_dtype dtype, void* z, fn_path path,
                              void* workspace, int64_t workspace_bytes, void* stream);

/* --------------------------------------------------------------------------
 * FFN with a GLU variant (NEXT-1, §2.2 Figs 3-4; readings c24, c25).
 * Bias-free FFN: y = (act(x W_gate) ⊙ (x W_up)) W_down with x = RMSNorm(a; g).
 *
 * flashnorm_fold_glu_weights — W*_gate = diag(g) W_gate, W*_up = diag(g) W_up,
 *   stored gate/up interleaved in 128-row blocks so one 256-row GEMM tile holds gate block
 *   t and up block t:  Wgu_star[256 t + c] = W*_gate^T[128 t + c],
 *                      Wgu_star[256 t + 128 + c] = W*_up^T[128 t + c],   c < 128.
 *   Wgt, Wut   [F][K] storage dtype (transposed paper W_gate, W_up: n x f), F % 128 == 0.
 *   g          [K] float32 or NULL (ones).   Wgu_star [2F][K] output (must not alias).
 *   Numerics: each element exactly as flashnorm_fold_weights (RN_dtype(RN_f32(g w))).
 *
 * flashnorm_glu_linear — the gate||up GEMM with the GLU epilogue (bf16 only):
 *   G = a W*_gate, U = a W*_up (fp32 accumulate), r_m = rsqrt(ssq_m/K + eps) (ssq beside the
 *   contraction, as flashnorm_linear);
 *   FN_GLU_SILU (SwiGLU, Fig 3(b)):     h = RN(silu(G r) * U),  s_m = r_m
 *   FN_GLU_RELU / FN_GLU_BILINEAR (Fig 4(b)): h = RN(act(G) * U), s_m = r_m^2 = 1/MSe(a_m)
 *   The FFN output is y = (h W_down) * s: pass s to flashnorm_linear_scaled (the deferred
 *   scaling at the FFN output).  h [M][F] bf16 output, s [M] float32 output (16-B aligned).
 *
 * flashnorm_linear_scaled — z = RN((a W*) * row_scale_m + c*) (bf16 only): a plain linear
 *   layer with a given per-row output scale (the down projection of Figs 3(b)/4(b)).
 * -------------------------------------------------------------------------- */
typedef enum { FN_GLU_SILU = 0, FN_GLU_RELU = 1, FN_GLU_BILINEAR = 2 } fn_glu_act;

/* flashnorm_relu_ffn_up — FFN with ReLU (not gated), Fig 2(b): the whole
 *   normalization is deferred to the FFN output because ReLU(s a) = s ReLU(a) for s >= 0:
 *   h = RN(relu(a W*_up)) (no scale), s_m = r_m = rsqrt(ssq_m/K + eps); the FFN output is
 *   y = (h W_down) * s via flashnorm_linear_scaled.  Wt_star [F][K] (W*_up^T), h [M][F] bf16,
 *   s [M] float32.  bf16 only, tcgen05 GEMM. */
fn_status flashnorm_relu_ffn_up(const void* a, const void* Wt_star, int64_t M, int64_t K, int64_t F, float eps,
                                fn_dtype dtype, void* h, float* s, void* stream);

fn_status flashnorm_fold_glu_weights(const void* Wgt, const void* Wut, int64_t F, int64_t K, fn_dtype dtype,
                                     const float* g, void* Wgu_star, void* stream);
fn_status flashnorm_glu_linear(const void* a, const void* Wgu_star, int64_t M, int64_t K, int64_t F, float eps,
                               fn_glu_act act, fn_dtype dtype, void* h, float* s, void* stream);
fn_status flashnorm_linear_scaled(const void* a, const void* Wt_star, const float* c_star, const float* row_scale,
                                  int64_t M, int64_t K, int64_t N, fn_dtype dtype, void* z, void* stream);
/* flashnorm_linear_scaled_ws — flashnorm_linear_scaled with the caller's workspace, exactly as
 *   flashnorm_linear_ws treats it for FN_NONE (size: flashnorm_linear_workspace_bytes(M, K, N,
 *   FN_NONE, ...); first 4 KiB zero before the call, left zero): lets the stream-K tail run on
 *   the down projection (K = F, usually >= 8192).  NULL workspace = flashnorm_linear_scaled. */
fn_status flashnorm_linear_scaled_ws(const void* a, const void* Wt_star, const float* c_star, const float* row_scale,
                                     int64_t M, int64_t K, int64_t N, fn_dtype dtype, void* z, void* workspace,
                                     int64_t workspace_bytes, void* stream);

/* --------------------------------------------------------------------------
 * flashnorm_qkv_rope_linear — the Q/K/V projection with RoPE (NEXT-2, PAPER.md:80-94,
 * §3 Fig 5(b); readings c26, c27), bias-free, bf16 only:
 *   acc = a W*^T (W* = folded [Q|K|V] weights, N rows: Q and K heads in the first n_rope rows,
 *   head_dim rows per head, V after), r_m = rsqrt(ssq_m/K + eps) reduced beside the contraction;
 *   Q/K columns: pairs (2i, 2i+1) of each head rotate with the per-token cos/sin scaled ONCE by
 *   r_m * qk_scale (shared by every head):
 *     z[m][2i]   = RN(acc_2i * c - acc_2i+1 * s),  z[m][2i+1] = RN(acc_2i+1 * c + acc_2i * s),
 *     c = cos_tab[pos_m][i'] * r_m * qk_scale,  s = sin_tab[pos_m][i'] * r_m * qk_scale,
 *     i' = (column mod head_dim) / 2;
 *   V columns (>= n_rope): z = RN(acc * r_m)  ("the V linear layer still needs the
 *   normalization at its output").
 *   positions [M] int32 (device), cos_tab / sin_tab [max_pos][head_dim/2] float32 (device;
 *   the caller guarantees 0 <= positions[m] < max_pos).  qk_scale: pass sqrt(1/sqrt(head_dim))
 *   to fold the scaled dot-product's 1/sqrt(head_dim), or 1.
 *   n_rope % head_dim == 0, n_rope % 32 == 0, head_dim even.  Decode (M <= 16) runs on the
 *   tcgen05 split-K kernel, prefill on the tcgen05 GEMM.
 * -------------------------------------------------------------------------- */
fn_status flashnorm_qkv_rope_linear(const void* a, const void* Wt_star, int64_t M, int64_t K, int64_t N,
                                    int64_t n_rope, int64_t head_dim, const int32_t* positions,
                                    const float* cos_tab, const float* sin_tab, float qk_scale, float eps,
                                    fn_dtype dtype, void* z, void* stream);

/* --------------------------------------------------------------------------
 * flashnorm_qk_norm_rope_linear — Q/K/V projection with OpenELM-style QK-normalization and
 * RoPE (NEXT-4 part, §4 Figs 6(b) + 7(b); reading c28), bf16 only:
 *   acc = a W*^T; Q heads = columns [0, n_q), K heads = [n_q, n_q + n_k), head_dim each, V after.
 *   Per token m and Q/K head b (head_dim values of acc; no 1/RMS(a) on this path, it cancels):
 *     s_b = rsqrt(MS(b) + eps_qk * MSe(a_m)),  MSe(a_m) = ssq_m/K + eps  (exact for any eps_qk)
 *     y_2i   = RN((b_2i cos_i g_2i - b_2i+1 sin_i g_2i+1) * s_b * qk_scale)
 *     y_2i+1 = RN((b_2i+1 cos_i g_2i+1 + b_2i sin_i g_2i) * s_b * qk_scale)
 *   with g = g_q (Q heads) or g_k (K heads) [head_dim] float32, cos_i / sin_i = table[pos_m][i];
 *   V columns: RN(acc * r_m).  head_dim in {32, 64, 128, 256}; decode (M <= 16) runs on the
 *   tcgen05 split-K kernel when head_dim divides 128, else on the tcgen05 GEMM.
 * -------------------------------------------------------------------------- */
fn_status flashnorm_qk_norm_rope_linear(const void* a, const void* Wt_star, int64_t M, int64_t K, int64_t N,
                                       int64_t n_q, int64_t n_k, int64_t head_dim, const float* g_q,
                                       const float* g_k, float eps_qk, const int32_t* positions,
                                       const float* cos_tab, const float* sin_tab, float qk_scale, float eps,
                                       fn_dtype dtype, void* z, void* stream);

/* --------------------------------------------------------------------------
 * LayerNorm deferred past the contraction WITHOUT a foldable preceding layer
 * (NEXT-4; reading c29).  LayerNorm = mean centering then RMSNorm
 * (PAPER.md:33); the §1.2 derivation moves the mean through a
 * linear layer by summing weights — applied to the layer AFTER the norm:
 *   (a - mu 1) W* = a W* - mu u,   u = 1^T W*  (u_j = sum_k W*t[j][k]).
 *
 * flashnorm_fold_colsum — offline: u[j] = RN_f32( fp64 sum_k W*t[j][k] ) in the
 *   c* order of "fold_weights numerics" above (lane l: 16-byte chunks l, l+32, ...
 *   ascending, elements ascending; xor butterfly 16,8,4,2,1), i.e. exactly the c*
 *   that flashnorm_fold_weights computes for b = 1, c = NULL on Wt_star.
 *   Wt_star [N][K] storage dtype (16-B aligned, K % 8 == 0); u [N] float32 output.
 *
 * flashnorm_layernorm_linear — per token, with the row statistics reduced beside
 *   the contraction from the same A tiles (shift a0 = a[m][0] against cancellation):
 *     mu_m  = a0 + S1/K,  var_m = max(S2/K - (S1/K)^2, 0),
 *     S1 = sum_k (a[m][k] - a0),  S2 = sum_k (a[m][k] - a0)^2     (fp32)
 *     z[m][j] = RN( fma( fma(-mu_m, u_j, acc[m][j]), rsqrt(var_m + eps), c*_j ) )
 *   with W* = diag(g) W and c* = c + b W from flashnorm_fold_weights (LayerNorm's g
 *   and b) and u from flashnorm_fold_colsum(W*).  a [M][K], z [M][N]; eps >= 0.
 *   bf16: tcgen05 GEMM kernels for every M (decode shapes run the 1-CTA kernel);
 *   f32: the FFMA kernel.  The correction subtracts mu u_j from acc, so rows with
 *   |mean| >> std lose relative accuracy in fp32 accumulation (reading c9).
 * -------------------------------------------------------------------------- */
fn_status flashnorm_fold_colsum(const void* Wt_star, int64_t N, int64_t K, fn_dtype dtype, float* u,
                                void* stream);
fn_status flashnorm_layernorm_linear(const void* a, const void* Wt_star, const float* u, const float* c_star,
                                     int64_t M, int64_t K, int64_t N, float eps, fn_dtype dtype, void* z,
                                     void* stream);

/* --------------------------------------------------------------------------
 * flashnorm_linear_gather — the column-parallel layer with the all-gather fused into the GEMM
 * epilogue (NEXT-3; W* column-sharded, activations replicated, no collective
 * needed to COMPUTE a shard).  This rank's shard z[:, col0 : col0 + N] = flashnorm_linear(a,
 * Wt_star, c_star, ...) is stored by the epilogue straight into each of the ndst destination
 * buffers z_dsts[d] ([M][ldz] bf16, row-major) — on a multi-GPU node these are the peer-mapped
 * gathered outputs of every rank (NVLink stores issued tile by tile, overlapping the next
 * tile's mainloop, instead of a separate all-gather + permute); on one device, any set of
 * local buffers.  Same arithmetic and bits as flashnorm_linear for every destination.
 *   z_dsts   HOST array of ndst device pointers (1 <= ndst <= 8), each 16-B aligned,
 *            none aliasing a; the caller orders the peers' readers after this call (e.g. a
 *            barrier after the stream completes).
 *   ldz      row stride of the destinations in elements, ldz >= col0 + N, ldz % 8 == 0;
 *   col0     first column of this shard, col0 % 8 == 0.
 *   bf16 only; runs the tcgen05 GEMM kernels for every M (decode shapes included).
 * -------------------------------------------------------------------------- */
fn_status flashnorm_linear_gather(const void* a, const void* Wt_star, const float* c_star, int64_t M, int64_t K,
                                  int64_t N, float eps, float alpha, fn_mode mode, fn_dtype dtype,
                                  void* const* z_dsts, int ndst, int64_t ldz, int64_t col0, void* stream);

/* flashnorm_linear_gather_multicast — the same fused gather through ONE NVLink-SHARP (NVLS) multicast
 * address: z_mc is the multicast mapping of a buffer bound on every rank (cuMulticastCreate /
 * cuMulticastBindMem, e.g. torch symmetric memory's multicast_ptr); the epilogue stores each 16-byte
 * segment of this rank's shard with multimem.st, and the NVSwitch writes it into every rank's
 * [M][ldz] buffer — each rank sends its shard once (M x N x 2 bytes) instead of P - 1 times.
 * Same arithmetic and bits as flashnorm_linear_gather.  z_mc must be a multicast address (a plain
 * pointer faults); ordering of the peers' readers is the caller's (a barrier after the stream).
 * ldz, col0 as flashnorm_linear_gather; bf16 only. */
fn_status flashnorm_linear_gather_multicast(const void* a, const void* Wt_star, const float* c_star, int64_t M,
                                            int64_t K, int64_t N, float eps, float alpha, fn_mode mode,
                                            fn_dtype dtype, void* z_mc, int64_t ldz, int64_t col0, void* stream);

/* --------------------------------------------------------------------------
 * Opt-in multi-GPU plumbing.  W* is column-sharded, the
 * activations replicated: every rank computes its shard z_local [M][N_local]
 * with flashnorm_linear and NO collective; only a caller that wants the
 * gathered z [M][P * N_local] on every rank calls flashnorm_allgather_columns.
 * NCCL is loaded at run time (libnccl.so.2; the instance PyTorch loaded, if
 * any); without it these calls return FN_ERR_NCCL.
 *
 *   flashnorm_comm_unique_id   writes an ncclUniqueId (FN_NCCL_UNIQUE_ID_BYTES)
 *                              on one rank; the caller broadcasts it.
 *   flashnorm_comm_init        ncclCommInitRank(nranks, id, rank) -> *comm
 *                              (one GPU per rank: call with that GPU current).
 *   flashnorm_comm_destroy     ncclCommDestroy (NULL is a no-op).
 *   flashnorm_comm_count       ncclCommCount: *nranks = the communicator's rank count P
 *                              (callers size z_full / workspace from it).
 *   flashnorm_allgather_columns  ncclAllGather(z_local -> workspace [P][M][N_local])
 *                              then the permute into z_full [M][P * N_local], both on
 *                              `stream`; P is the communicator's rank count (not an
 *                              argument); z_full must hold M*P*N_local elements and the
 *                              workspace flashnorm_allgather_workspace_bytes(P, ...) bytes.
 *                              bf16 or f32; workspace must not alias z_local / z_full.
 * The epilogue-fused alternative is flashnorm_linear_gather (peer-mapped outputs).
 * -------------------------------------------------------------------------- */
#define FN_NCCL_UNIQUE_ID_BYTES 128
fn_status flashnorm_comm_unique_id(void* id_out);
fn_status flashnorm_comm_init(const void* nccl_unique_id, int nranks, int rank, void** comm);
fn_status flashnorm_comm_destroy(void* comm);
fn_status flashnorm_comm_count(void* comm, int* nranks);
int64_t flashnorm_allgather_workspace_bytes(int64_t P, int64_t M, int64_t N_local, fn_dtype dtype);
fn_status flashnorm_allgather_columns(const void* z_local, int64_t M, int64_t N_local, fn_dtype dtype,
                                      void* z_full, void* workspace, void* comm, void* stream);

/* End-to-end variant: a_host / z_host are HOST pointers (pinned memory for
 * asynchronous copies); a_dev / z_dev are caller-owned device scratch of
 * M*K / M*N elements.  Enqueues H2D(a) -> flashnorm_linear -> D2H(z) and
 * returns without synchronizing (the caller synchronizes `stream` before
 * reading z_host).  For M >= 1024 the rows are pipelined in ~8 chunks over
 * two library-owned copy streams (per device) joined to `stream` by events:
 * H2D of chunk c+1 || the linear of chunk c on `stream` || D2H of chunk c-1.
 * Rows are independent, so z is identical to the unchunked call.  All work
 * of the call is ordered after earlier work on `stream` and before later
 * work on it. */
fn_status flashnorm_linear_from_host(const void* a_host, const void* Wt_star, const float* c_star,
                                     int64_t M, int64_t K, int64_t N, float eps, float alpha,
                                     fn_mode mode, fn_dtype dtype, void* a_dev, void* z_dev,
                                     void* z_host, void* stream);

/* --------------------------------------------------------------------------
 * Measurement-only pieces (not the method): the unfused two-kernel baseline
 * of BASELINE.json:5 — RMSNorm/LayerNorm writing y = RN(a*r*g + b) (Fig 1(a)
 * first half), then flashnorm_linear(mode = FN_NONE) on the ORIGINAL W.
 * -------------------------------------------------------------------------- */
fn_status flashnorm_baseline_norm(const void* a, const float* g, const float* b,
                                  int64_t M, int64_t K, float eps, fn_mode mode, float alpha,
                                  fn_dtype dtype, void* y, void* stream);

/* --------------------------------------------------------------------------
 * Multi-GPU helper: after an all-gather of P column shards z_parts[P][M][N_local]
 * (W* column-sharded, activations replicated), permute into
 * z[M][P*N_local].  Pure data movement.
 * -------------------------------------------------------------------------- */
fn_status flashnorm_gather_columns(const void* z_parts, int64_t P, int64_t M, int64_t N_local,
                                   fn_dtype dtype, void* z, void* stream);

/* Diagnostics. */
const char* flashnorm_status_string(fn_status s);
const char* flashnorm_last_error(void);
/* Number of kernels this library launched on the calling thread since the last
 * reset (used by bench.py's gpu_launches count). */
int64_t flashnorm_launch_count(void);
void flashnorm_reset_launch_count(void);
/* Library version string: "flashnorm-b200 <semver> sm_100a". */
const char* flashnorm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FLASHNORM_H_ */
