// api.cu — the extern "C" boundary declared in include/flashnorm.h.
//
// Validation (shapes, alignment, values -> fn_status + thread-local text),
// kernel selection, a mutex-guarded cache of TMA descriptors (cuTensorMapEncodeTiled
// obtained through cudaGetDriverEntryPoint, so the library never links libcuda),
// and the launch counter used by bench.py.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/flashnorm.h"
#include "kernels.h"
#include <algorithm>
#include <atomic>

namespace fn {

// Per-device, thread-safe launch prerequisites (a process may drive several GPUs from several
// threads): the SM count and the opt-in dynamic shared memory size are properties of the
// (device, kernel) pair, so they are cached per device, not once per process.
int device_sms() {
  constexpr int MAXDEV = 64;
  static std::atomic<int> cache[MAXDEV];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= MAXDEV) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

cudaError_t ensure_smem_attr(const void* fptr, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_pair(dev, fptr);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
  }
  e = cudaFuncSetAttribute(fptr, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& v = done[key];
  if (v < bytes) v = bytes;
  return cudaSuccess;
}

}  // namespace fn

namespace {

thread_local char g_err[512] = "";
thread_local int64_t g_launches = 0;

fn_status fail(fn_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

fn_status cuda_fail(cudaError_t e, const char* where) {
  return fail(FN_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int elem_bytes(fn_dtype dt) { return dt == FN_BF16 ? 2 : 4; }

fn_status check_dtype(fn_dtype dt) {
  if (dt != FN_BF16 && dt != FN_F32) return fail(FN_ERR_DTYPE, "unknown fn_dtype %d", (int)dt);
  return FN_OK;
}

// K and N must allow 16-byte vector access of every row
fn_status check_vec(const char* what, int64_t v, fn_dtype dt) {
  const int64_t q = dt == FN_BF16 ? 8 : 4;
  if (v % q != 0)
    return fail(FN_ERR_ALIGN, "%s = %lld must be a multiple of %lld for %s (16-byte rows)", what, (long long)v,
                (long long)q, dt == FN_BF16 ? "bf16" : "f32");
  return FN_OK;
}

fn_status check_ptr16(const char* what, const void* p) {
  if (p != nullptr && !aligned16(p)) return fail(FN_ERR_ALIGN, "%s = %p is not 16-byte aligned", what, p);
  return FN_OK;
}

int num_sms() { return fn::device_sms(); }

bool fold_k2_cluster() {  // FN_K2_VARIANT=1: the cluster K2 (needs no workspace)
  const char* e = getenv("FN_K2_VARIANT");
  return e != nullptr && atoi(e) == 1;
}

bool debug_layernorm() {
  static const bool on = [] {
    const char* e = getenv("FN_DEBUG_LAYERNORM");
    return e != nullptr && atoi(e) != 0;
  }();
  return on;
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fnp = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fnp = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fnp;
}

std::mutex g_tmap_mu;
std::map<std::tuple<uintptr_t, int64_t, int64_t, int>, CUtensorMap> g_tmaps;

}  // namespace

namespace fn {
// plain (unswizzled) row-major 2-D map [rows][cols] of elem_bytes elements, box box_cols x box_rows
// (the fold kernels' TMA rings); false if the driver entry point is missing or the encode fails
bool encode_plain_tmap(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int elem_bytes, int box_cols,
                       int box_rows) {
  auto enc = encode_fn();
  if (enc == nullptr) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * elem_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(out, elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
             const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace fn

namespace {

// Plain (unswizzled) row-major maps for the fold kernels (box bytes x rows).
fn_status get_tmap_fold(const void* ptr, int64_t rows, int64_t cols, fn_dtype dtype, CUtensorMap* out,
                        int box_bytes = fn::FOLD_BOX_BYTES, int box_rows = fn::FOLD_BOX_ROWS) {
  const int eb = dtype == FN_BF16 ? 2 : 4;
  if (!fn::encode_plain_tmap(out, ptr, rows, cols, eb, box_bytes / eb, box_rows))
    return fail(FN_ERR_CUDA, "cuTensorMapEncodeTiled failed for fold map [%lld x %lld] (box %d B x %d rows)",
                (long long)rows, (long long)cols, box_bytes, box_rows);
  return FN_OK;
}

fn_status get_tmap(const void* ptr, int64_t rows, int64_t cols, int box_rows, CUtensorMap* out) {
  const auto key = std::make_tuple(reinterpret_cast<uintptr_t>(ptr), rows, cols, box_rows);
  std::lock_guard<std::mutex> lk(g_tmap_mu);
  auto it = g_tmaps.find(key);
  if (it != g_tmaps.end()) {
    *out = it->second;
    return FN_OK;
  }
  auto enc = encode_fn();
  if (enc == nullptr) return fail(FN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FN_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for [%lld x %lld] box %d", (int)r,
                (long long)rows, (long long)cols, box_rows);
  if (g_tmaps.size() > 4096) g_tmaps.clear();
  g_tmaps.emplace(key, m);
  *out = m;
  return FN_OK;
}

// 3-D view of a row-major bf16 [rows][cols] matrix (cols % 64 == 0) as {64, rows, cols / 64} with strides
// {cols * 2, 128} bytes: one box {64, box_rows, 2} is two consecutive SW128 [box_rows x 64] tiles of
// k blocks kb, kb + 1 (the decode kernel's 32 KiB stage); cached like get_tmap
fn_status get_tmap_kpair(const void* ptr, int64_t rows, int64_t cols, int box_rows, CUtensorMap* out) {
  const auto key = std::make_tuple(reinterpret_cast<uintptr_t>(ptr), rows, cols, 100000 + box_rows);
  std::lock_guard<std::mutex> lk(g_tmap_mu);
  auto it = g_tmaps.find(key);
  if (it != g_tmaps.end()) {
    *out = it->second;
    return FN_OK;
  }
  auto enc = encode_fn();
  if (enc == nullptr) return fail(FN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
  CUtensorMap m;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FN_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for the k-pair view of [%lld x %lld] box %d", (int)r,
                (long long)rows, (long long)cols, box_rows);
  if (g_tmaps.size() > 4096) g_tmaps.clear();
  g_tmaps.emplace(key, m);
  *out = m;
  return FN_OK;
}

int stg_enabled() {
  static const int on = [] {
    const char* e = getenv("FN_GEMM2_STG");  // A/B knob: 256-bit epilogue stores (1 = on)
    return e != nullptr ? atoi(e) : 1;
  }();
  return on;
}

// stream-K tail policy, read at every call (A/B knob FN_GEMM2_SK): 0 (default) off, 1 the
// mode-none kernel only (DyT pre-pass, plain GEMM), 2 also the RMS / LayerNorm-retrofit kernel.
// Measured on config 4: mode none within +-2% (constant data +2.5%, random data
// -1.5%, CUDA graphs), RMS -4..-7%: the partial traffic, the finisher fixups and the ssq group's
// per-item reductions cost as much as the 13% shorter MMA span saves.
// Default (no FN_GEMM2_SK in the environment): the mode-none kernel at K >= 8192, where the fixup is
// amortized over a long K — the FFN down projection 4096 x 14336 -> 4096 runs +2.7 % with it
// (profiles/r03g_ab_sk_ffn_down.txt); RMS never by default.
bool sk_allowed(int kernel_mode, int64_t K) {
  const char* e = getenv("FN_GEMM2_SK");
  if (e == nullptr) return kernel_mode == fn::MODE_NONE && K >= 8192;
  const int pol = atoi(e);
  return kernel_mode == fn::MODE_NONE ? pol >= 1 : (kernel_mode == fn::MODE_RMS && pol >= 2);
}

// stream-K scratch of a pair-kernel launch (0: the shape does not use it); `ws_off`: its offset in
// the caller's workspace (after the DyT pre-pass buffer, 256-B aligned)
// the stream-K flags live in the first 4 KiB of a linear workspace, always (zero between calls)
constexpr int64_t kSkFlagBytes = 4096;
int64_t sk_scratch(int64_t M, int64_t K, int64_t N, int bn, int* sk_tiles, int* sk_dp_waves) {
  const int mb = (int)((M + 255) / 256), nb = (int)((N + bn - 1) / bn);
  return fn::gemm2_sk_plan(mb * nb, (int)((K + 63) / 64), num_sms(), sk_tiles, sk_dp_waves);
}
int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }

int kernel_mode(fn_mode m) {
  switch (m) {
    case FN_RMSNORM:
    case FN_LAYERNORM: return fn::MODE_RMS;
    case FN_DYT: return fn::MODE_DYT;
    default: return fn::MODE_NONE;
  }
}

// Extras beyond flashnorm_linear: the GLU epilogue (NEXT-1) and a given per-row output scale.
struct LinearExtras {
  int glu_act = -1;                 // >= 0: gate||up GEMM with the GLU epilogue, z = h [M][N/2]
  float* s_out = nullptr;           // GLU: output scale per row
  const float* row_scale = nullptr; // FN_NONE: z = RN(acc * row_scale[m] + c*)
  fn::RopeParams rope{nullptr, nullptr, nullptr, 0, 0, 1.0f, nullptr, nullptr, 0, 0.f};  // RoPE on [0, rope.n)
  const float* ln_u = nullptr;      // exact deferred LayerNorm (rmsnorm mode): u = 1^T W* [N]
  int ndst = 0, ldz = 0, col0 = 0;  // fused column gather: z shard -> ndst [M x ldz] buffers at col0
  void* const* zdst = nullptr;
  int mc = 0;                       // zdst[0] is an NVLS multicast address (multimem.st)
};

fn_status linear_impl(const void* a, const void* Wt_star, const float* c_star, int64_t M, int64_t K, int64_t N,
                      float eps, float alpha, fn_mode mode, fn_dtype dtype, void* z, fn_path path,
                      void* workspace, int64_t workspace_bytes, cudaStream_t stream,
                      const LinearExtras& ex = LinearExtras()) {
  fn_status s;
  if ((s = check_dtype(dtype)) != FN_OK) return s;
  if (mode < FN_RMSNORM || mode > FN_NONE) return fail(FN_ERR_VALUE, "unknown fn_mode %d", (int)mode);
  if (M < 0 || K <= 0 || N <= 0)
    return fail(FN_ERR_SHAPE, "a[%lld x %lld], Wt_star[%lld x %lld]: sizes must be positive (M >= 0)",
                (long long)M, (long long)K, (long long)N, (long long)K);
  if (M > INT32_MAX || K > INT32_MAX || N > INT32_MAX)
    return fail(FN_ERR_SHAPE, "dimension exceeds int32 range: M=%lld K=%lld N=%lld", (long long)M, (long long)K,
                (long long)N);
  if (Wt_star == nullptr || ((a == nullptr || z == nullptr) && M > 0))
    return fail(FN_ERR_NULL, "a=%p Wt_star=%p z=%p: required pointer is NULL", a, Wt_star, z);
  if ((s = check_vec("K", K, dtype)) != FN_OK) return s;
  if ((s = check_vec("N", N, dtype)) != FN_OK) return s;
  if ((s = check_ptr16("a", a)) != FN_OK || (s = check_ptr16("Wt_star", Wt_star)) != FN_OK ||
      (s = check_ptr16("z", z)) != FN_OK || (s = check_ptr16("c_star", c_star)) != FN_OK)
    return s;
  if ((mode == FN_RMSNORM || mode == FN_LAYERNORM) && (!(eps >= 0.0f) || !std::isfinite(eps)))
    return fail(FN_ERR_VALUE, "eps = %g must be finite and >= 0", (double)eps);
  if (mode == FN_DYT && !std::isfinite(alpha)) return fail(FN_ERR_VALUE, "alpha = %g must be finite", (double)alpha);
  if (M == 0) return FN_OK;
  if (a == z) return fail(FN_ERR_VALUE, "z must not alias a");
  if (mode == FN_LAYERNORM && debug_layernorm()) {
    // the LayerNorm mode trusts a mean-centered input: verify it in debug runs
    float ratio = 0.f;
    cudaError_t e = fn::layernorm_center_check(a, M, K, dtype == FN_BF16 ? 0 : 1, stream, &ratio);
    if (e != cudaSuccess) return cuda_fail(e, "layernorm center check");
    ++g_launches;
    if (!(ratio <= 1e-2f))
      return fail(FN_ERR_VALUE, "FN_LAYERNORM input is not mean-centered: max |mean(a_m)|/rms(a_m) = %g > 1e-2 "
                                "(fold the centering into the preceding layer with flashnorm_fold_mean_center)",
                  (double)ratio);
  }
  int km = kernel_mode(mode);
  if (workspace != nullptr) {
    if ((s = check_ptr16("workspace", workspace)) != FN_OK) return s;
    if (workspace == z || workspace == a || workspace == Wt_star)
      return fail(FN_ERR_VALUE, "workspace must not alias a, Wt_star or z");
  }

  if (dtype == FN_F32) {
    if (path != FN_PATH_AUTO && path != FN_PATH_SIMT)
      return fail(FN_ERR_UNSUPPORTED, "f32 supports only the SIMT path (path=%d)", (int)path);
    cudaError_t e = fn::launch_linear_f32(static_cast<const float*>(a), static_cast<const float*>(Wt_star), c_star,
                                          static_cast<float*>(z), (int)M, (int)K, (int)N, eps, alpha, km, stream,
                                          ex.ln_u);
    if (e != cudaSuccess) return cuda_fail(e, "linear_f32");
    ++g_launches;
    return FN_OK;
  }

  // the GLU epilogue lives in the GEMM kernels; a given row scale in the GEMM and tcgen05 decode kernels
  // QK-norm on the decode kernel needs whole heads inside its 128-row tiles (h | 128, R = 1)
  const bool qkn_tc_ok = ex.rope.g_q == nullptr ||
                         (128 % ex.rope.h == 0 && fn::gemv_tc_tile_rows(fn::MODE_RMS, (int)K, (int)N, num_sms()) == 128);
  // the exact deferred LayerNorm (ln_u) lives in the GEMM kernels only: decode shapes run the
  // 1-CTA tcgen05 kernel
  const bool tc_ok = ex.glu_act < 0 && ex.ln_u == nullptr && ex.ndst == 0 && qkn_tc_ok &&
                     fn::gemv_tc_supported((int)M, (int)N, num_sms());
  const bool mma_ok = ex.glu_act < 0 && ex.ln_u == nullptr && ex.ndst == 0 && ex.row_scale == nullptr &&
                      ex.rope.pos == nullptr &&
                      fn::gemv_supported((int)M, (int)K);
  const bool gemv_ok = tc_ok || mma_ok;
  if (path == FN_PATH_SIMT) return fail(FN_ERR_UNSUPPORTED, "SIMT path is f32-only");
  // batched decode, 17 <= M <= 128 (K4w): the swap-AB tcgen05 kernel with the tokens as the MMA N
  // DyT takes its tanh pre-pass (K8) into the caller's workspace, then runs in mode none
  const int64_t dyt_ws_off = align256(kSkFlagBytes);
  const bool wide_dyt = km == fn::MODE_DYT && workspace != nullptr && workspace_bytes >= dyt_ws_off + M * K * 2;
  const int km_wide = wide_dyt ? fn::MODE_NONE : km;
  const bool wide_ok = (path == FN_PATH_AUTO || path == FN_PATH_GEMV) && !gemv_ok && ex.glu_act < 0 &&
                       ex.ln_u == nullptr && ex.ndst == 0 &&
                       (ex.rope.pos == nullptr ||
                        (km_wide == fn::MODE_RMS && (ex.rope.g_q == nullptr || 128 % ex.rope.h == 0))) &&
                       (ex.row_scale == nullptr || km_wide == fn::MODE_NONE) &&
                       (km_wide == fn::MODE_RMS || km_wide == fn::MODE_NONE) &&
                       fn::gemv_wide_supported(km_wide, (int)M, (int)K, (int)N, num_sms());
  if (wide_ok) {
    if (wide_dyt) {
      void* ybuf = static_cast<uint8_t*>(workspace) + dyt_ws_off;
      cudaError_t e = fn::launch_dyt_prepass(static_cast<const __nv_bfloat16*>(a), static_cast<__nv_bfloat16*>(ybuf),
                                             M * K, alpha, num_sms(), stream);
      if (e != cudaSuccess) return cuda_fail(e, "dyt_prepass");
      ++g_launches;
      a = ybuf;
      km = fn::MODE_NONE;
    }
    CUtensorMap tw, ta;
    if ((s = get_tmap(Wt_star, N, K, 128, &tw)) != FN_OK) return s;
    if ((s = get_tmap(a, M, K, fn::gemv_wide_tokens((int)M), &ta)) != FN_OK) return s;
    cudaError_t e = fn::launch_gemv_wide(tw, ta, c_star, static_cast<__nv_bfloat16*>(z), (int)M, (int)K, (int)N, eps,
                                         km, num_sms(), stream, static_cast<const __nv_bfloat16*>(a), ex.row_scale,
                                         ex.rope);
    if (e != cudaSuccess) return cuda_fail(e, "gemv_wide");
    ++g_launches;
    return FN_OK;
  }
  if ((path == FN_PATH_GEMV && !gemv_ok) || (path == FN_PATH_GEMV_MMA && !mma_ok))
    return fail(FN_ERR_UNSUPPORTED, "decode path needs M <= 16 (or 17..128 for the batched-decode kernel: rmsnorm / layernorm / none, N <= 128 x #SMs) (M=%lld K=%lld)",
                (long long)M, (long long)K);
  const bool use_gemv = path == FN_PATH_GEMV || path == FN_PATH_GEMV_MMA || (path == FN_PATH_AUTO && gemv_ok);
  if (use_gemv && path != FN_PATH_GEMV_MMA && tc_ok) {
    CUtensorMap tw, ta;
    const int trows = std::min(fn::gemv_tc_tile_rows(km, (int)K, (int)N, num_sms()), 256);  // TMA box rows
    if (fn::gemv_tc_kblocks(km, (int)K, (int)N, num_sms()) == 2) {
      if ((s = get_tmap_kpair(Wt_star, N, K, trows, &tw)) != FN_OK) return s;
      if ((s = get_tmap_kpair(a, M, K, 16, &ta)) != FN_OK) return s;
    } else {
      if ((s = get_tmap(Wt_star, N, K, trows, &tw)) != FN_OK) return s;
      if ((s = get_tmap(a, M, K, 16, &ta)) != FN_OK) return s;
    }
    cudaError_t e = fn::launch_gemv_tc(tw, ta, c_star, static_cast<__nv_bfloat16*>(z), (int)M, (int)K, (int)N, eps,
                                       alpha, km, num_sms(), stream, ex.row_scale, ex.rope,
                                       static_cast<const __nv_bfloat16*>(Wt_star), static_cast<const __nv_bfloat16*>(a));
    if (e != cudaSuccess) return cuda_fail(e, "gemv_tc");
    ++g_launches;
    return FN_OK;
  }
  if (use_gemv) {
    cudaError_t e = fn::launch_gemv(static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(Wt_star),
                                    c_star, static_cast<__nv_bfloat16*>(z), (int)M, (int)K, (int)N, eps, alpha, km,
                                    num_sms(), stream);
    if (e != cudaSuccess) return cuda_fail(e, "gemv");
    ++g_launches;
    return FN_OK;
  }
  // Workspace layout (include/flashnorm.h flashnorm_linear_ws): [4 KiB stream-K flags][stream-K fp32
  // partials][DyT pre-pass buffer].  DyT with a workspace: K8 computes tanh(alpha a) once per element
  // (dyt.cu explains why the in-SMEM prologue is MUFU-bound), then the GEMM runs in mode NONE on it —
  // bit-identical z.
  int launches = 1;
  const bool prepass = km == fn::MODE_DYT && workspace != nullptr;
  const int km_gemm = prepass ? fn::MODE_NONE : km;
  // CTA-pair (cta_group::2, 256x256 tiles) kernel when M > 128; the 1-CTA kernel for M <= 128
  // and FN_PATH_GEMM1.
  const bool pair = M > 128 && (path != FN_PATH_GEMM1);
  // 224-wide pair tiles when they even out the last wave (plain / LayerNorm / scaled / gather
  // epilogues; GLU, RoPE and QK-norm keep their 256-column tile algebra, DyT its prologue)
  const bool allow_224 = km_gemm != fn::MODE_DYT && ex.glu_act < 0 && ex.rope.pos == nullptr;
  const int bn = pair ? fn::gemm2_pick_bn((int)M, (int)N, num_sms(), allow_224) : 256;
  // stream-K tail (pair kernel, plain RMS / LayerNorm-retrofit / none epilogues) when the caller's
  // workspace holds its scratch (flashnorm_linear_workspace_bytes counts it)
  int sk_tiles = 0, sk_waves = 0;
  int64_t sk_bytes = 0;
  if (pair && sk_allowed(km_gemm, K) && workspace != nullptr &&
      (km_gemm == fn::MODE_NONE || (km_gemm == fn::MODE_RMS && ex.ln_u == nullptr)) && ex.glu_act < 0 &&
      ex.rope.pos == nullptr && ex.ndst == 0)
    sk_bytes = sk_scratch(M, K, N, bn, &sk_tiles, &sk_waves);
  const int64_t dyt_off = (workspace != nullptr) ? align256(kSkFlagBytes + sk_bytes) : 0;
  if (workspace != nullptr && (sk_bytes > 0 || prepass) &&
      workspace_bytes < dyt_off + (prepass ? M * K * 2 : 0)) {
    sk_tiles = 0;  // too small for the stream-K scratch: whole tiles only
    sk_bytes = 0;
  }
  if (prepass) {
    const int64_t off = align256(kSkFlagBytes + sk_bytes);
    if (workspace_bytes < off + M * K * 2)
      return fail(FN_ERR_VALUE, "workspace_bytes = %lld < %lld (flashnorm_linear_workspace_bytes)",
                  (long long)workspace_bytes, (long long)(off + M * K * 2));
    void* ybuf = static_cast<uint8_t*>(workspace) + off;
    cudaError_t e = fn::launch_dyt_prepass(static_cast<const __nv_bfloat16*>(a), static_cast<__nv_bfloat16*>(ybuf),
                                           M * K, alpha, num_sms(), stream);
    if (e != cudaSuccess) return cuda_fail(e, "dyt_prepass");
    a = ybuf;
    km = fn::MODE_NONE;
    launches = 2;
  }
  CUtensorMap ta, tb;
  if ((s = get_tmap(a, M, K, 128, &ta)) != FN_OK) return s;
  if ((s = get_tmap(Wt_star, N, K, pair ? bn / 2 : 256, &tb)) != FN_OK) return s;
  fn::GemmParams p;
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.num_m_blocks = (int)(pair ? (M + 255) / 256 : (M + 127) / 128);
  p.num_n_blocks = (int)((N + bn - 1) / bn);
  p.bn = bn;
  // RMS / exact-LayerNorm side group reads each CTA's A stage after its OWN TMA barrier (afull), the
  // ordering the memory model states directly; FN_GEMM2_RMS_LOCAL=0 restores the older order (after
  // the leader's multicast MMA commit), ~1 % faster but ordered only through the MMA's own reads
  // (tools/ab_local.sh, profiles/r02q_ab_local.txt)
  static const int rms_local = [] {
    const char* e = getenv("FN_GEMM2_RMS_LOCAL");
    return e != nullptr ? atoi(e) : 1;
  }();
  p.rms_local = rms_local;
  static const int tile_rot = [] {
    const char* e = getenv("FN_GEMM2_TILE_ROT");  // A/B knob: 0 plain stride, 1 rotated, 2 matched table
    return e != nullptr ? atoi(e) : 2;
  }();
  p.tile_rot = tile_rot;
  p.num_tiles = p.num_m_blocks * p.num_n_blocks;
  {  // ~40 MB of A per tile group (L2 is 126 MB; W* tiles and z share it)
    const int64_t a_bytes_per_blk = (pair ? 256 : 128) * K * 2;
    static const int64_t group_mb = [] {
      const char* e = getenv("FN_GEMM2_GROUP_MB");  // A/B knob: A bytes per tile group, MiB
      return (int64_t)(e != nullptr ? atoi(e) : 40);
    }();
    int64_t G = (group_mb << 20) / a_bytes_per_blk;
    if (G < 1) G = 1;
    if (G > p.num_m_blocks) G = p.num_m_blocks;
    static const int balance = [] {
      const char* e = getenv("FN_GEMM2_GROUP_BAL");  // A/B knob: equal-sized tile groups
      return e != nullptr ? atoi(e) : 1;
    }();
    if (balance) {  // same group count, sizes differing by at most one block (no short last group)
      const int64_t ngroups = (p.num_m_blocks + G - 1) / G;
      G = (p.num_m_blocks + ngroups - 1) / ngroups;
    }
    p.group_m = (int)G;
  }
  p.num_k_blocks = (int)((K + 63) / 64);
  p.eps = eps;
  p.alpha = alpha;
  p.cstar = c_star;
  p.z = static_cast<__nv_bfloat16*>(z);
  p.a = static_cast<const __nv_bfloat16*>(a);
  p.glu_act = ex.glu_act;
  p.s_out = ex.s_out;
  p.row_scale = ex.row_scale;
  p.rope = ex.rope;
  p.ln_u = ex.ln_u;
  p.ndst = ex.ndst;
  p.mc = ex.mc;
  p.stg = stg_enabled();
  p.ldz = ex.ldz;
  p.col0 = ex.col0;
  for (int d = 0; d < fn::MAX_GATHER_DST; ++d)
    p.zdst[d] = d < ex.ndst ? static_cast<__nv_bfloat16*>(ex.zdst[d]) : nullptr;
  p.sk_tiles = sk_bytes > 0 ? sk_tiles : 0;
  p.sk_dp_waves = sk_waves;
  p.sk_flag = sk_bytes > 0 ? static_cast<unsigned*>(workspace) : nullptr;
  p.sk_part = sk_bytes > 0 ? reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + kSkFlagBytes) : nullptr;
  cudaError_t e = pair ? fn::launch_gemm2(ta, tb, p, km, num_sms(), stream)
                       : fn::launch_gemm(ta, tb, p, km, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, pair ? "gemm2_sm100" : "gemm_sm100");
  g_launches += launches;
  return FN_OK;
}

}  // namespace

namespace fn {
// error text for the other translation units of the C ABI (comm.cu)
fn_status api_fail(fn_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}
}  // namespace fn

extern "C" {

fn_status flashnorm_fold_weights(const void* Wt, int64_t N, int64_t K, fn_dtype dtype, const float* g,
                                 const float* b, const float* c, void* Wt_star, float* c_star, void* stream) {
  fn_status s;
  if ((s = check_dtype(dtype)) != FN_OK) return s;
  if (N <= 0 || K <= 0) return fail(FN_ERR_SHAPE, "Wt[%lld x %lld]: sizes must be positive", (long long)N, (long long)K);
  if (Wt == nullptr || Wt_star == nullptr) return fail(FN_ERR_NULL, "Wt=%p Wt_star=%p: NULL", Wt, Wt_star);
  if ((b != nullptr || c != nullptr) && c_star == nullptr)
    return fail(FN_ERR_NULL, "c_star is NULL but b=%p / c=%p given", (const void*)b, (const void*)c);
  if ((s = check_vec("K", K, dtype)) != FN_OK) return s;
  if ((s = check_ptr16("Wt", Wt)) != FN_OK || (s = check_ptr16("Wt_star", Wt_star)) != FN_OK ||
      (s = check_ptr16("g", g)) != FN_OK || (s = check_ptr16("b", b)) != FN_OK)
    return s;
  if (Wt == Wt_star) return fail(FN_ERR_VALUE, "Wt_star must not alias Wt");
  cudaError_t e = fn::launch_fold_weights(Wt, N, K, dtype == FN_BF16 ? 0 : 1, g, b, c, Wt_star, c_star,
                                          static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fold_weights");
  ++g_launches;
  return FN_OK;
}

int64_t flashnorm_fold_mean_center_workspace_bytes(int64_t n_out, int64_t d_in) {
  if (n_out <= 0 || d_in <= 0) return 0;
  return fn::fold_mean_center_workspace(n_out, d_in);
}

fn_status flashnorm_fold_mean_center(const void* Vt, int64_t n_out, int64_t d_in, fn_dtype dtype,
                                     const float* b_prev, void* Vt_star, float* b_prev_star, void* workspace,
                                     void* stream) {
  fn_status s;
  if ((s = check_dtype(dtype)) != FN_OK) return s;
  if (n_out <= 0 || d_in <= 0)
    return fail(FN_ERR_SHAPE, "Vt[%lld x %lld]: sizes must be positive", (long long)n_out, (long long)d_in);
  if (Vt == nullptr || Vt_star == nullptr)
    return fail(FN_ERR_NULL, "Vt=%p Vt_star=%p: NULL", Vt, Vt_star);
  if (workspace == nullptr && flashnorm_fold_mean_center_workspace_bytes(n_out, d_in) > 0 &&
      !fold_k2_cluster())
    return fail(FN_ERR_NULL, "workspace is NULL (flashnorm_fold_mean_center_workspace_bytes = %lld)",
                (long long)flashnorm_fold_mean_center_workspace_bytes(n_out, d_in));
  if ((b_prev == nullptr) != (b_prev_star == nullptr))
    return fail(FN_ERR_NULL, "b_prev=%p and b_prev_star=%p must be both NULL or both set", (const void*)b_prev,
                (const void*)b_prev_star);
  if ((s = check_vec("d_in", d_in, dtype)) != FN_OK) return s;
  if ((s = check_ptr16("Vt", Vt)) != FN_OK || (s = check_ptr16("Vt_star", Vt_star)) != FN_OK ||
      (s = check_ptr16("workspace", workspace)) != FN_OK)
    return s;
  if (Vt == Vt_star) return fail(FN_ERR_VALUE, "Vt_star must not alias Vt");
  if (n_out > INT32_MAX || d_in > INT32_MAX)
    return fail(FN_ERR_SHAPE, "Vt[%lld x %lld]: dimension exceeds int32 range", (long long)n_out, (long long)d_in);
  CUtensorMap tm3, tm, tms;
  if ((s = get_tmap_fold(Vt, n_out, d_in, dtype, &tm3, 512, 32)) != FN_OK) return s;
  if ((s = get_tmap_fold(Vt, n_out, d_in, dtype, &tm)) != FN_OK) return s;
  if ((s = get_tmap_fold(Vt_star, n_out, d_in, dtype, &tms)) != FN_OK) return s;
  int launches = 0;
  cudaError_t e = fn::launch_fold_mean_center(tm3, tm, tms, Vt, n_out, d_in, dtype == FN_BF16 ? 0 : 1, b_prev, Vt_star,
                                              b_prev_star, workspace, static_cast<cudaStream_t>(stream), &launches);
  if (e != cudaSuccess) return cuda_fail(e, "fold_mean_center");
  g_launches += launches;
  return FN_OK;
}

fn_status flashnorm_linear(const void* a, const void* Wt_star, const float* c_star, int64_t M, int64_t K, int64_t N,
                           float eps, float alpha, fn_mode mode, fn_dtype dtype, void* z, void* stream) {
  return linear_impl(a, Wt_star, c_star, M, K, N, eps, alpha, mode, dtype, z, FN_PATH_AUTO, nullptr, 0,
                     static_cast<cudaStream_t>(stream));
}

fn_status flashnorm_linear_ex(const void* a, const void* Wt_star, const float* c_star, int64_t M, int64_t K,
                              int64_t N, float eps, float alpha, fn_mode mode, fn_dtype dtype, void* z, fn_path path,
                              void* stream) {
  if (path < FN_PATH_AUTO || path > FN_PATH_GEMV_MMA) return fail(FN_ERR_VALUE, "unknown fn_path %d", (int)path);
  return linear_impl(a, Wt_star, c_star, M, K, N, eps, alpha, mode, dtype, z, path, nullptr, 0,
                     static_cast<cudaStream_t>(stream));
}

int64_t flashnorm_linear_workspace_bytes(int64_t M, int64_t K, int64_t N, fn_mode mode, fn_dtype dtype,
                                         fn_path path) {
  if (dtype != FN_BF16 || M <= 0 || K <= 0 || N <= 0) return 0;
  if (path == FN_PATH_GEMV || path == FN_PATH_GEMV_MMA || path == FN_PATH_SIMT) return 0;
  const bool gemv_ok = fn::gemv_tc_supported((int)M, (int)N, num_sms()) || fn::gemv_supported((int)M, (int)K);
  if (path == FN_PATH_AUTO && gemv_ok) return 0;  // decode: tanh is computed once per CTA anyway
  // the pair kernel's stream-K scratch (same decision as linear_impl; DyT runs it in mode none)
  int64_t sk = 0;
  const bool pair = M > 128 && path != FN_PATH_GEMM1;
  const int km = (mode == FN_RMSNORM || mode == FN_LAYERNORM) ? fn::MODE_RMS : fn::MODE_NONE;  // DyT: pre-pass + none
  if (pair && sk_allowed(km, K)) {
    const int bn = fn::gemm2_pick_bn((int)M, (int)N, num_sms(), true);
    int skt = 0, skw = 0;
    sk = sk_scratch(M, K, N, bn, &skt, &skw);
  }
  if (sk == 0 && mode != FN_DYT) return 0;
  return align256(kSkFlagBytes + sk) + (mode == FN_DYT ? M * K * 2 : 0);
}

fn_status flashnorm_linear_ws(const void* a, const void* Wt_star, const float* c_star, int64_t M, int64_t K,
                              int64_t N, float eps, float alpha, fn_mode mode, fn_dtype dtype, void* z, fn_path path,
                              void* workspace, int64_t workspace_bytes, void* stream) {
  if (path < FN_PATH_AUTO || path > FN_PATH_GEMV_MMA) return fail(FN_ERR_VALUE, "unknown fn_path %d", (int)path);
  if (workspace == nullptr && workspace_bytes != 0)
    return fail(FN_ERR_NULL, "workspace is NULL but workspace_bytes = %lld", (long long)workspace_bytes);
  return linear_impl(a, Wt_star, c_star, M, K, N, eps, alpha, mode, dtype, z, path, workspace, workspace_bytes,
                     static_cast<cudaStream_t>(stream));
}

fn_status flashnorm_fold_colsum(const void* Wt_star, int64_t N, int64_t K, fn_dtype dtype, float* u, void* stream) {
  fn_status s;
  if ((s = check_dtype(dtype)) != FN_OK) return s;
  if (N <= 0 || K <= 0)
    return fail(FN_ERR_SHAPE, "Wt_star[%lld x %lld]: sizes must be positive", (long long)N, (long long)K);
  if (Wt_star == nullptr || u == nullptr) return fail(FN_ERR_NULL, "Wt_star=%p u=%p: NULL", Wt_star, (void*)u);
  if ((s = check_vec("K", K, dtype)) != FN_OK) return s;
  if ((s = check_ptr16("Wt_star", Wt_star)) != FN_OK) return s;
  cudaError_t e = fn::launch_fold_colsum(Wt_star, N, K, dtype == FN_BF16 ? 0 : 1, u, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fold_colsum");
  ++g_launches;
  return FN_OK;
}

fn_status flashnorm_layernorm_linear(const void* a, const void* Wt_star, const float* u, const float* c_star,
                                     int64_t M, int64_t K, int64_t N, float eps, fn_dtype dtype, void* z,
                                     void* stream) {
  if (u == nullptr) return fail(FN_ERR_NULL, "u (column sums of W*) is NULL");
  fn_status s;
  if ((s = check_ptr16("u", u)) != FN_OK) return s;
  LinearExtras ex;
  ex.ln_u = u;
  return linear_impl(a, Wt_star, c_star, M, K, N, eps, 0.0f, FN_RMSNORM, dtype, z, FN_PATH_AUTO, nullptr, 0,
                     static_cast<cudaStream_t>(stream), ex);
}

fn_status flashnorm_linear_gather(const void* a, const void* Wt_star, const float* c_star, int64_t M, int64_t K,
                                  int64_t N, float eps, float alpha, fn_mode mode, fn_dtype dtype,
                                  void* const* z_dsts, int ndst, int64_t ldz, int64_t col0, void* stream) {
  if (dtype != FN_BF16) return fail(FN_ERR_UNSUPPORTED, "flashnorm_linear_gather is bf16-only");
  if (ndst < 1 || ndst > fn::MAX_GATHER_DST)
    return fail(FN_ERR_VALUE, "ndst = %d must be in [1, %d]", ndst, fn::MAX_GATHER_DST);
  if (z_dsts == nullptr) return fail(FN_ERR_NULL, "z_dsts is NULL");
  if (col0 < 0 || ldz < col0 + N || ldz > INT32_MAX)
    return fail(FN_ERR_SHAPE, "shard columns [%lld, %lld) do not fit rows of ldz = %lld", (long long)col0,
                (long long)(col0 + N), (long long)ldz);
  if (ldz % 8 != 0 || col0 % 8 != 0)
    return fail(FN_ERR_ALIGN, "ldz = %lld and col0 = %lld must be multiples of 8 (16-byte rows)", (long long)ldz,
                (long long)col0);
  fn_status s;
  for (int d = 0; d < ndst; ++d) {
    if (z_dsts[d] == nullptr) return fail(FN_ERR_NULL, "z_dsts[%d] is NULL", d);
    if ((s = check_ptr16("z_dsts[d]", z_dsts[d])) != FN_OK) return s;
    if (z_dsts[d] == a) return fail(FN_ERR_VALUE, "z_dsts[%d] aliases a", d);
  }
  LinearExtras ex;
  ex.ndst = ndst;
  ex.ldz = (int)ldz;
  ex.col0 = (int)col0;
  ex.zdst = z_dsts;
  // z (the plain output) is unused on this path: pass the first destination for the checks
  return linear_impl(a, Wt_star, c_star, M, K, N, eps, alpha, mode, dtype, z_dsts[0], FN_PATH_GEMM, nullptr, 0,
                     static_cast<cudaStream_t>(stream), ex);
}

fn_status flashnorm_linear_gather_multicast(const void* a, const void* Wt_star, const float* c_star, int64_t M,
                                            int64_t K, int64_t N, float eps, float alpha, fn_mode mode,
                                            fn_dtype dtype, void* z_mc, int64_t ldz, int64_t col0, void* stream) {
  if (dtype != FN_BF16) return fail(FN_ERR_UNSUPPORTED, "flashnorm_linear_gather_multicast is bf16-only");
  if (z_mc == nullptr) return fail(FN_ERR_NULL, "z_mc is NULL");
  if (col0 < 0 || ldz < col0 + N || ldz > INT32_MAX)
    return fail(FN_ERR_SHAPE, "shard columns [%lld, %lld) do not fit rows of ldz = %lld", (long long)col0,
                (long long)(col0 + N), (long long)ldz);
  if (ldz % 8 != 0 || col0 % 8 != 0)
    return fail(FN_ERR_ALIGN, "ldz = %lld and col0 = %lld must be multiples of 8 (16-byte rows)", (long long)ldz,
                (long long)col0);
  fn_status s;
  if ((s = check_ptr16("z_mc", z_mc)) != FN_OK) return s;
  if (z_mc == a) return fail(FN_ERR_VALUE, "z_mc aliases a");
  void* dsts[1] = {z_mc};
  LinearExtras ex;
  ex.ndst = 1;
  ex.ldz = (int)ldz;
  ex.col0 = (int)col0;
  ex.zdst = dsts;
  ex.mc = 1;
  return linear_impl(a, Wt_star, c_star, M, K, N, eps, alpha, mode, dtype, z_mc, FN_PATH_GEMM, nullptr, 0,
                     static_cast<cudaStream_t>(stream), ex);
}

fn_status flashnorm_linear_scaled(const void* a, const void* Wt_star, const float* c_star, const float* row_scale,
                                  int64_t M, int64_t K, int64_t N, fn_dtype dtype, void* z, void* stream) {
  if (dtype != FN_BF16) return fail(FN_ERR_UNSUPPORTED, "flashnorm_linear_scaled is bf16-only");
  if (row_scale == nullptr && M > 0) return fail(FN_ERR_NULL, "row_scale is NULL");
  fn_status s;
  if ((s = check_ptr16("row_scale", row_scale)) != FN_OK) return s;
  LinearExtras ex;
  ex.row_scale = row_scale;
  return linear_impl(a, Wt_star, c_star, M, K, N, 0.0f, 0.0f, FN_NONE, dtype, z, FN_PATH_AUTO, nullptr, 0,
                     static_cast<cudaStream_t>(stream), ex);
}

fn_status flashnorm_linear_scaled_ws(const void* a, const void* Wt_star, const float* c_star, const float* row_scale,
                                     int64_t M, int64_t K, int64_t N, fn_dtype dtype, void* z, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  if (dtype != FN_BF16) return fail(FN_ERR_UNSUPPORTED, "flashnorm_linear_scaled is bf16-only");
  if (row_scale == nullptr && M > 0) return fail(FN_ERR_NULL, "row_scale is NULL");
  if (workspace == nullptr && workspace_bytes != 0)
    return fail(FN_ERR_NULL, "workspace is NULL but workspace_bytes = %lld", (long long)workspace_bytes);
  fn_status s;
  if ((s = check_ptr16("row_scale", row_scale)) != FN_OK) return s;
  LinearExtras ex;
  ex.row_scale = row_scale;
  return linear_impl(a, Wt_star, c_star, M, K, N, 0.0f, 0.0f, FN_NONE, dtype, z, FN_PATH_AUTO, workspace,
                     workspace_bytes, static_cast<cudaStream_t>(stream), ex);
}

fn_status flashnorm_qkv_rope_linear(const void* a, const void* Wt_star, int64_t M, int64_t K, int64_t N,
                                    int64_t n_rope, int64_t head_dim, const int32_t* positions, const float* cos_tab,
                                    const float* sin_tab, float qk_scale, float eps, fn_dtype dtype, void* z,
                                    void* stream) {
  if (dtype != FN_BF16) return fail(FN_ERR_UNSUPPORTED, "flashnorm_qkv_rope_linear is bf16-only");
  if (head_dim <= 0 || head_dim % 2 != 0 || head_dim > 65536)
    return fail(FN_ERR_SHAPE, "head_dim = %lld must be even and positive", (long long)head_dim);
  if (n_rope < 0 || n_rope > N || n_rope % head_dim != 0 || n_rope % 32 != 0)
    return fail(FN_ERR_SHAPE, "n_rope = %lld must be a multiple of head_dim (%lld) and of 32, <= N = %lld",
                (long long)n_rope, (long long)head_dim, (long long)N);
  if (M > 0 && n_rope > 0 && (positions == nullptr || cos_tab == nullptr || sin_tab == nullptr))
    return fail(FN_ERR_NULL, "positions=%p cos_tab=%p sin_tab=%p: NULL", (const void*)positions,
                (const void*)cos_tab, (const void*)sin_tab);
  if (!std::isfinite(qk_scale)) return fail(FN_ERR_VALUE, "qk_scale = %g must be finite", (double)qk_scale);
  LinearExtras ex;
  if (n_rope > 0)
    ex.rope = fn::RopeParams{positions, cos_tab, sin_tab, (int)n_rope, (int)head_dim, qk_scale, nullptr, nullptr, 0, 0.f};
  return linear_impl(a, Wt_star, nullptr, M, K, N, eps, 0.0f, FN_RMSNORM, dtype, z, FN_PATH_AUTO, nullptr, 0,
                     static_cast<cudaStream_t>(stream), ex);
}

fn_status flashnorm_qk_norm_rope_linear(const void* a, const void* Wt_star, int64_t M, int64_t K, int64_t N,
                                       int64_t n_q, int64_t n_k, int64_t head_dim, const float* g_q,
                                       const float* g_k, float eps_qk, const int32_t* positions,
                                       const float* cos_tab, const float* sin_tab, float qk_scale, float eps,
                                       fn_dtype dtype, void* z, void* stream) {
  if (dtype != FN_BF16) return fail(FN_ERR_UNSUPPORTED, "flashnorm_qk_norm_rope_linear is bf16-only");
  if (head_dim != 32 && head_dim != 64 && head_dim != 128 && head_dim != 256)
    return fail(FN_ERR_SHAPE, "head_dim = %lld must be 32, 64, 128 or 256", (long long)head_dim);
  if (n_q < 0 || n_k < 0 || n_q % head_dim != 0 || n_k % head_dim != 0 || n_q + n_k > N)
    return fail(FN_ERR_SHAPE, "n_q = %lld, n_k = %lld must be multiples of head_dim (%lld) with n_q + n_k <= N = %lld",
                (long long)n_q, (long long)n_k, (long long)head_dim, (long long)N);
  if (M > 0 && n_q + n_k > 0 &&
      (positions == nullptr || cos_tab == nullptr || sin_tab == nullptr || g_q == nullptr || g_k == nullptr))
    return fail(FN_ERR_NULL, "positions / cos_tab / sin_tab / g_q / g_k must not be NULL");
  fn_status s;
  if ((s = check_ptr16("g_q", g_q)) != FN_OK || (s = check_ptr16("g_k", g_k)) != FN_OK ||
      (s = check_ptr16("cos_tab", cos_tab)) != FN_OK || (s = check_ptr16("sin_tab", sin_tab)) != FN_OK)
    return s;
  if (!std::isfinite(qk_scale) || !(eps_qk >= 0.0f) || !std::isfinite(eps_qk))
    return fail(FN_ERR_VALUE, "qk_scale = %g, eps_qk = %g: must be finite (eps_qk >= 0)", (double)qk_scale,
                (double)eps_qk);
  LinearExtras ex;
  if (n_q + n_k > 0)
    ex.rope = fn::RopeParams{positions, cos_tab, sin_tab, (int)(n_q + n_k), (int)head_dim, qk_scale,
                             g_q, g_k, (int)n_q, eps_qk};
  return linear_impl(a, Wt_star, nullptr, M, K, N, eps, 0.0f, FN_RMSNORM, dtype, z, FN_PATH_AUTO, nullptr, 0,
                     static_cast<cudaStream_t>(stream), ex);
}

fn_status flashnorm_relu_ffn_up(const void* a, const void* Wt_star, int64_t M, int64_t K, int64_t F, float eps,
                                fn_dtype dtype, void* h, float* s_out, void* stream) {
  if (dtype != FN_BF16) return fail(FN_ERR_UNSUPPORTED, "flashnorm_relu_ffn_up is bf16-only");
  if (s_out == nullptr && M > 0) return fail(FN_ERR_NULL, "s_out is NULL");
  fn_status s;
  if ((s = check_ptr16("s_out", s_out)) != FN_OK) return s;
  LinearExtras ex;
  ex.glu_act = fn::RELU_FFN;
  ex.s_out = s_out;
  return linear_impl(a, Wt_star, nullptr, M, K, F, eps, 0.0f, FN_RMSNORM, dtype, h, FN_PATH_AUTO, nullptr, 0,
                     static_cast<cudaStream_t>(stream), ex);
}

fn_status flashnorm_fold_glu_weights(const void* Wgt, const void* Wut, int64_t F, int64_t K, fn_dtype dtype,
                                     const float* g, void* Wgu_star, void* stream) {
  fn_status s;
  if ((s = check_dtype(dtype)) != FN_OK) return s;
  if (F <= 0 || K <= 0) return fail(FN_ERR_SHAPE, "Wgt/Wut[%lld x %lld]: sizes must be positive", (long long)F,
                                    (long long)K);
  if (F % 128 != 0) return fail(FN_ERR_SHAPE, "F = %lld must be a multiple of 128 (gate/up interleave)", (long long)F);
  if (Wgt == nullptr || Wut == nullptr || Wgu_star == nullptr)
    return fail(FN_ERR_NULL, "Wgt=%p Wut=%p Wgu_star=%p: NULL", Wgt, Wut, Wgu_star);
  if ((s = check_vec("K", K, dtype)) != FN_OK) return s;
  if ((s = check_ptr16("Wgt", Wgt)) != FN_OK || (s = check_ptr16("Wut", Wut)) != FN_OK ||
      (s = check_ptr16("Wgu_star", Wgu_star)) != FN_OK || (s = check_ptr16("g", g)) != FN_OK)
    return s;
  if (Wgu_star == Wgt || Wgu_star == Wut) return fail(FN_ERR_VALUE, "Wgu_star must not alias Wgt / Wut");
  const int dt = dtype == FN_BF16 ? 0 : 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = fn::launch_fold_weights(Wgt, F, K, dt, g, nullptr, nullptr, Wgu_star, nullptr, st, 0);
  if (e == cudaSuccess) e = fn::launch_fold_weights(Wut, F, K, dt, g, nullptr, nullptr, Wgu_star, nullptr, st, 1);
  if (e != cudaSuccess) return cuda_fail(e, "fold_glu_weights");
  g_launches += 2;
  return FN_OK;
}

fn_status flashnorm_glu_linear(const void* a, const void* Wgu_star, int64_t M, int64_t K, int64_t F, float eps,
                               fn_glu_act act, fn_dtype dtype, void* h, float* s_out, void* stream) {
  if (dtype != FN_BF16) return fail(FN_ERR_UNSUPPORTED, "flashnorm_glu_linear is bf16-only");
  if (act < FN_GLU_SILU || act > FN_GLU_BILINEAR) return fail(FN_ERR_VALUE, "unknown fn_glu_act %d", (int)act);
  if (F <= 0 || F % 128 != 0)
    return fail(FN_ERR_SHAPE, "F = %lld must be a positive multiple of 128 (gate/up interleave)", (long long)F);
  if (s_out == nullptr && M > 0) return fail(FN_ERR_NULL, "s_out is NULL");
  fn_status s;
  if ((s = check_ptr16("s_out", s_out)) != FN_OK) return s;
  if (h != nullptr && (h == a || h == Wgu_star)) return fail(FN_ERR_VALUE, "h must not alias a or Wgu_star");
  LinearExtras ex;
  ex.glu_act = (int)act;
  ex.s_out = s_out;
  // the GEMM over the interleaved [2F][K] weights; z = h is [M][F]
  return linear_impl(a, Wgu_star, nullptr, M, K, 2 * F, eps, 0.0f, FN_RMSNORM, dtype, h, FN_PATH_AUTO, nullptr, 0,
                     static_cast<cudaStream_t>(stream), ex);
}

namespace {
// copy streams + events of the end-to-end entry, one set per (calling thread, device), created
// on first use: concurrent callers on different host threads never share an event (an event
// re-recorded by another thread between this call's record and wait would order the wrong work).
// The set lives as long as the thread (not destroyed at thread exit: the CUDA context may already
// be gone then).
struct E2EPipe {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t start = nullptr, done = nullptr;
  cudaEvent_t h[16] = {}, g[16] = {};
};
thread_local std::map<int, E2EPipe> g_e2e;
cudaError_t e2e_pipe(E2EPipe** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  auto it = g_e2e.find(dev);
  if (it == g_e2e.end()) {
    E2EPipe p;
    if ((e = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming)) != cudaSuccess) return e;
    for (int c = 0; c < 16; ++c) {
      if ((e = cudaEventCreateWithFlags(&p.h[c], cudaEventDisableTiming)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&p.g[c], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    it = g_e2e.emplace(dev, p).first;
  }
  *out = &it->second;
  return cudaSuccess;
}
}  // namespace

fn_status flashnorm_linear_from_host(const void* a_host, const void* Wt_star, const float* c_star, int64_t M,
                                     int64_t K, int64_t N, float eps, float alpha, fn_mode mode, fn_dtype dtype,
                                     void* a_dev, void* z_dev, void* z_host, void* stream) {
  fn_status s;
  if ((s = check_dtype(dtype)) != FN_OK) return s;
  if (a_host == nullptr || z_host == nullptr || a_dev == nullptr || z_dev == nullptr)
    return fail(FN_ERR_NULL, "a_host=%p z_host=%p a_dev=%p z_dev=%p: NULL", a_host, z_host, a_dev, z_dev);
  if (M < 0 || K <= 0 || N <= 0) return fail(FN_ERR_SHAPE, "M=%lld K=%lld N=%lld", (long long)M, (long long)K, (long long)N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t eb = (size_t)elem_bytes(dtype);
  // Row chunks pipelined over three engines: H2D of chunk c+1 (copy stream) || the FlashNorm
  // linear of chunk c (the caller's stream) || D2H of chunk c-1 (second copy stream).  Rows are
  // independent (RMS is per token), so chunking changes nothing in z.  Decode-sized calls and
  // tiny problems take one chunk.
  int64_t MC = M;
  if (M >= 1024) MC = ((M / 8 + 255) / 256) * 256;  // ~8 chunks of a multiple of 256 rows
  const int nc = (int)((M + MC - 1) / MC);
  if (nc <= 1) {
    cudaError_t e = cudaMemcpyAsync(a_dev, a_host, (size_t)M * K * eb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "H2D a");
    if ((s = linear_impl(a_dev, Wt_star, c_star, M, K, N, eps, alpha, mode, dtype, z_dev, FN_PATH_AUTO, nullptr, 0,
                         st)) != FN_OK)
      return s;
    e = cudaMemcpyAsync(z_host, z_dev, (size_t)M * N * eb, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "D2H z");
    return FN_OK;
  }
  E2EPipe* pp = nullptr;
  cudaError_t e = e2e_pipe(&pp);
  if (e != cudaSuccess) return cuda_fail(e, "e2e streams");
  // everything earlier on the caller's stream (e.g. the previous call reading a_dev / z_dev)
  // precedes this call's copies
  if ((e = cudaEventRecord(pp->start, st)) != cudaSuccess) return cuda_fail(e, "event");
  if ((e = cudaStreamWaitEvent(pp->h2d, pp->start, 0)) != cudaSuccess) return cuda_fail(e, "event wait");
  if ((e = cudaStreamWaitEvent(pp->d2h, pp->start, 0)) != cudaSuccess) return cuda_fail(e, "event wait");
  const uint8_t* ah = static_cast<const uint8_t*>(a_host);
  uint8_t* ad = static_cast<uint8_t*>(a_dev);
  uint8_t* zd = static_cast<uint8_t*>(z_dev);
  uint8_t* zh = static_cast<uint8_t*>(z_host);
  for (int c = 0; c < nc; ++c) {
    const int64_t r0 = c * MC, mc = std::min(MC, M - r0);
    if ((e = cudaMemcpyAsync(ad + r0 * K * eb, ah + r0 * K * eb, (size_t)(mc * K) * eb, cudaMemcpyHostToDevice,
                             pp->h2d)) != cudaSuccess)
      return cuda_fail(e, "H2D a");
    if ((e = cudaEventRecord(pp->h[c], pp->h2d)) != cudaSuccess) return cuda_fail(e, "event");
    if ((e = cudaStreamWaitEvent(st, pp->h[c], 0)) != cudaSuccess) return cuda_fail(e, "event wait");
    if ((s = linear_impl(ad + r0 * K * eb, Wt_star, c_star, mc, K, N, eps, alpha, mode, dtype, zd + r0 * N * eb,
                         FN_PATH_AUTO, nullptr, 0, st)) != FN_OK)
      return s;
    if ((e = cudaEventRecord(pp->g[c], st)) != cudaSuccess) return cuda_fail(e, "event");
    if ((e = cudaStreamWaitEvent(pp->d2h, pp->g[c], 0)) != cudaSuccess) return cuda_fail(e, "event wait");
    if ((e = cudaMemcpyAsync(zh + r0 * N * eb, zd + r0 * N * eb, (size_t)(mc * N) * eb, cudaMemcpyDeviceToHost,
                             pp->d2h)) != cudaSuccess)
      return cuda_fail(e, "D2H z");
  }
  // the caller's stream completes only after the last copy
  if ((e = cudaEventRecord(pp->done, pp->d2h)) != cudaSuccess) return cuda_fail(e, "event");
  if ((e = cudaStreamWaitEvent(st, pp->done, 0)) != cudaSuccess) return cuda_fail(e, "event wait");
  return FN_OK;
}

fn_status flashnorm_baseline_norm(const void* a, const float* g, const float* b, int64_t M, int64_t K, float eps,
                                  fn_mode mode, float alpha, fn_dtype dtype, void* y, void* stream) {
  fn_status s;
  if ((s = check_dtype(dtype)) != FN_OK) return s;
  if (M < 0 || K <= 0) return fail(FN_ERR_SHAPE, "a[%lld x %lld]: bad sizes", (long long)M, (long long)K);
  if (a == nullptr || y == nullptr) return fail(FN_ERR_NULL, "a=%p y=%p: NULL", a, y);
  if (mode == FN_NONE) return fail(FN_ERR_VALUE, "baseline_norm needs a normalization mode");
  if ((mode == FN_RMSNORM || mode == FN_LAYERNORM) && (!(eps >= 0.0f) || !std::isfinite(eps)))
    return fail(FN_ERR_VALUE, "eps = %g must be finite and >= 0", (double)eps);
  if (M == 0) return FN_OK;
  const int kind = mode == FN_RMSNORM ? 0 : mode == FN_LAYERNORM ? 1 : 2;
  cudaError_t e = fn::launch_baseline_norm(a, g, b, M, K, eps, kind, alpha, dtype == FN_BF16 ? 0 : 1, y,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "baseline_norm");
  ++g_launches;
  return FN_OK;
}

fn_status flashnorm_gather_columns(const void* z_parts, int64_t P, int64_t M, int64_t N_local, fn_dtype dtype, void* z,
                                   void* stream) {
  fn_status s;
  if ((s = check_dtype(dtype)) != FN_OK) return s;
  if (P <= 0 || M < 0 || N_local <= 0)
    return fail(FN_ERR_SHAPE, "z_parts[%lld][%lld][%lld]: bad sizes", (long long)P, (long long)M, (long long)N_local);
  if (z_parts == nullptr || z == nullptr) return fail(FN_ERR_NULL, "z_parts=%p z=%p: NULL", z_parts, z);
  if ((s = check_vec("N_local", N_local, dtype)) != FN_OK) return s;
  if ((s = check_ptr16("z_parts", z_parts)) != FN_OK || (s = check_ptr16("z", z)) != FN_OK) return s;
  if (M == 0) return FN_OK;
  cudaError_t e = fn::launch_gather_columns(z_parts, P, M, N_local, elem_bytes(dtype), z,
                                            static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "gather_columns");
  ++g_launches;
  return FN_OK;
}

const char* flashnorm_status_string(fn_status s) {
  switch (s) {
    case FN_OK: return "FN_OK";
    case FN_ERR_NULL: return "FN_ERR_NULL";
    case FN_ERR_SHAPE: return "FN_ERR_SHAPE";
    case FN_ERR_DTYPE: return "FN_ERR_DTYPE";
    case FN_ERR_ALIGN: return "FN_ERR_ALIGN";
    case FN_ERR_VALUE: return "FN_ERR_VALUE";
    case FN_ERR_UNSUPPORTED: return "FN_ERR_UNSUPPORTED";
    case FN_ERR_CUDA: return "FN_ERR_CUDA";
    case FN_ERR_NCCL: return "FN_ERR_NCCL";
  }
  return "FN_ERR_UNKNOWN";
}

const char* flashnorm_last_error(void) { return g_err; }
int64_t flashnorm_launch_count(void) { return g_launches; }
void flashnorm_reset_launch_count(void) { g_launches = 0; }
const char* flashnorm_version(void) { return "flashnorm-b200 0.1.0 sm_100a"; }

}  // extern "C"
