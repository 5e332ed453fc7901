// 2D TMA (SW128 boxes of 128 rows x 64 bf16) L2 -> SMEM throughput per CTA, decode-kernel pattern:
// (a) row-major W*[6144 x 4096] (each box = 128 rows of 128 B, 8 KiB apart),
// (b) the same bytes pre-tiled so each box is one contiguous 16 KiB block,
// (c) 1D cp.async.bulk of the contiguous block.  48*S CTAs (48 tiles x S K splits), W* L2-resident.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>  // 0 rowmajor 2D, 1 tiled 2D, 2 tiled 1D bulk
__global__ void __launch_bounds__(128) k(const __grid_constant__ CUtensorMap tm, const uint8_t* tiled, int nkb_cta, int S, unsigned* out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int ST = 12, STAGE = 16384;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[ST];
  const int tile = blockIdx.x / S, rank = blockIdx.x % S;
  const int kb0 = rank * nkb_cta;
  if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&full[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  auto issue = [&](int t) {
    int s = t % ST;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s])), "r"(STAGE));
    if (MODE == 0) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(su32(sm + s * STAGE)), "l"(&tm), "r"((kb0 + t) * 64), "r"(tile * 128), "r"(su32(&full[s])) : "memory");
    } else if (MODE == 1) {
      const int blk = tile * (nkb_cta * S) + kb0 + t;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(su32(sm + s * STAGE)), "l"(&tm), "r"(0), "r"(blk * 128), "r"(su32(&full[s])) : "memory");
    } else {
      const size_t blk = (size_t)tile * (nkb_cta * S) + kb0 + t;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32(sm + s * STAGE)), "l"(tiled + blk * STAGE), "r"(STAGE), "r"(su32(&full[s])) : "memory");
    }
  };
  if (threadIdx.x == 0) for (int t = 0; t < ST && t < nkb_cta; ++t) issue(t);
  uint32_t acc = 0;
  for (int t = 0; t < nkb_cta; ++t) {
    int s = t % ST; uint32_t ph = (t / ST) & 1;
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" :: "r"(su32(&full[s])), "r"(ph) : "memory");
    acc ^= reinterpret_cast<const uint32_t*>(sm + s * STAGE)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && t + ST < nkb_cta) issue(t + ST);
  }
  if (acc == 0x12345678u) out[0] = acc;
}
static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}
static CUtensorMap tmap(void* ptr, uint64_t rows, uint64_t cols) {
  CUtensorMap m; cuuint64_t dims[2] = {cols, rows}; cuuint64_t str[1] = {cols * 2};
  cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("tmap err %d\n", (int)r);
  return m;
}
template <typename K, typename... A>
void launch_pdl(K kk, int grid, int block, size_t smem, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(block); cfg.dynamicSmemBytes = smem; cfg.stream = 0;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kk, args...);
}
int main() {
  const int N = 6144, K = 4096;
  uint8_t* w; cudaMalloc(&w, (size_t)N * K * 2); cudaMemset(w, 1, (size_t)N * K * 2);
  unsigned* out; cudaMalloc(&out, 64);
  CUtensorMap trow = tmap(w, N, K), ttile = tmap(w, (uint64_t)N * K / 64, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t smem = 12 * 16384 + 1024;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* nm[3] = {"2D row-major W* box 128x64", "2D pre-tiled (contiguous box)", "1D bulk pre-tiled 16 KiB"};
  for (int S : {1, 2, 3}) {
    const int grid = 48 * S, nkb = 64 / S;
    for (int m = 0; m < 3; ++m) {
      auto f = [&]() {
        if (m == 0) launch_pdl(k<0>, grid, 128, smem, trow, (const uint8_t*)w, nkb, S, out);
        else if (m == 1) launch_pdl(k<1>, grid, 128, smem, ttile, (const uint8_t*)w, nkb, S, out);
        else launch_pdl(k<2>, grid, 128, smem, trow, (const uint8_t*)w, nkb, S, out);
      };
      for (int i = 0; i < 20; ++i) f();
      cudaEventRecord(a); for (int i = 0; i < 200; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); double us = ms * 1e3 / 200;
      const double per = (double)nkb * 16384;
      printf("S=%d grid=%3d %-32s %6.2f us  %6.1f GB/s per CTA  %6.0f GB/s total (%s)\n", S, grid, nm[m], us, per / us / 1e3,
             grid * per / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
