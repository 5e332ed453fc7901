// stream_bw.cu — HBM read bandwidth of the access shapes the fold kernels use (B200 measurement
// tool, not part of the library).  Reads a [rows x cols] bf16 matrix once per launch, rotating
// over buffers > 3x L2, and reports GB/s for:
//   ldg   : LDG.128, each warp reads 512 contiguous bytes of a row per instruction
//   tma W : a persistent CTA per SM streams [R rows x W bytes] boxes through a 192 KiB TMA ring,
//           one elected thread issuing, all threads consuming (one LDS per 16 B) and releasing
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro/stream_bw \
//        tools/micro/stream_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

__device__ unsigned g_sink;

__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n16, int unroll) {
  unsigned x = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
    x ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n16; i += stride) x ^= __ldcs(p + i).x;
  if (x == 0x12345678u) g_sink = x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256, 1) tma_kernel(const __grid_constant__ CUtensorMap tm, int rows, int cols_b,
                                                   int box_w, int box_r, int colmajor, int hint, int ring_max) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[64];
  const int box = box_w * box_r;
  const int ring = min(ring_max, min(64, (220 * 1024) / box));
  const int nbx = cols_b / box_w, nby = rows / box_r;
  const int nboxes = nbx * nby;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ring; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  int issued = 0, k = 0;
  auto issue = [&](int upto) {
    while (issued < upto) {
      const int bi = blockIdx.x + issued * gridDim.x;
      if (bi >= nboxes) return;
      const int slot = issued % ring;
      const int x = (colmajor ? bi / nby : bi % nbx) * (box_w / 2), y = (colmajor ? bi % nby : bi / nbx) * box_r;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])), "r"(box));
      if (hint)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%3, %4}], [%2], %5;"
            ::"r"(smem_u32(sm + (size_t)slot * box)), "l"(&tm), "r"(smem_u32(&full[slot])), "r"(x), "r"(y),
            "l"(0x12F0000000000000ull)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
            ::"r"(smem_u32(sm + (size_t)slot * box)), "l"(&tm), "r"(smem_u32(&full[slot])), "r"(x), "r"(y)
            : "memory");
      ++issued;
    }
  };
  if (threadIdx.x == 0) issue(ring);
  unsigned xacc = 0;
  for (int bi = blockIdx.x; bi < nboxes; bi += gridDim.x, ++k) {
    const int slot = k % ring;
    const uint32_t par = (k / ring) & 1;
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
            smem_u32(&full[slot])),
        "r"(par)
        : "memory");
    const uint4* b4 = reinterpret_cast<const uint4*>(sm + (size_t)slot * box);
    for (int i = threadIdx.x; i < box / 16; i += blockDim.x) xacc ^= b4[i].x;
    __syncthreads();
    if (threadIdx.x == 0) issue(k + 1 + ring);
  }
  if (xacc == 0x12345678u) g_sink = xacc;
}

int main(int argc, char** argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 4096 * 4, cols = 4096;  // bf16 [rows x 4096]
  const int ring_boxes = argc > 2 ? atoi(argv[2]) : 6;
  const size_t bytes = (size_t)rows * cols * 2;
  const int NB = rows >= 16384 ? 4 : 8;
  std::vector<void*> bufs(NB);
  for (auto& b : bufs) {
    cudaMalloc(&b, bytes);
    cudaMemset(b, 1, bytes);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch, int reps) {
    for (int i = 0; i < 2; ++i) launch(i % NB);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch(i % NB);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return bytes * reps / (ms * 1e-3) / 1e9;
  };
  for (int bpsm : {8})
    for (int thr : {512}) {
      const double gbs = timeit([&](int i) { ldg_kernel<<<sms * bpsm, thr>>>((const uint4*)bufs[i], bytes / 16, 4); }, 8);
      printf("ldg   blocks/SM %2d x %3d thr: %7.0f GB/s\n", bpsm, thr, gbs);
    }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
  const int shapes[][2] = {{256, 128}, {512, 64}};
  for (auto& sh : shapes) {
    std::vector<CUtensorMap> maps(NB);
    for (int i = 0; i < NB; ++i) {
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t str[1] = {(cuuint64_t)cols * 2};
      cuuint32_t box[2] = {(cuuint32_t)(sh[0] / 2), (cuuint32_t)sh[1]};
      cuuint32_t es[2] = {1, 1};
      enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, bufs[i], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int cm = 0; cm < 2; ++cm)
      for (int hint = 0; hint < 2; ++hint) {
        const double gbs = timeit(
            [&](int i) { tma_kernel<<<sms, 256, 224 * 1024>>>(maps[i], rows, cols * 2, sh[0], sh[1], cm, hint, ring_boxes); }, 8);
        printf("tma   box %4d B x %3d rows (%6d B), 1 CTA/SM, %s%s: %7.0f GB/s  (%s)\n", sh[0], sh[1], sh[0] * sh[1],
               cm ? "column-major" : "row-major   ", hint ? " evict_first" : "            ", gbs,
               cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
