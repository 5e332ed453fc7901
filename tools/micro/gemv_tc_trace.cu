// Timeline of back-to-back PDL launches of the tcgen05 decode kernel (globaltimer):
// CTA start, griddepcontrol.wait released (producer), accumulator complete, CTA exit.
#define FN_GEMV_TC_TRACE 1
#include "../../paper_2407_09577_b200/csrc/gemv_tc.cu"
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include <algorithm>
static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || p == nullptr) { fprintf(stderr, "no cuTensorMapEncodeTiled: %s\n", cudaGetErrorString(e)); exit(1); }
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}
static CUtensorMap tmap(void* ptr, int rows, int cols, int box_rows) {
  CUtensorMap m; cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}; cuuint32_t es[2] = {1, 1};
  enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}
int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int K = 4096, N = 6144, M = argc > 1 ? atoi(argv[1]) : 1;
  const int MODE = argc > 3 ? atoi(argv[3]) : 0;  // fn::MODE_RMS = 0, MODE_DYT = 1
  std::vector<__nv_bfloat16*> W(4);
  for (auto& w : W) { cudaMalloc(&w, (size_t)K * N * 2); cudaMemset(w, 0, (size_t)K * N * 2); }
  __nv_bfloat16 *a, *z; cudaMalloc(&a, K * 2 * 16); cudaMalloc(&z, N * 2 * 16); cudaMemset(a, 0, K * 32);
  printf("alloc ok\n");
  CUtensorMap tw[4], ta = tmap(a, M, K, 16);
  printf("tmap ok\n");
  const int tr_rows = fn::gemv_tc_tile_rows(0, K, N, 148);
  printf("tile rows %d\n", tr_rows);
  for (int i = 0; i < 4; ++i) tw[i] = tmap(W[i], N, K, tr_rows);
  auto launch = [&](int i) {
    unsigned v = (unsigned)i; cudaMemcpyToSymbolAsync(fn::g_tc_launch, &v, 4, 0, cudaMemcpyHostToDevice, 0);
    fn::launch_gemv_tc(tw[i % 4], ta, nullptr, z, M, K, N, 1e-5f, 0.5f, MODE, 148, 0, nullptr, fn::RopeParams{nullptr, nullptr, nullptr, 0, 0, 1.f, nullptr, nullptr, 0, 0.f}, nullptr, a);
  };
  auto launch_plain = [&](int i) { fn::launch_gemv_tc(tw[i % 4], ta, nullptr, z, M, K, N, 1e-5f, 0.5f, MODE, 148, 0, nullptr, fn::RopeParams{nullptr, nullptr, nullptr, 0, 0, 1.f, nullptr, nullptr, 0, 0.f}, nullptr, a); };
  {
    cudaError_t le = fn::launch_gemv_tc(tw[0], ta, nullptr, z, M, K, N, 1e-5f, 0.5f, MODE, 148, 0, nullptr, fn::RopeParams{nullptr, nullptr, nullptr, 0, 0, 1.f, nullptr, nullptr, 0, 0.f}, nullptr, a);
    printf("launch: %s\n", cudaGetErrorString(le));
    int n = -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(96); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = fn::dtc::Cfg<1>::smem(12);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&n, (const void*)fn::flashnorm_gemv_tc_kernel<0, 1>, &cfg);
    printf("occupancy clusters of 2 (12 stages): %d (%s)\n", n, cudaGetErrorString(oe));
    int nb = -1;
    oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)fn::flashnorm_gemv_tc_kernel<0, 1>, 192,
                                                       fn::dtc_smem(1, 2));
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)fn::flashnorm_gemv_tc_kernel<0, 1>);
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    size_t avail = 0;
    cudaOccupancyAvailableDynamicSMemPerBlock(&avail, (const void*)fn::flashnorm_gemv_tc_kernel<0, 1>, 2, 192);
    printf("regs %d static smem %zu maxdyn %d carveout %d | SM smem %zu reserved/block %zu regs/SM %d | avail dyn smem at 2 blocks %zu\n",
           fa.numRegs, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.preferredShmemCarveout,
           pr.sharedMemPerMultiprocessor, pr.reservedSharedMemPerBlock, pr.regsPerMultiprocessor, avail);
    for (size_t sm : {(size_t)0, (size_t)50000, (size_t)100000, (size_t)112640}) {
      int b2 = -1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, (const void*)fn::flashnorm_gemv_tc_kernel<0, 1>, 192, sm);
      int b3 = -1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b3, (const void*)fn::flashnorm_gemv_tc_kernel<0, 1>, 128, sm);
      printf("  smem %zu: blocks/SM %d (192 thr) %d (128 thr)\n", sm, b2, b3);
    }
    cudaGetLastError();
    printf("blocks per SM at the configured ring (%zu B): %d (%s)\n", fn::dtc_smem(1, 2), nb, cudaGetErrorString(oe));
  }
  for (int i = 0; i < 40; ++i) launch_plain(i);
  printf("warm sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  printf("split S = %d\n", fn::gemv_tc_split(K, N, 148));
  unsigned v0 = 0; cudaMemcpyToSymbol(fn::g_tc_launch, &v0, 4);
  for (int i = 0; i < 6; ++i) launch_plain(i);  // launches 0..5: parities 0,1,0,1,0,1 -> 4 = A, 5 = B
  cudaDeviceSynchronize();
  static unsigned long long tr[2][160][16];
  cudaMemcpyFromSymbol(tr, fn::g_tc_trace, sizeof(tr));
  int nct = 0;
  while (nct < 160 && tr[0][nct][0] != 0) ++nct;
  printf("CTAs per launch: %d\n", nct);
  if (nct == 0) return 1;
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < nct; ++b) t0 = std::min(t0, tr[0][b][0]);
  const char* nm[4] = {"start", "wait released", "acc complete", "exit"};
  for (int L = 0; L < 2; ++L)
    for (int e = 0; e < 4; ++e) {
      std::vector<double> v;
      for (int b = 0; b < nct; ++b) v.push_back(((double)tr[L][b][e] - (double)t0) * 1e-3);
      std::sort(v.begin(), v.end());
      printf("%s %-14s min %6.2f p50 %6.2f max %6.2f us\n", L ? "B" : "A", nm[e], v[0], v[nct / 2], v[nct - 1]);
    }
  if (FILE* f = fopen(argc > 2 ? argv[2] : "gpurun_out/gemv_tc_trace.csv", "w")) {
    fprintf(f, "launch,cta,smid,start,wait_released,first_stage,ring_refill,last_stage,acc_complete,part_stored,csync1,reduced,csync2,z_stored,joined,exit\n");
    for (int L = 0; L < 2; ++L)
      for (int b = 0; b < nct; ++b) {
        auto T = [&](int e) { return ((double)tr[L][b][e] - (double)t0) * 1e-3; };
        fprintf(f, "%d,%d,%llu,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f\n", L, b, tr[L][b][4], T(0), T(1), T(5), T(6), T(7),
                T(2), T(8), T(9), T(10), T(11), T(12), T(13), T(3));
      }
    fclose(f);
  }
  {
    static long long st[4][64];
    cudaMemcpyFromSymbol(st, fn::g_tc_stage, sizeof(st));
    printf("CTA0 per-stage clocks (relative to stage-0 MMA): i, mma_full, prod_issue, side_rel\n");
    for (int i = 0; i < 40; ++i)
      if (st[0][i]) printf("  %2d %8lld %8lld %8lld\n", i, st[0][i] - st[0][0], st[1][i] - st[0][0], st[2][i] - st[0][0]);
  }
  {
    static long long ep[2][8];
    cudaMemcpyFromSymbol(ep, fn::g_tc_epi, sizeof(ep));
    printf("epilogue clocks rel. to tfull (CTA0 leader / CTA1 peer): tmem_ld, push/recv start, push/recv done, z stored, joined, dealloc\n");
    for (int c = 0; c < 2; ++c) printf("  CTA%d: %lld %lld %lld %lld %lld %lld\n", c, ep[c][1] - ep[c][0], ep[c][2] - ep[c][0], ep[c][3] - ep[c][0], ep[c][4] - ep[c][0], ep[c][5] - ep[c][0], ep[c][6] - ep[c][0]);
    printf("  reduced (before z): CTA0 %lld CTA1 %lld\n", ep[0][7] - ep[0][0], ep[1][7] - ep[1][0]);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); for (int i = 0; i < 200; ++i) launch_plain(i); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("back-to-back: %.2f us/launch (%s)\n", ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
}
