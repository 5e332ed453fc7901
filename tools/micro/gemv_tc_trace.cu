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
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
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
  const int K = 4096, N = 6144, M = argc > 1 ? atoi(argv[1]) : 1;
  std::vector<__nv_bfloat16*> W(4);
  for (auto& w : W) { cudaMalloc(&w, (size_t)K * N * 2); cudaMemset(w, 0, (size_t)K * N * 2); }
  __nv_bfloat16 *a, *z; cudaMalloc(&a, K * 2 * 16); cudaMalloc(&z, N * 2 * 16); cudaMemset(a, 0, K * 32);
  CUtensorMap tw[4], ta = tmap(a, M, K, 16);
  const int tr_rows = fn::gemv_tc_tile_rows(0, K, N, 148);
  printf("tile rows %d\n", tr_rows);
  for (int i = 0; i < 4; ++i) tw[i] = tmap(W[i], N, K, tr_rows);
  auto launch = [&](int i) {
    unsigned v = (unsigned)i; cudaMemcpyToSymbolAsync(fn::g_tc_launch, &v, 4, 0, cudaMemcpyHostToDevice, 0);
    fn::launch_gemv_tc(tw[i % 4], ta, nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0);
  };
  auto launch_plain = [&](int i) { fn::launch_gemv_tc(tw[i % 4], ta, nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0); };
  for (int i = 0; i < 40; ++i) launch_plain(i);
  cudaDeviceSynchronize();
  printf("split S = %d\n", fn::gemv_tc_split(K, N, 148));
  unsigned v0 = 0; cudaMemcpyToSymbol(fn::g_tc_launch, &v0, 4);
  for (int i = 0; i < 6; ++i) launch_plain(i);  // launches 0..5: parities 0,1,0,1,0,1 -> 4 = A, 5 = B
  cudaDeviceSynchronize();
  static unsigned long long tr[2][160][8];
  cudaMemcpyFromSymbol(tr, fn::g_tc_trace, sizeof(tr));
  int nct = 0;
  while (nct < 160 && tr[0][nct][0] != 0) ++nct;
  printf("CTAs per launch: %d\n", nct);
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
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); for (int i = 0; i < 200; ++i) launch_plain(i); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("back-to-back: %.2f us/launch (%s)\n", ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
}
