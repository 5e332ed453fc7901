// k2p_trace.cu — timeline of the persistent K2 (fold_mean_center_persist_kernel): globaltimer stamps
// per CTA (FN_K2_TRACE), calls back to back on 6 rotating V.  Measurement tool only.
// build (after python -m paper_2407_09577_b200.build):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DFN_K2_TRACE -I include \
//        -o tools/micro/k2p_trace tools/micro/k2p_trace.cu $(ls paper_2407_09577_b200/_build/*.o | grep -v '/api.o\|/fold.o') -ldl
#include "../../paper_2407_09577_b200/csrc/api.cu"
#include "../../paper_2407_09577_b200/csrc/fold.cu"
#include <algorithm>
#include <vector>
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4096;
  const int NB = 6;
  std::vector<void*> V(NB), Vs(NB);
  void* ws;
  cudaMalloc(&ws, flashnorm_fold_mean_center_workspace_bytes(n, n));
  for (int i = 0; i < NB; ++i) {
    cudaMalloc(&V[i], (size_t)n * n * 2);
    cudaMalloc(&Vs[i], (size_t)n * n * 2);
    cudaMemset(V[i], 0x3c, (size_t)n * n * 2);
  }
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int it = 0; it < 12; ++it) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    fn_status s = flashnorm_fold_mean_center(V[it % NB], n, n, FN_BF16, nullptr, Vs[it % NB], nullptr, ws, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("call %d: status %d, %.1f us (%s)\n", it, (int)s, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> tr(160 * 32);
  cudaMemcpyFromSymbol(tr.data(), fn::g_k2_trace, tr.size() * 8);
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < 160; ++b)
    if (tr[b * 32]) t0 = std::min(t0, tr[b * 32]);
  const char* names[] = {"start", "issued", "tile0", "p1done", "sync1", "Rdone", "sync2", "p2issued", "end"};
  for (int i = 0; i < 9; ++i) {
    double mn = 1e30, mx = -1, sum = 0;
    int cnt = 0;
    for (int b = 0; b < 160; ++b) {
      if (!tr[b * 32 + i]) continue;
      const double x = (double)(tr[b * 32 + i] - t0) / 1e3;
      mn = std::min(mn, x);
      mx = std::max(mx, x);
      sum += x;
      ++cnt;
    }
    printf("%-9s min %6.2f  mean %6.2f  max %6.2f us  (%d CTAs)\n", names[i], mn, cnt ? sum / cnt : 0, mx, cnt);
  }
  return 0;
}
