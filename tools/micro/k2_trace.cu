// k2_trace.cu — timeline of the K2 fold_mean_center kernel (globaltimer stamps per CTA), built with
// the library sources in one translation unit and FN_K2_TRACE defined.  Measurement tool only.
// build (after python -m paper_2407_09577_b200.build):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DFN_K2_TRACE -I include \
//        -o tools/micro/k2_trace tools/micro/k2_trace.cu $(ls paper_2407_09577_b200/_build/*.o | grep -v '/api.o\|/fold.o') -ldl
#include "../../paper_2407_09577_b200/csrc/api.cu"
#include "../../paper_2407_09577_b200/csrc/fold.cu"
#include <vector>
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4096;
  const int NB = 6;
  std::vector<void*> V(NB), Vs(NB);
  for (int i = 0; i < NB; ++i) {
    cudaMalloc(&V[i], (size_t)n * n * 2);
    cudaMalloc(&Vs[i], (size_t)n * n * 2);
    cudaMemset(V[i], 0x3c, (size_t)n * n * 2);
  }
  for (int it = 0; it < 8; ++it) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    fn_status st = flashnorm_fold_mean_center(V[it % NB], n, n, FN_BF16, nullptr, Vs[it % NB], nullptr, nullptr, nullptr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("call %d: status %d, %.1f us (%s)\n", it, (int)st, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> tr(160 * 32);
  cudaMemcpyFromSymbol(tr.data(), fn::g_k2_trace, tr.size() * 8);
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < 160; ++b)
    if (tr[b * 32]) t0 = std::min(t0, tr[b * 32]);
  auto us = [&](unsigned long long x) { return x ? (double)(x - t0) / 1e3 : -1.0; };
  for (int b : {0, 1, 7, 8, 64, 127, 128, 143}) {
    printf("CTA %3d start %.2f clsync %.2f |", b, us(tr[b * 32]), us(tr[b * 32 + 1]));
    for (int i = 0; i < 4; ++i)
      printf(" s%d box0 %.2f boxlast %.2f lanes %.2f gotlanes %.2f mu %.2f p2done %.2f |", i, us(tr[b * 32 + 6 + 6 * i]),
             us(tr[b * 32 + 7 + 6 * i]), us(tr[b * 32 + 2 + 6 * i]), us(tr[b * 32 + 3 + 6 * i]), us(tr[b * 32 + 4 + 6 * i]),
             us(tr[b * 32 + 5 + 6 * i]));
    printf(" end %.2f\n", us(tr[b * 32 + 30]));
  }
  return 0;
}
