// sk_trace.cu — per-item timeline of the CTA-pair GEMM with the stream-K tail (config 4 shape),
// globaltimer stamps: MMA item start/end, epilogue start, partial acquired, accumulator ready, end.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DFN_SK_TRACE -I include \
//        -o tools/micro/sk_trace tools/micro/sk_trace.cu $(ls paper_2407_09577_b200/_build/*.o | grep -v '/api.o\|/gemm2_sm100.o') -ldl
#include "../../paper_2407_09577_b200/csrc/api.cu"
#include "../../paper_2407_09577_b200/csrc/gemm2_sm100.cu"
#include <vector>
int main(int argc, char** argv) {
  const int M = 2048, K = 4096, N = 4096;
  void *a, *w, *z, *ws;
  cudaMalloc(&a, (size_t)M * K * 2);
  cudaMalloc(&w, (size_t)N * K * 2);
  cudaMalloc(&z, (size_t)M * N * 2);
  cudaMemset(a, 0x3c, (size_t)M * K * 2);
  cudaMemset(w, 0x3c, (size_t)N * K * 2);
  const int64_t wb = flashnorm_linear_workspace_bytes(M, K, N, FN_NONE, FN_BF16, FN_PATH_AUTO);
  cudaMalloc(&ws, wb + 16);
  float* u;
  cudaMalloc(&u, N * sizeof(float));
  cudaMemset(u, 0, N * sizeof(float));
  cudaMemset(ws, 0, wb + 16);
  printf("workspace %lld\n", (long long)wb);
  const int ncalls = (argc > 2 && argv[2][0] == 'x') ? 7 : 6;  // an odd count leaves the whole-tile call's trace
  for (int it = 0; it < ncalls; ++it) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fn_status st = argc > 1 && argv[1][0] == 'l'
                       ? flashnorm_layernorm_linear(a, w, u, nullptr, M, K, N, 1e-5f, FN_BF16, z, nullptr)
                       : flashnorm_linear_ws(a, w, nullptr, M, K, N, 0.f, 0.f,
                                             argc > 1 && argv[1][0] == 'r' ? FN_RMSNORM : FN_NONE, FN_BF16, z,
                                             FN_PATH_AUTO, it % 2 ? ws : nullptr, it % 2 ? wb : 0, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("call %d (%s): status %d %.1f us (%s)\n", it, it % 2 ? "stream-K" : "whole tiles", (int)st, ms * 1e3,
           cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> tr(160 * 4 * 6);
  cudaMemcpyFromSymbol(tr.data(), fn::g_sk_trace, tr.size() * 8);
  unsigned long long t0 = ~0ull;
  for (size_t i = 0; i < tr.size(); ++i)
    if (tr[i]) t0 = std::min(t0, tr[i]);
  auto us = [&](unsigned long long x) { return x ? (double)(x - t0) / 1e3 : -1.0; };
  for (int b : {0, 1, 2, 3, 40, 41, 146, 147}) {
    printf("CTA %3d:", b);
    for (int i = 0; i < 4; ++i) {
      const unsigned long long* e = &tr[(b * 4 + i) * 6];
      printf(" | it%d mma %.1f-%.1f epi %.1f flag %.1f acc %.1f end %.1f", i, us(e[0]), us(e[1]), us(e[2]), us(e[3]),
             us(e[4]), us(e[5]));
    }
    printf("\n");
  }
  {  // span of the traced call over ALL CTAs: first MMA start -> last epilogue end
    unsigned long long lo = ~0ull, hi = 0;
    for (int b = 0; b < 148; ++b)
      for (int i = 0; i < 4; ++i) {
        const unsigned long long* e = &tr[(b * 4 + i) * 6];
        if (e[0]) lo = std::min(lo, e[0]);
        if (e[5]) hi = std::max(hi, e[5]);
      }
    printf("traced call span over all CTAs: %.2f us\n", (hi - lo) / 1e3);
    if (argc > 3)
      for (int b = 0; b < 148; b += 2) {
        printf("pair %2d:", b / 2);
        for (int i = 0; i < 4; ++i) {
          const unsigned long long* e = &tr[(b * 4 + i) * 6];
          if (e[0]) printf(" [mma %.1f-%.1f (%.1f) acc %.1f end %.1f%s]", (e[0] - lo) / 1e3, (e[1] - lo) / 1e3,
                           (e[1] - e[0]) / 1e3, (e[4] - lo) / 1e3, (e[5] - lo) / 1e3, e[3] ? " F" : "");
        }
        printf("\n");
      }
  }
  for (int mode = 0; mode < 2; ++mode) {  // back-to-back launches (GPU-bound: ~40 us kernels)
    auto call = [&] {
      if (argc > 1 && argv[1][0] == 'l') {
        flashnorm_layernorm_linear(a, w, u, nullptr, M, K, N, 1e-5f, FN_BF16, z, nullptr);
        return;
      }
      flashnorm_linear_ws(a, w, nullptr, M, K, N, 0.f, 0.f, argc > 1 && argv[1][0] == 'r' ? FN_RMSNORM : FN_NONE,
                          FN_BF16, z, FN_PATH_AUTO, mode ? ws : nullptr, mode ? wb : 0, nullptr);
    };
    for (int i = 0; i < 5; ++i) call();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) call();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("back-to-back x50 %s: %.2f us/call = %.0f TFLOP/s\n", mode ? "stream-K" : "whole tiles", ms * 1e3 / 50,
           2.0 * M * K * N / (ms * 1e-3 / 50) / 1e12);
  }
  std::vector<unsigned long long> ch(160 * 4 * 4 * 8 * 2);
  cudaMemcpyFromSymbol(ch.data(), fn::g_sk_chunk, ch.size() * 8);
  for (int b : {0, 2, 146}) {
    for (int i = 0; i < 3; ++i) {
      for (int w = 0; w < 4; w += 3) {
        printf("CTA %3d it%d warp %d chunks (ready/stored):", b, i, w);
        for (int j = 0; j < 8; ++j) {
          const unsigned long long* e = &ch[((((size_t)b * 4 + i) * 4 + w) * 8 + j) * 2];
          printf(" %.2f/%.2f", us(e[0]), us(e[1]));
        }
        printf("\n");
      }
    }
  }
  return 0;
}
