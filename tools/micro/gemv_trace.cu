// Per-CTA timeline of two back-to-back decode launches (globaltimer, PDL-chained):
// entry, griddepcontrol.wait released, first stage landed, CTA done — for launch A and
// the launch B that follows it.  Builds gemv.cu with FN_GEMV_TRACE.
#define FN_GEMV_TRACE 1
#include "../../paper_2407_09577_b200/csrc/gemv.cu"
#include <cstdio>
#include <vector>
#include <algorithm>
#include <chrono>
int main() {
  const int K = 4096, N = 6144, M = 1;
  size_t wb = (size_t)K * N * 2;
  std::vector<__nv_bfloat16*> W(4);
  for (auto& w : W) { cudaMalloc(&w, wb); cudaMemset(w, 0, wb); }
  __nv_bfloat16 *a, *z; cudaMalloc(&a, K * 2 * 16); cudaMalloc(&z, N * 2 * 16); cudaMemset(a, 0, K * 32);
  for (int it = 0; it < 51; ++it) fn::launch_gemv(a, W[it % 4], nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0);
  cudaDeviceSynchronize();
  for (int it = 0; it < 6; ++it) fn::launch_gemv(a, W[it % 4], nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0);
  cudaDeviceSynchronize();
  static unsigned long long tr[2][148 * 8];
  cudaMemcpyFromSymbol(tr, fn::g_gemv_trace, sizeof(tr));
  // 51 + 6 launches: the last two used slot parities (55 % 64) & 1 = 1 (A) and (56 % 64) & 1 = 0 (B)
  const int A = 1, B = 0;
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < 148; ++b) t0 = std::min(t0, tr[A][b * 8]);
  auto stats = [&](const char* n, int L, int slot) {
    std::vector<double> v;
    for (int b = 0; b < 148; ++b) v.push_back(((double)tr[L][b * 8 + slot] - (double)t0) * 1e-3);
    std::sort(v.begin(), v.end());
    printf("%-30s min %6.2f  p50 %6.2f  max %6.2f us\n", n, v[0], v[v.size() / 2], v.back());
  };
  {  // per SM: A exit -> B start
    std::vector<double> aexit(256, -1), bstart(256, -1);
    for (int b = 0; b < 148; ++b) {
      aexit[tr[A][b * 8 + 4]] = ((double)tr[A][b * 8 + 5] - (double)t0) * 1e-3;
      bstart[tr[B][b * 8 + 4]] = ((double)tr[B][b * 8 + 0] - (double)t0) * 1e-3;
    }
    std::vector<std::pair<double, int>> gap;
    for (int sm = 0; sm < 256; ++sm)
      if (aexit[sm] >= 0 && bstart[sm] >= 0) gap.push_back({bstart[sm] - aexit[sm], sm});
    std::sort(gap.begin(), gap.end());
    printf("SMs with both: %zu; A-exit -> B-start gap: min %.2f p50 %.2f max %.2f us (sm %d: A exit %.2f, B start %.2f)\n",
           gap.size(), gap.front().first, gap[gap.size() / 2].first, gap.back().first, gap.back().second,
           aexit[gap.back().second], bstart[gap.back().second]);
    int late = 0;
    for (auto& x : gap) late += x.first > 2.0;
    printf("SMs with gap > 2 us: %d\n", late);
  }
  {
    static unsigned long long tt[2][16][6];
    cudaMemcpyFromSymbol(tt, fn::g_gemv_ttrace, sizeof(tt));
    printf("block 0 of launch A, per tile (us from A's first CTA start): issue | w0 got stage | w0 stored | w14 stored | reducer done\n");
    for (int q = 0; q < 8; ++q) {
      auto f = [&](int ev) { return tt[A][q][ev] ? ((double)tt[A][q][ev] - (double)t0) * 1e-3 : -1.0; };
      printf("  seq %d: %6.2f | %6.2f | %6.2f | %6.2f | %6.2f\n", q, f(0), f(1), f(2), f(4), f(3));
    }
  }
  stats("A CTA start", A, 0); stats("A wait released", A, 2); stats("A first stage landed", A, 1); stats("A producer last issue+", A, 6); stats("A CTA done", A, 3); stats("A CTA exit", A, 5);
  { std::vector<int> nt; for (int b = 0; b < 148; ++b) nt.push_back((int)tr[A][b * 8 + 7]); std::sort(nt.begin(), nt.end());
    printf("A tiles per CTA: min %d p50 %d max %d\n", nt[0], nt[74], nt[147]); }
  stats("B CTA start", B, 0); stats("B wait released", B, 2); stats("B first stage landed", B, 1); stats("B CTA done", B, 3);
  {
    auto h0 = std::chrono::steady_clock::now();
    for (int it = 0; it < 200; ++it) fn::launch_gemv(a, W[it % 4], nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0);
    auto h1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    printf("host enqueue: %.2f us/launch\n", std::chrono::duration<double, std::micro>(h1 - h0).count() / 200);
  }
  {  // CUDA graph of 200 PDL-chained launches
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int it = 0; it < 200; ++it) fn::launch_gemv(a, W[it % 4], nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, st);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEvent_t g0, g1; cudaEventCreate(&g0); cudaEventCreate(&g1);
    cudaEventRecord(g0, st); cudaGraphLaunch(ge, st); cudaEventRecord(g1, st); cudaEventSynchronize(g1);
    float gms; cudaEventElapsedTime(&gms, g0, g1);
    printf("graph of 200: %.2f us/launch (%s)\n", gms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
    // timeline of the last two launches of the graph
    static unsigned long long tg[2][148 * 8];
    cudaMemcpyFromSymbol(tg, fn::g_gemv_trace, sizeof(tg));
    unsigned long long u0 = ~0ull;
    for (int b = 0; b < 148; ++b) u0 = std::min(u0, std::min(tg[0][b * 8], tg[1][b * 8]));
    for (int L = 0; L < 2; ++L) {
      const char* nm[4] = {"start", "first landed", "wait released", "done"};
      for (int sl = 0; sl < 4; ++sl) {
        std::vector<double> v;
        for (int b = 0; b < 148; ++b) v.push_back(((double)tg[L][b * 8 + sl] - (double)u0) * 1e-3);
        std::sort(v.begin(), v.end());
        printf("graph parity %d %-14s min %6.2f p50 %6.2f max %6.2f\n", L, nm[sl], v[0], v[74], v[147]);
      }
    }
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); for (int it = 0; it < 200; ++it) fn::launch_gemv(a, W[it % 4], nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("back-to-back: %.2f us/launch (%s)\n", ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
}
