// Per-CTA timeline of the decode kernel (globaltimer): entry, first stage landed,
// last stage landed, last reduction stored.  Builds gemv.cu with FN_GEMV_TRACE.
#define FN_GEMV_TRACE 1
#include "../../paper_2407_09577_b200/csrc/gemv.cu"
#include <cstdio>
#include <vector>
#include <algorithm>
int main() {
  const int K = 4096, N = 6144, M = 1;
  size_t wb = (size_t)K * N * 2;
  std::vector<__nv_bfloat16*> W(4);
  for (auto& w : W) { cudaMalloc(&w, wb); cudaMemset(w, 0, wb); }
  __nv_bfloat16 *a, *z; cudaMalloc(&a, K * 2 * 16); cudaMalloc(&z, N * 2 * 16); cudaMemset(a, 0, K * 32);
  for (int it = 0; it < 50; ++it) fn::launch_gemv(a, W[it % 4], nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0);
  cudaDeviceSynchronize();
  fn::launch_gemv(a, W[1], nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0);  // isolated launch (no PDL overlap)
  cudaDeviceSynchronize();
  unsigned long long tr[148 * 8];
  cudaMemcpyFromSymbol(tr, fn::g_gemv_trace, sizeof(tr));
  unsigned long long t0 = ~0ull, tmax = 0;
  for (int b = 0; b < 148; ++b) { t0 = std::min(t0, tr[b * 8]); tmax = std::max(tmax, tr[b * 8 + 3]); }
  std::vector<double> st, f1, f2, en, m5, m6;
  for (int b = 0; b < 148; ++b) { st.push_back((tr[b*8]-t0)*1e-3); f1.push_back((tr[b*8+1]-t0)*1e-3); f2.push_back((tr[b*8+2]-t0)*1e-3); en.push_back((tr[b*8+3]-t0)*1e-3); m5.push_back((tr[b*8+5]-t0)*1e-3); m6.push_back((tr[b*8+6]-t0)*1e-3); }
  auto stats = [](const char* n, std::vector<double> v) { std::sort(v.begin(), v.end()); printf("%-22s min %6.2f  p50 %6.2f  max %6.2f us\n", n, v[0], v[v.size()/2], v.back()); };
  stats("CTA start", st); stats("first stage landed", f1); stats("CTA done", en);
  printf("last launch span (first start -> last done): %.2f us\n", (tmax - t0) * 1e-3);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); for (int it = 0; it < 200; ++it) fn::launch_gemv(a, W[it % 4], nullptr, z, M, K, N, 1e-5f, 0.5f, 0, 148, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("back-to-back: %.2f us/launch (%s)\n", ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
}
