// Gram timing harness: tc_gram at the configs[2] block shape (n' × 286, ld 288),
// exact (3xTF32) and inexact (tf32), symmetric.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 -I.. scripts/dbg/gram_prof.cu -lcuda -o scripts/dbg/gram_prof
#include "../../paper_2110_12782_b200/csrc/tc_gemm.cu"
#include <cstdio>
using namespace netmfp;
namespace netmfp { void set_last_error(const std::string &) {} }
int main(int argc, char **argv) {
  Ctx c; cudaStreamCreate(&c.stream);
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0); c.num_sms = prop.multiProcessorCount;
  const int64_t n = argc > 1 ? atoll(argv[1]) : 406727, K = argc > 2 ? atoi(argv[2]) : 286, ld = (K + 31) / 32 * 32;
  float *A; double *G;
  cudaMalloc(&A, n * ld * 4); cudaMalloc(&G, K * K * 8);
  cudaMemset(A, 0, n * ld * 4);
  Mat Am{A, n, K, ld};
  for (int ex = 0; ex < 2; ++ex)
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      const int reps = rep ? 20 : 1;
      cudaEventRecord(e0, c.stream);
      for (int r = 0; r < reps; ++r) tc_gram(c, Am, Am, nullptr, 0.f, G, K, ex == 1);
      cudaEventRecord(e1, c.stream);
      cudaStreamSynchronize(c.stream);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
#ifdef TC_PROF
      unsigned long long zero[1024 * 8] = {}, hp[1024 * 8];
      cudaMemcpyToSymbol(g_tcprof, zero, sizeof(zero));
      tc_gram(c, Am, Am, nullptr, 0.f, G, K, ex == 1);
      cudaStreamSynchronize(c.stream);
      cudaMemcpyFromSymbol(hp, g_tcprof, sizeof(hp));
      double tot[8] = {};
      for (int b = 0; b < 148; ++b) for (int i = 0; i < 8; ++i) tot[i] += hp[b * 8 + i] / 148.0;
      if (rep) printf("  cycles/CTA (first 148 chains): prod-wait-empty %.0f mma-wait-split %.0f work-wait-full %.0f epi-wait-done %.0f issue-body %.0f work-body %.0f\n",
             tot[0], tot[2], tot[3], tot[4], tot[5], tot[6]);
#endif
      printf("exact=%d %.4f ms/call (%s)  read %.1f GB/s\n", ex, ms / reps, cudaGetErrorString(cudaGetLastError()),
             n * ld * 4.0 / (ms / reps) / 1e6);
    }
  return 0;
}
