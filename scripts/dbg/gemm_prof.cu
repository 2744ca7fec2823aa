#define TC_PROF
#include "../../paper_2110_12782_b200/csrc/tc_gemm.cu"
#include <cstdio>
#include <vector>
using namespace netmfp;
namespace netmfp { void set_last_error(const std::string &) {} void dist_allreduce(Ctx &, void *, size_t, DType) {} }
int main() {
  Ctx c; cudaStreamCreate(&c.stream);
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0); c.num_sms = prop.multiProcessorCount;
  const int64_t n = 406727, K = 286, ld = 288;
  float *A, *C; double *B;
  cudaMalloc(&A, n * ld * 4); cudaMalloc(&C, n * ld * 4); cudaMalloc(&B, K * K * 8);
  cudaMemset(A, 0, n * ld * 4); cudaMemset(B, 0, K * K * 8);
  Mat Am{A, n, K, ld}, Cm{C, n, K, ld};
  for (int tri = 0; tri < 3; ++tri)
  for (int rep = 0; rep < 2; ++rep) {
#ifdef TC_PROF
    unsigned long long zero[1024 * 8] = {};
    cudaMemcpyToSymbol(g_tcprof, zero, sizeof(zero));
#endif
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = rep ? 10 : 1;
    cudaEventRecord(e0, c.stream);
    for (int r = 0; r < reps; ++r) {
      if (tri == 2) tc_gemm_tall_tri(c, Am, B, K, K, nullptr, 0.f, Cm, false); else if (tri) tc_gemm_tall_tri(c, Am, B, K, K, nullptr, 0.f, Cm); else tc_gemm_tall(c, Am, B, K, K, nullptr, 0.f, Cm);
    }
    cudaEventRecord(e1, c.stream);
    cudaStreamSynchronize(c.stream);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    unsigned long long hp[1024 * 8] = {};
#ifdef TC_PROF
    cudaMemcpyFromSymbol(hp, g_tcprof, sizeof(hp));
#endif
    double tot[8] = {};
    for (int b = 0; b < 148; ++b) for (int i = 0; i < 8; ++i) tot[i] += hp[b * 8 + i] / 148.0;
    printf("tri=%d %.3f ms (%s): cycles/CTA prod-wait-empty %.0f mma-wait-tfree %.0f mma-wait-split %.0f split-wait-full %.0f epi-wait-done %.0f epi-work %.0f mma-issue %.0f\n",
           tri, ms, cudaGetErrorString(cudaGetLastError()), tot[0], tot[1], tot[2], tot[3], tot[4], tot[5], tot[6]);
  }
  return 0;
}
