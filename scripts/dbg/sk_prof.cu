// wait-cycle breakdown of the fused sketch kernel at configs[2] shapes
#define SK_PROF
#include "../../paper_2110_12782_b200/csrc/tc_gemm.cu"
#include "../../paper_2110_12782_b200/csrc/sketch_tc.cu"
#include <cstdio>
#include <vector>
using namespace netmfp;
namespace netmfp { void set_last_error(const std::string &) {} void dist_allreduce(Ctx &, void *, size_t, DType) {} }
int main() {
  Ctx c; cudaStreamCreate(&c.stream);
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0); c.num_sms = prop.multiProcessorCount;
  const int64_t n = 1 << 20, k = 256, h = 228, z = 8;
  float *A, *F, *Y, *sg; int32_t *rows;
  cudaMalloc(&A, n * k * 4); cudaMalloc(&F, n * k * 4); cudaMalloc(&Y, n * 256 * 4);
  cudaMalloc(&rows, h * z * 4); cudaMalloc(&sg, h * z * 4);
  cudaMemset(A, 0, n * k * 4); cudaMemset(F, 0, n * k * 4);
  std::vector<int32_t> hr(h * z); std::vector<float> hs(h * z);
  for (int i = 0; i < h * z; ++i) { hr[i] = (i * 7919) % n; hs[i] = (i & 1) ? 1.f : -1.f; }
  cudaMemcpy(rows, hr.data(), h * z * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(sg, hs.data(), h * z * 4, cudaMemcpyHostToDevice);
  Mat Fm{F, n, k, k}, Ym{Y, n, h, 256};
  double *Cd; cudaMalloc(&Cd, k * k * 8);
  { std::vector<double> I(k * k, 0.0); for (int i = 0; i < k; ++i) I[i * k + i] = 1.0; cudaMemcpy(Cd, I.data(), k * k * 8, cudaMemcpyHostToDevice); }
  { std::vector<float> hf(n * k); for (int64_t i = 0; i < n * k; ++i) hf[i] = ((i * 2654435761u) % 1000) * 1e-3f - 0.5f; cudaMemcpy(F, hf.data(), n * k * 4, cudaMemcpyHostToDevice); }
  try {
    for (int rep = 0; rep < 3; ++rep) {
      unsigned long long zero[148 * 8] = {};
      cudaMemcpyToSymbol(g_skprof, zero, sizeof(zero));
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, c.stream);
      tc_sketch_y(c, Fm, Cd, k, rows, sg, h, z, 6e5f, 0, Ym, 0);
      cudaEventRecord(e1, c.stream);
      cudaStreamSynchronize(c.stream);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long hp[148 * 8];
      cudaMemcpyFromSymbol(hp, g_skprof, sizeof(hp));
      double tot[8] = {};
      for (int b = 0; b < 148; ++b) for (int i = 0; i < 8; ++i) tot[i] += hp[b * 8 + i] / 148.0;
      printf("%.3f ms (%s): cycles/CTA  prod-wait-empty %.0f  mma-wait-tfree %.0f  mma-wait-split %.0f  split-wait-full %.0f  epi-wait-done %.0f  epi-work %.0f\n",
             ms, cudaGetErrorString(cudaGetLastError()), tot[0], tot[1], tot[2], tot[3], tot[4], tot[5]);
    }
  } catch (std::exception &e) { printf("exc %s\n", e.what()); }
  return 0;
}
