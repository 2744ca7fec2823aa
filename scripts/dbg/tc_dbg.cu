// Debug harness: builds the library's TC kernels standalone and checks small cases.
#include "../../paper_2110_12782_b200/csrc/tc_gemm.cu"
#include <cstdio>
#include <cmath>
using namespace netmfp;
namespace netmfp { void set_last_error(const std::string &) {} }
int main() {
  Ctx c;
  cudaStreamCreate(&c.stream);
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0); c.num_sms = prop.multiProcessorCount;
  try {
    // tall GEMM: C[n×b] = A[n×K] B[K×b]
    for (int trial = 0; trial < 2; ++trial) {
      int n = 300, K = trial ? 64 : 32, b = 48;
      std::vector<float> hA(n * 64, 0.f); std::vector<double> hB(K * b);
      for (int i = 0; i < n; ++i) for (int k = 0; k < K; ++k) hA[i * 64 + k] = (float)((i * 7 + k * 3) % 11) - 5.f;
      for (int k = 0; k < K; ++k) for (int j = 0; j < b; ++j) hB[k * b + j] = (k == j) ? 1.0 : ((k + j) % 5 == 0 ? 0.5 : 0.0);
      float *dA, *dC; double *dB;
      cudaMalloc(&dA, n * 64 * 4); cudaMalloc(&dC, n * 64 * 4); cudaMalloc(&dB, K * b * 8);
      cudaMemcpy(dA, hA.data(), n * 64 * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, hB.data(), K * b * 8, cudaMemcpyHostToDevice);
      cudaMemset(dC, 0, n * 64 * 4);
      Mat A{dA, n, K, 64}, C{dC, n, b, 64};
      tc_gemm_tall(c, A, dB, b, b, nullptr, 0.f, C);
      cudaError_t e = cudaStreamSynchronize(c.stream);
      std::vector<float> hC(n * 64);
      cudaMemcpy(hC.data(), dC, n * 64 * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0; int bad = 0;
      for (int i = 0; i < n; ++i) for (int j = 0; j < b; ++j) {
        double r = 0; for (int k = 0; k < K; ++k) r += hA[i * 64 + k] * hB[k * b + j];
        double d = fabs(r - hC[i * 64 + j]); if (d > 1e-4) { if (bad < 5) printf("gemm bad (%d,%d) got %f ref %f\n", i, j, hC[i*64+j], r); bad++; }
        maxerr = fmax(maxerr, d);
      }
      printf("gemm trial %d err=%s maxerr=%g bad=%d\n", trial, cudaGetErrorString(e), maxerr, bad);
    }
    // gram: G = AᵀA
    for (int trial = 0; trial < 3; ++trial) {
      int n = trial == 0 ? 32 : 1000, a = trial == 2 ? 64 : 32;
      std::vector<float> hA(n * 64, 0.f);
      for (int i = 0; i < n; ++i) for (int k = 0; k < a; ++k) hA[i * 64 + k] = (float)((i * 5 + k * 3) % 7) - 3.f;
      float *dA; double *dG;
      cudaMalloc(&dA, n * 64 * 4); cudaMalloc(&dG, a * a * 8);
      cudaMemcpy(dA, hA.data(), n * 64 * 4, cudaMemcpyHostToDevice);
      cudaMemset(dG, 0, a * a * 8);
      Mat A{dA, n, a, 64};
      tc_gram(c, A, A, nullptr, 0.f, dG, a);
      cudaError_t e = cudaStreamSynchronize(c.stream);
      std::vector<double> hG(a * a);
      cudaMemcpy(hG.data(), dG, a * a * 8, cudaMemcpyDeviceToHost);
      double maxerr = 0; int bad = 0;
      for (int i = 0; i < a; ++i) for (int j = 0; j < a; ++j) {
        double r = 0; for (int k = 0; k < n; ++k) r += (double)hA[k * 64 + i] * hA[k * 64 + j];
        double d = fabs(r - hG[i * a + j]); if (d > 1e-3) { if (bad < 8) printf("gram bad (%d,%d) got %f ref %f\n", i, j, hG[i*a+j], r); bad++; }
        maxerr = fmax(maxerr, d);
      }
      printf("gram trial %d err=%s maxerr=%g bad=%d\n", trial, cudaGetErrorString(e), maxerr, bad);
    }
  } catch (std::exception &ex) { printf("exception: %s\n", ex.what()); }
  return 0;
}
