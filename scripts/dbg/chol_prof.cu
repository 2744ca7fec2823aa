#define CDF_PROF
#include "../../paper_2110_12782_b200/csrc/chol_df.cu"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace netmfp;
namespace netmfp { void set_last_error(const std::string &) {} }
int main() {
  Ctx c; cudaStreamCreate(&c.stream);
  const int l = 286;
  std::vector<double> h(l * l);
  // SPD: G = B Bᵀ + l I
  for (int i = 0; i < l; ++i) for (int j = 0; j < l; ++j) h[i * l + j] = (i == j ? l : 0.0) + 1.0 / (1 + abs(i - j));
  double *G, *R; int *flag;
  cudaMalloc(&G, l * l * 8); cudaMalloc(&R, l * l * 8); cudaMalloc(&flag, 4); cudaMemset(flag, 0, 4);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(G, h.data(), l * l * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, c.stream);
    chol_inv_df(c, G, l, l, R, flag, 0.0);
    cudaEventRecord(e1, c.stream);
    cudaStreamSynchronize(c.stream);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long t[64 * 16];
    cudaMemcpyFromSymbol(t, g_cdf_t, sizeof(t));
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < 37; ++b) t0 = std::min(t0, t[b * 16]);
    double mx[7] = {};
    for (int b = 0; b < 37; ++b) for (int i = 0; i < 7; ++i) mx[i] = std::max(mx[i], (double)(t[b * 16 + i] - t0));
    if (rep == 2) {
      const int nb = 9;
      int base = 0;
      for (int J = 0; J < nb; ++J) {
        const int d = base, o = base + 1;  // (J,J) and (J+1,J)
        printf("   m9 %.2f m10 %.2f m12 %.2f m14 %.2f m11 %.2f\n", (t[d*16+9]-t0)/1e3, (t[d*16+10]-t0)/1e3, (t[d*16+12]-t0)/1e3, (t[d*16+14]-t0)/1e3, (t[d*16+11]-t0)/1e3);
        printf("J=%d diag: upd_done %.2f fact_done %.2f pub %.2f | offdiag(J+1,J): upd_done %.2f pub %.2f\n", J,
               (t[d * 16 + 4] - t0) / 1e3, (t[d * 16 + 11] - t0) / 1e3, (t[d * 16 + 7] - t0) / 1e3,
               J + 1 < nb ? (t[o * 16 + 4] - t0) / 1e3 : 0.0, J + 1 < nb ? (t[o * 16 + 7] - t0) / 1e3 : 0.0);
        base += nb - J;
      }
    }
    printf("\n%.3f ms %s | max over CTAs (us): start %.1f g0sync %.1f chol %.1f sync %.1f inv %.1f sync %.1f end %.1f\n", ms,
           cudaGetErrorString(cudaGetLastError()), mx[0] / 1e3, mx[1] / 1e3, mx[2] / 1e3, mx[3] / 1e3, mx[4] / 1e3,
           mx[5] / 1e3, mx[6] / 1e3);
  }
  return 0;
}
