#define TD_PROF
#include "../../paper_2110_12782_b200/csrc/small.cu"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace netmfp;
namespace netmfp { void set_last_error(const std::string &) {} void chol_inv_df(Ctx &, double *, int64_t, int64_t, double *, int *) {} }
int main() {
  Ctx c; cudaStreamCreate(&c.stream); c.num_sms = 148;
  const int l = 286;
  std::vector<double> h(l * l);
  for (int i = 0; i < l; ++i) for (int j = 0; j < l; ++j) h[i * l + j] = 1.0 / (1 + abs(i - j)) + (i == j ? 2.0 : 0.0);
  double *S, *lam, *V;
  cudaMalloc(&S, l * l * 8); cudaMalloc(&lam, l * 8); cudaMalloc(&V, l * l * 8);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(S, h.data(), l * l * 8, cudaMemcpyHostToDevice);
    sym_eig(c, S, l, lam, V, true);
    cudaStreamSynchronize(c.stream);
  }
  static unsigned long long t[8][4][512];
  cudaMemcpyFromSymbol(t, g_td_t, sizeof(t));
  double a01 = 0, a12 = 0, a23 = 0, a30 = 0; int n = 0;
  for (int j = 10; j + 3 < l - 10; ++j) {
    // rank 0 phases: start->owner done (1), S1 wait (2), matvec/push (3), S2 + update -> next start
    a01 += t[0][1][j] - t[0][0][j]; a12 += t[0][2][j] - t[0][1][j]; a23 += t[0][3][j] - t[0][2][j];
    a30 += t[0][0][j + 1] - t[0][3][j]; ++n;
  }
  printf("per step (ns, rank 0): reflector %.0f  S1 %.0f  matvec+push %.0f  S2+update %.0f  total %.0f\n", a01 / n, a12 / n,
         a23 / n, a30 / n, (a01 + a12 + a23 + a30) / n);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
