// sketch.cu — rows a5-a7: sparse-sign matrices (Alg. 3),
// the sketch entry point (Eq. 5; the fused tensor-core kernel is in
// sketch_tc.cu) and the signed gathers Ψᵀ X / Πᵀ X of Alg. 4 steps 6-7.

#include "common.cuh"
#include "kernels.cuh"

namespace netmfp {

// ---------------------------------------------------------------------------
// Alg. 3: column j draws z distinct rows by sequential rejection from the
// Philox stream (j, r, 0, tag); sign = +1 if w1 even [R1]
// ---------------------------------------------------------------------------
constexpr int kMaxZ = 64;

__global__ void k_ss_gen(int64_t n, int64_t h, int z, uint32_t k0, uint32_t k1, uint32_t tag,
                         int32_t *__restrict__ rows, float *__restrict__ signs) {
  grid_dep_enter();
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= h) return;
  int32_t chosen[kMaxZ];
  int cnt = 0;
  uint32_t r = 0;
  while (cnt < z) {
    U4 w = philox4x32_10(U4{(uint32_t)j, r, 0u, tag}, k0, k1);
    ++r;
    int32_t row = (int32_t)(((uint64_t)w.x * (uint64_t)n) >> 32);
    bool dup = false;
    for (int t = 0; t < cnt; ++t) dup |= (chosen[t] == row);
    if (dup) continue;
    chosen[cnt] = row;
    rows[j * z + cnt] = row;
    signs[j * z + cnt] = (w.y & 1u) ? -1.f : 1.f;
    ++cnt;
  }
}

void gen_sparse_sign(Ctx &c, int64_t n, int64_t h, int64_t z, uint64_t seed, uint32_t tag, SparseSign &S) {
  NM_REQUIRE(z >= 2 && z <= n && z <= kMaxZ, "sparse-sign: need 2 <= z <= min(n, 64)");
  NM_REQUIRE(h >= 1, "sparse-sign: h >= 1");
  const int64_t cnt = h * z;
  S.n = n; S.h = h; S.z = z;
  S.rows.alloc(cnt, c.stream);
  S.signs.alloc(cnt, c.stream);
  NM_LAUNCH(c, "ss_gen", launch_pdl(c.stream, k_ss_gen, ceil_div(h, 128), 128, 0, n, h, (int)z, (uint32_t)(seed & 0xFFFFFFFFu),
                                                                           (uint32_t)(seed >> 32), tag, S.rows, S.signs));
}

// Out[j, :] = Σ_t sign[j,t] X[rows[j,t], :]  (fp64 accumulate)
__global__ void k_sign_gather(const int32_t *__restrict__ rows, const float *__restrict__ signs, int64_t h, int z,
                              Mat X, int64_t row0, double *__restrict__ Out, int64_t ldo) {
  grid_dep_enter();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= h * X.cols) return;
  int64_t j = idx / X.cols, cc = idx % X.cols;
  double s = 0.0;
  for (int t = 0; t < z; ++t) {
    const int64_t r = (int64_t)rows[j * z + t] - row0;
    if (r >= 0 && r < X.rows) s += (double)signs[j * z + t] * (double)X.p[r * X.ld + cc];
  }
  Out[j * ldo + cc] = s;
}

void sign_gather_T(Ctx &c, const SparseSign &S, const Mat &X, double *Out, int64_t ldo, int64_t row0) {
  NM_LAUNCH(c, "sign_gather", launch_pdl(c.stream, k_sign_gather, ceil_div(S.h * X.cols, 256), 256, 0, S.rows, S.signs, S.h, (int)S.z, X, row0, Out, ldo));
}

__global__ void k_f32_to_f64(const float *__restrict__ src, int64_t lds, double *__restrict__ dst, int64_t ldd,
                             int64_t rows, int64_t cols) {
  grid_dep_enter();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  dst[(idx / cols) * ldd + idx % cols] = (double)src[(idx / cols) * lds + idx % cols];
}

void f32_to_f64(Ctx &c, const float *src, int64_t lds, double *dst, int64_t ldd, int64_t rows, int64_t cols) {
  NM_LAUNCH(c, "f32_to_f64", launch_pdl(c.stream, k_f32_to_f64, ceil_div(rows * cols, 256), 256, 0, src, lds, dst, ldd, rows,
                                                                                              cols));
}

}  // namespace netmfp
