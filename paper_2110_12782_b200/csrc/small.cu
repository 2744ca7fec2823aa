// small.cu — fp64 dense kernels for the l×l problems of Alg. 2/4 (l <= ~460):
//   * cholesky_upper  — CholeskyQR's R (north_star; [R7]); left-looking blocked,
//                       one CTA, 32-column panels in shared memory, device-side
//                       shifted retry on breakdown
//   * tri_inv_upper   — R^-1, one warp per column
//   * sym_eig         — eig(S) of Alg. 2 step 8 / svd(S) of Alg. 4 step 8:
//                       Householder tridiagonalisation on an 8-CTA cluster with
//                       the matrix resident in distributed shared memory,
//                       bisection (Sturm counts) for eigenvalues, inverse
//                       iteration with in-cluster modified Gram–Schmidt for
//                       eigenvectors, reflector back-transformation
//   * gemm64 and small helpers
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace netmfp {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
__device__ double block_sum(double v, double *red) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32, ln = threadIdx.x % 32;
  __syncthreads();
  if (ln == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (threadIdx.x < NT / 32) ? red[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// ---------------------------------------------------------------------------
// gemm64: C = alpha op(A) op(B) + beta C
// ---------------------------------------------------------------------------
// 32×32 output tile per 256-thread CTA (2×2 per thread), K in steps of 32
// with the next step's operands prefetched into registers while the current
// one is consumed from shared memory (small l×l problems: the grid, not the
// FMA rate, is what limits them, so tiles are small and many).  Long K is
// split over the CTAs of a cluster (gridDim.z = cluster size); rank 0 adds
// the other ranks' partial tiles from their shared memory in rank order
// (deterministic).
__global__ void __launch_bounds__(256) k_gemm64(bool ta, bool tb, int64_t M, int64_t N, int64_t K,
                                                double alpha, const double *__restrict__ A, int64_t lda,
                                                const double *__restrict__ B, int64_t ldb, double beta,
                                                double *__restrict__ C, int64_t ldc) {
  grid_dep_enter();
  __shared__ double As[32][33];  // [k][m]
  __shared__ double Bs[32][33];  // [k][n]
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.y * 32, n0 = (int64_t)blockIdx.x * 32;
  const int64_t kchunk = (K + 32 * gridDim.z - 1) / (32 * gridDim.z) * 32;
  const int64_t kb = (int64_t)blockIdx.z * kchunk, ke = min(K, kb + kchunk);
  // loader mapping: 4 elements of A and 4 of B per thread per K step
  double ra[4], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + 256 * q;  // 0..1023 over a 32×32 tile
      int kk, mm;
      if (ta) { mm = idx % 32; kk = idx / 32; } else { kk = idx % 32; mm = idx / 32; }  // coalesced source
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[q] = (gm < M && gk < ke) ? (ta ? A[gk * lda + gm] : A[gm * lda + gk]) : 0.0;
      int nn;
      if (tb) { kk = idx % 32; nn = idx / 32; } else { nn = idx % 32; kk = idx / 32; }
      const int64_t gn = n0 + nn, gk2 = k0 + kk;
      rb[q] = (gn < N && gk2 < ke) ? (tb ? B[gn * ldb + gk2] : B[gk2 * ldb + gn]) : 0.0;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + 256 * q;
      if (ta) As[idx / 32][idx % 32] = ra[q]; else As[idx % 32][idx / 32] = ra[q];
      if (tb) Bs[idx % 32][idx / 32] = rb[q]; else Bs[idx / 32][idx % 32] = rb[q];
    }
  };
  double acc[2][2] = {};
  load(kb);
  for (int64_t k0 = kb; k0 < ke; k0 += 32) {
    stash();
    __syncthreads();
    if (k0 + 32 < ke) load(k0 + 32);
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const double a0 = As[kk][ty], a1 = As[kk][ty + 16];
      const double b0 = Bs[kk][tx], b1 = Bs[kk][tx + 16];
      acc[0][0] = fma(a0, b0, acc[0][0]);
      acc[0][1] = fma(a0, b1, acc[0][1]);
      acc[1][0] = fma(a1, b0, acc[1][0]);
      acc[1][1] = fma(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
  if (gridDim.z > 1) {
    __shared__ double part[4][256];
#pragma unroll
    for (int q = 0; q < 4; ++q) part[q][threadIdx.x] = acc[q / 2][q % 2];
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    if (blockIdx.z == 0)
      for (unsigned r = 1; r < gridDim.z; ++r) {
        const double *rp = cl.map_shared_rank(&part[0][0], r);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q / 2][q % 2] += rp[q * 256 + threadIdx.x];
      }
    cl.sync();  // remote partials stay alive until rank 0 has read them
    if (blockIdx.z != 0) return;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
      if (gm < M && gn < N) {
        double *c = C + gm * ldc + gn;
        *c = alpha * acc[i][j] + (beta != 0.0 ? beta * *c : 0.0);
      }
    }
}

void gemm64(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
            int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  const int64_t tiles = ceil_div(N, 32) * ceil_div(M, 32);
  // split K over a cluster while the tile grid leaves SMs idle (<= 2 CTAs per SM)
  int split = 1;
  while (split < 8 && tiles * split * 2 <= 2 * c.num_sms && K >= 64 * split * 2) split *= 2;
  dim3 grid(ceil_div(N, 32), ceil_div(M, 32), split);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = c.stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = split;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  NM_LAUNCH(c, "gemm64", NM_CUDA(cudaLaunchKernelEx(&cfg, k_gemm64, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc)));
}

__global__ void k_symmetrize(double *S, int64_t l, int64_t ld) {
  grid_dep_enter();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t i = idx / l, j = idx % l;
  if (i >= l || j <= i) return;
  double v = 0.5 * (S[i * ld + j] + S[j * ld + i]);
  S[i * ld + j] = v;
  S[j * ld + i] = v;
}
void symmetrize64(Ctx &c, double *S, int64_t l, int64_t ld) {
  NM_LAUNCH(c, "symmetrize", launch_pdl(c.stream, k_symmetrize, ceil_div(l * l, 256), 256, 0, S, l, ld));
}

// mode 0: A[:, j] *= s[j]; mode 1: A[i, :] *= s[i]
__global__ void k_scale64(double *A, int64_t rows, int64_t cols, int64_t ld, const double *s, int mode) {
  grid_dep_enter();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  int64_t i = idx / cols, j = idx % cols;
  A[i * ld + j] *= (mode == 0 ? s[j] : s[i]);
}
void scale_cols64(Ctx &c, double *A, int64_t rows, int64_t cols, int64_t ld, const double *s, int mode) {
  NM_LAUNCH(c, "scale64", launch_pdl(c.stream, k_scale64, ceil_div(rows * cols, 256), 256, 0, A, rows, cols, ld, s, mode));
}

__global__ void k_identity(double *A, int64_t l, int64_t ld) {
  grid_dep_enter();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= l * l) return;
  int64_t i = idx / l, j = idx % l;
  A[i * ld + j] = (i == j) ? 1.0 : 0.0;
}
void set_identity64(Ctx &c, double *A, int64_t l, int64_t ld) {
  NM_LAUNCH(c, "identity", launch_pdl(c.stream, k_identity, ceil_div(l * l, 256), 256, 0, A, l, ld));
}

__global__ void k_axpy64(int64_t n, double a, const double *x, double *y) {
  grid_dep_enter();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}
void axpy64(Ctx &c, int64_t n, double alpha, const double *x, double *y) {
  NM_LAUNCH(c, "axpy64", launch_pdl(c.stream, k_axpy64, ceil_div(n, 256), 256, 0, n, alpha, x, y));
}

// ---------------------------------------------------------------------------
// Cholesky  G = Rᵀ R  (one CTA, left-looking, 32-column panels in smem)
// ---------------------------------------------------------------------------
constexpr int CHP = 32;

__global__ void __launch_bounds__(1024) k_cholesky(double *G, int l, int64_t ld, double *G0, int *flag) {
  grid_dep_enter();
  extern __shared__ double P[];  // (l) x CHP panel
  __shared__ int fail;
  __shared__ double maxdiag;
  const int tid = threadIdx.x, nt = blockDim.x;
  // keep the original for shifted retries
  for (int64_t idx = tid; idx < (int64_t)l * l; idx += nt) G0[idx] = G[(idx / l) * ld + idx % l];
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < l; ++i) m = fmax(m, G0[(int64_t)i * l + i]);
    maxdiag = m;
  }
  __syncthreads();
  for (int attempt = 0; attempt < 6; ++attempt) {
    const double shift = attempt == 0 ? 0.0 : maxdiag * 1e-7 * pow(100.0, (double)(attempt - 1));
    if (attempt > 0) {
      for (int64_t idx = tid; idx < (int64_t)l * l; idx += nt) {
        int64_t i = idx / l, j = idx % l;
        G[i * ld + j] = G0[idx] + (i == j ? shift : 0.0);
      }
    }
    if (tid == 0) fail = 0;
    __syncthreads();
    for (int J = 0; J < l && !fail; J += CHP) {
      const int jb = min(CHP, l - J), rows = l - J;
      // panel = G[J:, J:J+jb] - L[J:, :J] L[J:J+jb, :J]^T   (lower part r >= c)
      for (int idx = tid; idx < rows * jb; idx += nt) {
        int r = idx / jb, cc = idx % jb;
        double s = 0.0;
        if (r >= cc) {
          s = G[(int64_t)(J + r) * ld + J + cc];
          const double *Lr = G + (int64_t)(J + r) * ld;
          const double *Lc = G + (int64_t)(J + cc) * ld;
          for (int t = 0; t < J; ++t) s -= Lr[t] * Lc[t];
        }
        P[r * CHP + cc] = s;
      }
      __syncthreads();
      for (int j = 0; j < jb; ++j) {
        if (tid == 0) {
          double piv = P[j * CHP + j];
          const double g0 = G0[(int64_t)(J + j) * l + J + j];
          double ref = g0 + shift;
          if (g0 == 0.0) P[j * CHP + j] = 1.0;  // exactly-zero column: identity pivot [R10]
          else if (!(piv > 1e-12 * ref) || !isfinite(piv)) fail = 1;
          else P[j * CHP + j] = sqrt(piv);
        }
        __syncthreads();
        if (fail) break;
        const double pj = P[j * CHP + j];
        for (int r = j + 1 + tid; r < rows; r += nt) P[r * CHP + j] /= pj;
        __syncthreads();
        const int w = jb - j - 1;
        for (int idx = tid; idx < (rows - j - 1) * w; idx += nt) {
          int r = j + 1 + idx / w, cc = j + 1 + idx % w;
          if (r >= cc) P[r * CHP + cc] -= P[r * CHP + j] * P[cc * CHP + j];
        }
        __syncthreads();
      }
      if (fail) break;
      for (int idx = tid; idx < rows * jb; idx += nt) {
        int r = idx / jb, cc = idx % jb;
        if (r >= cc) G[(int64_t)(J + r) * ld + J + cc] = P[r * CHP + cc];
      }
      __syncthreads();
    }
    __syncthreads();
    if (!fail) {
      if (attempt > 0 && tid == 0) atomicAdd(flag, 1);
      // R = L^T in the upper triangle, zero the strict lower
      for (int64_t idx = tid; idx < (int64_t)l * l; idx += nt) {
        int64_t i = idx / l, j = idx % l;
        if (j > i) G[i * ld + j] = G[j * ld + i];
      }
      __syncthreads();
      for (int64_t idx = tid; idx < (int64_t)l * l; idx += nt) {
        int64_t i = idx / l, j = idx % l;
        if (j < i) G[i * ld + j] = 0.0;
      }
      return;
    }
  }
  if (tid == 0) atomicOr(flag, 1 << 30);
}

void cholesky_upper(Ctx &c, double *G, int64_t l, int64_t ld, int *flag) {
  NM_REQUIRE(l > 0 && l <= 4096, "cholesky: l out of range");
  DBuf<double> G0((size_t)l * l, c.stream);
  size_t smem = (size_t)l * CHP * sizeof(double);
  smem_attr(k_cholesky, 200 * 1024);
  NM_REQUIRE(smem <= 200 * 1024, "cholesky: l too large for one CTA panel");
  NM_LAUNCH(c, "cholesky", launch_pdl(c.stream, k_cholesky, 1, 1024, smem, G, (int)l, ld, G0, flag));
}

// ---------------------------------------------------------------------------
// Fused Cholesky + inverse:  G = Rᵀ R (R upper),  Rinv = R⁻¹  — one CTA.
// L = Rᵀ (lower) is built in place in G's lower triangle by 32-column panels:
//   (a) LsT[t][c] = L[J+c][t] (t < J) staged in shared memory;
//   (b) P[r][c] = G[J+r][J+c] − Σ_t L[J+r][t] LsT[t][c]   (left-looking update);
//   (c) warp 0 factors the 32×32 diagonal block in registers (shuffles only);
//   (d) every thread owning a row below solves against it (forward substitution).
// Then X = L⁻¹ by 32-row block rows: X_II = L_II⁻¹ (warp 0, registers),
// X_IJ = −X_II Σ_K L_IK X_KJ, and finally Rinv = Xᵀ in place.  A breakdown
// (pivot <= 1e-12 · original diagonal, or non-finite) restarts from the saved
// G with a diagonal shift (shifted CholeskyQR), as cholesky_upper does.
// ---------------------------------------------------------------------------
constexpr int CI_T = 512;
constexpr int CI_MAXL = 320;
constexpr int CI_LD = 33;                  // row stride of 32-wide panels
constexpr int CI_R = CI_MAXL * CI_LD;      // doubles per big region
constexpr int CI_K = (CI_MAXL * 32 + CI_T - 1) / CI_T;  // outputs per thread

__global__ void __launch_bounds__(CI_T) k_chol_inv(double *G, int l, int64_t ld, double *G0, double *Rinv,
                                                   int *flag, double drop_tol) {
  grid_dep_enter();
  extern __shared__ double sm[];
  double *R1 = sm;             // phase 1: L rows chunk [rows][33];   phase 2: L_I rows [32][l+1]
  double *R2 = sm + CI_R;      // phase 1: panel P [rows][33];        phase 2: X chunk / T [32][l+1]
  double *R3 = sm + 2 * CI_R;  // phase 1: LsT chunk [32][33];        phase 2: X_II [32][33]
  __shared__ double diag0[CI_MAXL];
  __shared__ unsigned char dropped[CI_MAXL];  // dependent columns of the successful attempt
  __shared__ int fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t idx = tid; idx < (int64_t)l * l; idx += CI_T) G0[idx] = G[(idx / l) * ld + idx % l];
  for (int i = tid; i < l; i += CI_T) diag0[i] = G[(int64_t)i * ld + i];
  __syncthreads();
  double maxdiag = 0.0;
  for (int i = 0; i < l; ++i) maxdiag = fmax(maxdiag, diag0[i]);
  bool ok = false;
  double acc[CI_K];
  for (int attempt = 0; attempt < 6 && !ok; ++attempt) {
    const double shift = attempt == 0 ? 0.0 : maxdiag * 1e-7 * pow(100.0, (double)(attempt - 1));
    if (attempt > 0) {
      for (int64_t idx = tid; idx < (int64_t)l * l; idx += CI_T) {
        const int64_t i = idx / l, j = idx % l;
        G[i * ld + j] = G0[idx] + (i == j ? shift : 0.0);
      }
    }
    if (tid == 0) fail = 0;
    for (int i = tid; i < l; i += CI_T) dropped[i] = 0;
    __syncthreads();
    for (int J = 0; J < l; J += 32) {
      const int jb = min(32, l - J), rows = l - J, np = rows * jb;
      // (b) P = G[J:, J:J+jb] − L[J:, :J] L[J:J+jb, :J]ᵀ, tiled over 32-wide t chunks
#pragma unroll
      for (int k = 0; k < CI_K; ++k) {
        const int idx = tid + k * CI_T;
        acc[k] = idx < np ? G[(int64_t)(J + idx / jb) * ld + J + idx % jb] : 0.0;
      }
      for (int t0 = 0; t0 < J; t0 += 32) {
        for (int idx = tid; idx < rows * 32; idx += CI_T)
          R1[(idx >> 5) * CI_LD + (idx & 31)] = G[(int64_t)(J + (idx >> 5)) * ld + t0 + (idx & 31)];
        for (int idx = tid; idx < jb * 32; idx += CI_T)
          R3[(idx & 31) * CI_LD + (idx >> 5)] = G[(int64_t)(J + (idx >> 5)) * ld + t0 + (idx & 31)];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < CI_K; ++k) {
          const int idx = tid + k * CI_T;
          if (idx < np) {
            const double *a = R1 + (idx / jb) * CI_LD;
            const double *b = R3 + idx % jb;
            double s = 0.0;
#pragma unroll 8
            for (int tt = 0; tt < 32; ++tt) s += a[tt] * b[tt * CI_LD];
            acc[k] -= s;
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int k = 0; k < CI_K; ++k) {
        const int idx = tid + k * CI_T;
        if (idx < np) {
          const int r = idx / jb, cc = idx % jb;
          R2[r * CI_LD + cc] = (r < jb && r < cc) ? 0.0 : acc[k];
        }
      }
      __syncthreads();
      // (c) diagonal block by warp 0, lane r = row r
      if (warp == 0) {
        bool bad = false;
        for (int j = 0; j < jb; ++j) {
          // an exactly-zero column of the Gram's input (zero row and column
          // of G) gets an identity pivot: that column of Y R⁻¹ stays zero and
          // the others are untouched — orth on range(Y) [R10]
          const bool zc = diag0[J + j] == 0.0;
          double d = zc ? 1.0 : R2[j * CI_LD + j];
          // numerically dependent column of an orthonormalising pass [R10]
          const bool dr = !zc && drop_tol > 0.0 && isfinite(d) && d < drop_tol * (diag0[J + j] + shift);
          if (dr) {
            d = 1.0;
            if (lane == 0) dropped[J + j] = 1;
          }
          if (!zc && !dr && (!(d > 1e-12 * (diag0[J + j] + shift)) || !isfinite(d))) bad = true;
          const double sq = sqrt(fmax(d, 1e-300));
          __syncwarp();
          if (lane == j) R2[j * CI_LD + j] = sq;
          if (lane > j && lane < jb) R2[lane * CI_LD + j] /= sq;
          __syncwarp();
          if (lane > j && lane < jb) {
            const double lr = R2[lane * CI_LD + j];
            for (int cc = j + 1; cc <= lane; ++cc) R2[lane * CI_LD + cc] -= lr * R2[cc * CI_LD + j];
          }
          __syncwarp();
        }
        if (bad && lane == 0) fail = 1;
      }
      __syncthreads();
      if (fail) break;
      // (d) rows below the diagonal block: forward substitution
      for (int r = jb + tid; r < rows; r += CI_T) {
        double *Pr = R2 + r * CI_LD;
        for (int cc = 0; cc < jb; ++cc) {
          double v = Pr[cc];
          for (int t = 0; t < cc; ++t) v -= Pr[t] * R2[cc * CI_LD + t];
          Pr[cc] = v / R2[cc * CI_LD + cc];
        }
      }
      __syncthreads();
      for (int idx = tid; idx < np; idx += CI_T) {
        const int r = idx / jb, cc = idx % jb;
        if (r >= cc) G[(int64_t)(J + r) * ld + J + cc] = R2[r * CI_LD + cc];
      }
      __syncthreads();
    }
    __syncthreads();
    ok = !fail;
    if (ok && attempt > 0 && tid == 0) atomicAdd(flag, 1);
  }
  if (!ok) {
    if (tid == 0) atomicOr(flag, 1 << 30);
    return;
  }
  // ---- X = L⁻¹ (lower, row-major in Rinv), block row by block row
  const int WL = l + 1;
  for (int I = 0; I < l; I += 32) {
    const int ib = min(32, l - I), nt = ib * I;
    for (int idx = tid; idx < ib * (I + ib); idx += CI_T) {
      const int r = idx / (I + ib), t = idx % (I + ib);
      R1[r * WL + t] = G[(int64_t)(I + r) * ld + t];
    }
    __syncthreads();
    // (i) X_II = L_II⁻¹ (warp 0; lane = column)
    if (warp == 0) {
      for (int r = 0; r < 32; ++r) {
        double v = 0.0;
        if (r < ib && lane < ib && r >= lane) {
          v = (r == lane) ? 1.0 : 0.0;
          const double *Lr = R1 + r * WL + I;
          for (int t = lane; t < r; ++t) v -= Lr[t] * R3[t * CI_LD + lane];
          v /= Lr[r];
        }
        R3[r * CI_LD + lane] = v;
        __syncwarp();
      }
    }
    // (ii) T = L[I:I+ib, :I] · X[:I, :I], tiled over 32-row chunks of X
#pragma unroll
    for (int k = 0; k < CI_K; ++k) acc[k] = 0.0;
    for (int t0 = 0; t0 < I; t0 += 32) {
      for (int idx = tid; idx < 32 * I; idx += CI_T) {
        const int tt = idx / I, cc = idx % I;
        R2[tt * WL + cc] = Rinv[(int64_t)(t0 + tt) * l + cc];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < CI_K; ++k) {
        const int idx = tid + k * CI_T;
        if (idx < nt) {
          const double *a = R1 + (idx / I) * WL + t0;
          const double *b = R2 + idx % I;
          double s = 0.0;
#pragma unroll 8
          for (int tt = 0; tt < 32; ++tt) s += a[tt] * b[tt * WL];
          acc[k] += s;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < CI_K; ++k) {
      const int idx = tid + k * CI_T;
      if (idx < nt) R2[(idx / I) * WL + idx % I] = acc[k];
    }
    __syncthreads();
    // (iii) X[I+r][c] = −Σ_s X_II[r][s] T[s][c] (c < I); diagonal block = X_II
    for (int idx = tid; idx < ib * l; idx += CI_T) {
      const int r = idx / l, cc = idx % l;
      double v = 0.0;
      if (cc < I) {
        for (int s2 = 0; s2 <= r; ++s2) v -= R3[r * CI_LD + s2] * R2[s2 * WL + cc];
      } else if (cc < I + ib) {
        v = R3[r * CI_LD + (cc - I)];
      }
      Rinv[(int64_t)(I + r) * l + cc] = v;
    }
    __syncthreads();
  }
  // ---- Rinv = Xᵀ (upper) in place
  for (int64_t idx = tid; idx < (int64_t)l * l; idx += CI_T) {
    const int64_t i = idx / l, j = idx % l;
    if (i < j) {
      const double v = Rinv[j * l + i];
      Rinv[i * l + j] = v;
      Rinv[j * l + i] = 0.0;
    }
  }
  __syncthreads();
  // dependent columns: zero columns of R⁻¹ (Q's column comes out exactly zero)
  for (int64_t idx = tid; idx < (int64_t)l * l; idx += CI_T)
    if (dropped[idx % l]) Rinv[idx] = 0.0;
}

void chol_inv_upper(Ctx &c, double *G, int64_t l, int64_t ld, double *Rinv, int *flag, double drop_tol) {
  // tile dataflow on many SMs while the lower triangle fits in co-resident CTAs
  if (l > 64 && (l + 31) / 32 * ((l + 31) / 32 + 1) / 2 <= c.num_sms) {
    chol_inv_df(c, G, l, ld, Rinv, flag, drop_tol);
    return;
  }
  if (l > CI_MAXL) {
    cholesky_upper(c, G, l, ld, flag);
    tri_inv_upper(c, G, ld, Rinv, l);
    return;
  }
  DBuf<double> G0((size_t)l * l, c.stream);
  const size_t smem = ((size_t)2 * CI_R + 32 * CI_LD) * sizeof(double);
  smem_attr(k_chol_inv, smem);
  NM_LAUNCH(c, "chol_inv", launch_pdl(c.stream, k_chol_inv, 1, CI_T, smem, G, (int)l, ld, G0, Rinv, flag, drop_tol));
}

// ---------------------------------------------------------------------------
// Rinv = R^-1 (upper), one warp per column, x in shared memory
// ---------------------------------------------------------------------------
__global__ void k_trinv(const double *__restrict__ R, int64_t ld, double *__restrict__ Rinv, int l) {
  grid_dep_enter();
  extern __shared__ double xs[];
  const int w = threadIdx.x / 32, ln = threadIdx.x % 32;
  const int j = blockIdx.x * (blockDim.x / 32) + w;
  if (j >= l) return;
  double *x = xs + (int64_t)w * l;
  for (int i = j; i >= 0; --i) {
    double s = 0.0;
    for (int k = i + 1 + ln; k <= j; k += 32) s += R[(int64_t)i * ld + k] * x[k];
    s = warp_sum(s);
    if (ln == 0) x[i] = ((i == j ? 1.0 : 0.0) - s) / R[(int64_t)i * ld + i];
    __syncwarp();
  }
  for (int i = ln; i < l; i += 32) Rinv[(int64_t)i * l + j] = (i <= j) ? x[i] : 0.0;
}

void tri_inv_upper(Ctx &c, const double *R, int64_t ld, double *Rinv, int64_t l) {
  const int wpb = 8;
  size_t smem = (size_t)wpb * l * sizeof(double);
  smem_attr(k_trinv, 200 * 1024);
  NM_REQUIRE(smem <= 200 * 1024, "tri_inv: l too large");
  NM_LAUNCH(c, "trinv", launch_pdl(c.stream, k_trinv, ceil_div(l, wpb), wpb * 32, smem, R, ld, Rinv, (int)l));
}

// ---------------------------------------------------------------------------
// symmetric eigensolver
// ---------------------------------------------------------------------------
#ifdef TD_PROF
__device__ unsigned long long g_td_t[8][4][512];
#define TD_MARK(ph)                                                        \
  do {                                                                     \
    if (threadIdx.x == 0 && j < 512) {                                     \
      unsigned long long _t;                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));               \
      g_td_t[rank][ph][j] = _t;                                            \
    }                                                                      \
  } while (0)
#else
#define TD_MARK(ph)
#endif
constexpr int TDC = 8;     // cluster size (CTAs) for the tridiagonalisation (4 and 16: measured slower)
// split cluster barrier (every thread arrives; release / acquire at cluster scope)
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
constexpr int TDT = 512;   // threads per CTA
static_assert(TDT / 32 == 16, "tridiagonalisation partial slots assume 16 warps");

// Householder tridiagonalisation Qᵀ S Q = T, Q = H_0 … H_{l-3}, H_j = I - beta_j v_j v_jᵀ
// (v_j non-zero on indices j+1..l-1, stored in row j of Hv).  Row i of S lives in
// CTA i % TDC of the cluster (local row i / TDC).  Step j, with p = beta A v and
// K = beta vᵀp / 2:  A -= v pᵀ + p vᵀ - 2K v vᵀ  (= v wᵀ + w vᵀ, w = p - K v).
// Every exchange is a PUSH into the other CTAs' shared memory (remote stores,
// no remote loads on the critical path) and a step costs two cluster barriers:
//   S1: the owner of row j has pushed v_j and beta_j (split arrive / wait:
//       the owner updates row j first during step j-1's update, pushes the
//       reflector and arrives before updating its other rows — look-ahead);
//   S2: every CTA has pushed its rows' p_i and its partial vᵀp.
// v and beta (pushed before S1) are double-buffered by step parity: a buffer
// is rewritten two steps later, after every CTA has passed the barrier that
// follows its last read.  p and the partials are pushed after S1 and are
// double-buffered the same way (the owner of step j+1 arrives at S1(j+1)
// before its other rows are updated with p_j, so step j+1's pushes must not
// land in p_j's buffer).
__global__ void __cluster_dims__(TDC, 1, 1) __launch_bounds__(TDT)
    k_tridiag(const double *__restrict__ S, int l, double *__restrict__ dd, double *__restrict__ ee,
              double *__restrict__ Hv, double *__restrict__ hbeta) {
  grid_dep_enter();
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x, nt = blockDim.x;
  const int wid = tid / 32, ln = tid % 32;
  const int nloc = (l - rank + TDC - 1) / TDC;
  // identical shared-memory layout in every CTA (DSMEM addresses are mapped
  // rank to rank), sized for the largest per-rank row count
  const int nmax = (l + TDC - 1) / TDC;
  extern __shared__ double sm[];
  double *A = sm;                          // nmax × l (first nloc rows used)
  double *vbuf = A + (int64_t)nmax * l;    // 2 × l
  double *pfb = vbuf + 2 * l;              // 2 × l (p, double-buffered like v)
  double *red = pfb + 2 * l;               // 40
  double *xchg = red + 40;                 // [parity][TDC][16 warps] partials, [32 TDC + parity] beta
  for (int64_t idx = tid; idx < (int64_t)nloc * l; idx += nt) {
    int li = (int)(idx / l), k = (int)(idx % l);
    A[idx] = S[(int64_t)(li * TDC + rank) * l + k];
  }
  __syncthreads();
  // reflector of step j from row j (entries j+1..l-1; owner CTA only), pushed
  // with beta_j to every CTA's parity buffer
  // The reflector's global outputs (Hv row j, d_j, e_j, beta_j) are written
  // AFTER the owner arrives at S1: the barrier's release waits for every
  // outstanding store of the CTA, and global stores to L2 pending at the
  // arrive held the owner (and with it the whole cluster) ~1000 cycles per
  // step (ncu: ERRBAR).  Each thread keeps the one entry it computed (l <= nt).
  int hk = -1;
  double hv = 0.0, h_alpha = 0.0, h_beta = 0.0, h_d = 0.0;
  auto reflector = [&](int j) {
    const int par = j & 1;
    double *v = vbuf + par * l;
    const double *x = A + (int64_t)(j / TDC) * l;
    double ss = 0.0;
    for (int k = j + 2 + tid; k < l; k += nt) ss += x[k] * x[k];
    ss = block_sum<TDT>(ss, red);
    const double x0 = x[j + 1];
    double beta = 0.0, alpha = x0, v0 = 0.0;
    if (ss > 0.0) {
      const double nrm = sqrt(ss + x0 * x0);
      alpha = x0 >= 0 ? -nrm : nrm;
      v0 = x0 - alpha;
      beta = 2.0 / (ss + v0 * v0);
    }
    hk = -1;
    for (int k = j + 1 + tid; k < l; k += nt) {
      const double val = ss > 0.0 ? (k == j + 1 ? v0 : x[k]) : 0.0;
#pragma unroll
      for (int r = 0; r < TDC; ++r) cl.map_shared_rank(v, r)[k] = val;
      hk = k;
      hv = val;
    }
    if (tid < TDC) cl.map_shared_rank(xchg, tid)[32 * TDC + par] = beta;
    h_alpha = alpha;
    h_beta = beta;
    h_d = x[j];
  };
  auto reflector_out = [&](int j) {  // after the arrive
    if (hk >= 0) Hv[(int64_t)j * l + hk] = hv;
    if (tid == 0) {
      dd[j] = h_d;
      ee[j] = h_alpha;
      hbeta[j] = h_beta;
    }
  };
  if (l >= 3 && rank == 0) reflector(0);
  cluster_arrive();  // S1(0)
  if (l >= 3 && rank == 0) reflector_out(0);
  for (int j = 0; j + 2 < l; ++j) {
    const int par = j & 1;
    const double *v = vbuf + par * l;
    double *pf = pfb + par * l;
    TD_MARK(0);
    TD_MARK(1);
    cluster_wait();  // S1(j): v_j, beta_j pushed
    TD_MARK(2);
    const double beta = xchg[32 * TDC + par];
    // (2) p_i = beta A[i, j+1:] · v for own rows i > j, pushed to every CTA by
    // the warp that computed it; per-warp partials of vᵀp pushed likewise
    // (no CTA barrier in this phase)
    double part = 0.0;
    for (int li = wid; li < nloc; li += nt / 32) {
      const int i = li * TDC + rank;
      if (i <= j) continue;
      const double *Ai = A + (int64_t)li * l;
      double sacc = 0.0;
      for (int k = j + 1 + ln; k < l; k += 32) sacc += Ai[k] * v[k];
      sacc = warp_sum(sacc) * beta;
      if (ln < TDC) cl.map_shared_rank(pf, ln)[i] = sacc;
      part += sacc * v[i];
    }
    if (ln < TDC) cl.map_shared_rank(xchg, ln)[par * TDC * 16 + rank * 16 + wid] = part;
    TD_MARK(3);
    cl.sync();  // S2
    double vtp = 0.0;
    for (int q = ln; q < TDC * 16; q += 32) vtp += xchg[par * TDC * 16 + q];
    vtp = warp_sum(vtp);
    const double K2 = vtp * beta;  // 2K
    // (4) A_i -= v_i p + p_i v - 2K v_i v  (own rows i > j, columns > j).
    // Look-ahead: the owner of step j+1 updates row j+1 first, then builds
    // and pushes reflector j+1 and arrives at S1(j+1) before its other rows.
    const int jn = j + 1;
    const bool next_owner = jn + 2 < l && rank == jn % TDC;
    if (next_owner) {
      double *Ai = A + (int64_t)(jn / TDC) * l;
      const double vi = v[jn], pi = pf[jn], ci = pi - K2 * vi;
      for (int k = j + 1 + tid; k < l; k += nt) Ai[k] -= vi * pf[k] + ci * v[k];
      __syncthreads();
      reflector(jn);
      cluster_arrive();  // S1(j+1)
      reflector_out(jn);
    }
    for (int li = wid; li < nloc; li += nt / 32) {
      const int i = li * TDC + rank;
      if (i <= j || (next_owner && i == jn)) continue;
      double *Ai = A + (int64_t)li * l;
      const double vi = v[i], pi = pf[i], ci = pi - K2 * vi;
      for (int k = j + 1 + ln; k < l; k += 32) Ai[k] -= vi * pf[k] + ci * v[k];
    }
    if (!next_owner) cluster_arrive();  // S1(j+1): this CTA is done with v_j, pf and the partials
    // CTA barrier: rows of this step are final before the next owner reads them
    __syncthreads();
  }
  if (l >= 3) cluster_wait();  // the last arrive (S1 after the final step)
  // trailing 2×2 (or 1×1)
  if (l >= 2) {
    const int i0 = l - 2, i1 = l - 1;
    if (rank == i0 % TDC && tid == 0) {
      dd[i0] = A[(int64_t)(i0 / TDC) * l + i0];
      ee[i0] = A[(int64_t)(i0 / TDC) * l + i1];
    }
    if (rank == i1 % TDC && tid == 0) dd[i1] = A[(int64_t)(i1 / TDC) * l + i1];
  } else if (rank == 0 && tid == 0) {
    dd[0] = A[0];
  }
  cl.sync();  // no CTA may exit while others still read its shared memory
}

// Sturm count: number of eigenvalues of T strictly less than x
__device__ int sturm_count(const double *d, const double *e, int l, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0;
  for (int i = 1; i < l; ++i) {
    q = d[i] - x - e[i - 1] * e[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0;
  }
  return cnt;
}

// eigenvalue m (ascending) by bisection; also computes the 1-norm bound
__global__ void k_bisect(const double *__restrict__ d, const double *__restrict__ e, int l,
                         double *__restrict__ w) {
  grid_dep_enter();
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= l) return;
  double lo = 1e300, hi = -1e300, emax = 0.0;
  for (int i = 0; i < l; ++i) {
    double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < l ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    if (i + 1 < l) emax = fmax(emax, e[i] * e[i]);
  }
  const double tnorm = fmax(fabs(lo), fabs(hi));
  const double eps = 2.220446049250313e-16;
  const double pivmin = fmax(1e-300, 4.0 * 2.2250738585072014e-308 * fmax(1.0, emax));
  lo -= 2.0 * eps * tnorm + pivmin;
  hi += 2.0 * eps * tnorm + pivmin;
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin) break;
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(d, e, l, mid, pivmin) > m) hi = mid; else lo = mid;
  }
  w[m] = 0.5 * (lo + hi);
}

// Eigenvalue m (ascending) by multisection: one block of MSW warps per
// eigenvalue, its lanes evaluate Sturm counts at 64·MSW interior points of
// the current bracket (two interleaved recurrences per lane) and ballots pick
// the sub-interval holding the m-th eigenvalue (7 bits per round instead of
// 1); T's diagonal / off-diagonal squares live in shared memory.  The Sturm
// recurrences are fp64-issue bound: small blocks spread the l eigenvalues
// over every SM (one or two warps per SM sub-partition).
constexpr int MSW = 2;  // warps per block, all on one eigenvalue (64·MSW points per round)
__device__ __forceinline__ double pow2_of_exponent(double m) {  // 2^-e for m = f · 2^e, f in [1, 2)
  const int e = ((__double2hiint(m) >> 20) & 0x7ff) - 1023;
  const int be = min(max(1023 - e, 1), 2046);
  return __hiloint2double(be << 20, 0);
}

// Sturm count of the (power-of-2 scaled) tridiagonal T at two shifts, by the
// three-term recurrence p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2} of the
// leading principal minors (no division on the dependence chain; the pair is
// rescaled by a power of two every 8 steps).  Count = sign changes of p;
// an exact zero takes the sign opposite to its predecessor.
__device__ __forceinline__ void sturm2(const double *sd, const double *se2, int l, double xa, double xb, int &ca,
                                       int &cb) {
  double a0 = 1.0, a1 = sd[0] - xa, b0 = 1.0, b1 = sd[0] - xb;
  if (a1 == 0.0) a1 = -1e-300;
  if (b1 == 0.0) b1 = -1e-300;
  ca = a1 < 0.0;
  cb = b1 < 0.0;
  for (int i = 1; i < l; ++i) {
    double a2 = (sd[i] - xa) * a1 - se2[i - 1] * a0;
    double b2 = (sd[i] - xb) * b1 - se2[i - 1] * b0;
    if (a2 == 0.0) a2 = -1e-300 * a1;
    if (b2 == 0.0) b2 = -1e-300 * b1;
    ca += (a2 < 0.0) != (a1 < 0.0);
    cb += (b2 < 0.0) != (b1 < 0.0);
    a0 = a1; a1 = a2;
    b0 = b1; b1 = b2;
    if ((i & 7) == 0) {
      const double sa = pow2_of_exponent(fmax(fabs(a0), fabs(a1)));
      const double sb = pow2_of_exponent(fmax(fabs(b0), fabs(b1)));
      a0 *= sa; a1 *= sa;
      b0 *= sb; b1 *= sb;
    }
  }
}

__global__ void __launch_bounds__(MSW * 32) k_multisect(const double *__restrict__ d, const double *__restrict__ e,
                                                        int l, double *__restrict__ w) {
  grid_dep_enter();
  extern __shared__ double ms_sh[];
  double *sd = ms_sh, *se2 = ms_sh + l;
  const int lane = threadIdx.x & 31;
  // exact power-of-two scale of T to norm <= 1 (Gershgorin), all warps
  double tn = 0.0;
  for (int i = lane; i < l; i += 32) {
    const double r = fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < l ? fabs(e[i]) : 0.0);
    tn = fmax(tn, r);
  }
  for (int o = 16; o > 0; o >>= 1) tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
  const double inv = tn > 0.0 ? 0.5 * pow2_of_exponent(tn) : 1.0;  // 2^-(e+1): |T| / 2^(e+1) < 1
  for (int i = threadIdx.x; i < l; i += blockDim.x) {
    sd[i] = d[i] * inv;
    se2[i] = (i + 1 < l) ? (e[i] * inv) * (e[i] * inv) : 0.0;
  }
  __syncthreads();
  const int m = blockIdx.x, wi = threadIdx.x >> 5;
  __shared__ unsigned masks[2 * MSW];
  double lo = 1e300, hi = -1e300;
  for (int i = lane; i < l; i += 32) {
    const double r = (i > 0 ? fabs(e[i - 1]) * inv : 0.0) + (i + 1 < l ? fabs(e[i]) * inv : 0.0);
    lo = fmin(lo, sd[i] - r);
    hi = fmax(hi, sd[i] + r);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const double eps = 2.220446049250313e-16;
  lo -= 4.0 * eps + 1e-300;
  hi += 4.0 * eps + 1e-300;
  // 64·MSW points per round (two per lane; warp wi takes points 64 wi + 1 ..
  // 64 wi + 64).  Every
  // thread takes the same (block-uniform) decision from the shared ballots.
  constexpr int NP = 64 * MSW;
  // stop at 2 ulp relative or 4 eps absolute in the scaled T (||T|| in [1/2, 1)):
  // eigenvalues near 0 are only determined to ~eps ||T|| by the Householder
  // reduction anyway, and bisecting them to 1e-300 took up to 40 rounds
  for (int it = 0; it < 40; ++it) {
    if (hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi)) + 4.0 * eps) break;
    const double step = (hi - lo) / (double)(NP + 1);
    int ca, cb;
    sturm2(sd, se2, l, lo + step * (double)(64 * wi + lane + 1), lo + step * (double)(64 * wi + lane + 33), ca, cb);
    const unsigned above_a = __ballot_sync(0xffffffffu, ca > m), above_b = __ballot_sync(0xffffffffu, cb > m);
    if (lane == 0) {
      masks[2 * wi] = above_a;
      masks[2 * wi + 1] = above_b;
    }
    __syncthreads();
    int jf = NP;
#pragma unroll
    for (int q = 2 * MSW - 1; q >= 0; --q)
      if (masks[q]) jf = 32 * q + __ffs(masks[q]) - 1;
    __syncthreads();
    const double nlo = jf == 0 ? lo : lo + step * (double)jf;
    const double nhi = jf == NP ? hi : lo + step * (double)(jf + 1);
    if (!(nhi < hi || nlo > lo)) break;  // no progress at this precision
    lo = nlo;
    hi = nhi;
  }
  if (threadIdx.x == 0) w[m] = 0.5 * (lo + hi) / inv;
}

// Inverse iteration (dstein-style): one warp per cluster of (near-)degenerate
// eigenvalues, gap <= 1e-9 ||T|| (isolated eigenvalues converge to vectors whose
// mutual angle is ~eps ||T|| / gap).  The LU of T - sigma I (dgttrf with partial
// pivoting) lives in shared memory; the c right-hand sides of a cluster are
// solved in parallel, one lane each, then orthonormalised together (MGS).
constexpr int IVW = 4;  // warps per block

__global__ void __launch_bounds__(IVW * 32) k_invit(const double *__restrict__ d, const double *__restrict__ e,
                                                    int l, const double *__restrict__ w,
                                                    const int *__restrict__ cstart, const int *__restrict__ ncl_dev,
                                                    double *__restrict__ Zt, uint32_t seed) {
  grid_dep_enter();
  extern __shared__ double ivs[];
  const int wib = threadIdx.x / 32, ln = threadIdx.x % 32;
  const int gw = blockIdx.x * IVW + wib;
  if (gw >= *ncl_dev) return;  // launched for the worst case (every eigenvalue isolated)
  double *dl = ivs + (int64_t)wib * 4 * l;
  double *dg = dl + l, *du = dg + l, *du2 = du + l;
  int8_t *piv = reinterpret_cast<int8_t *>(ivs + (int64_t)IVW * 4 * l) + wib * l;
  double tnorm = 0.0;
  for (int i = ln; i < l; i += 32) {
    double r = fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < l ? fabs(e[i]) : 0.0);
    tnorm = fmax(tnorm, r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tnorm = fmax(tnorm, __shfl_xor_sync(0xffffffffu, tnorm, o));
  const double eps = 2.220446049250313e-16;
  const double tiny = eps * fmax(tnorm, 1e-300);
  const int m0 = cstart[gw], m1 = cstart[gw + 1];
  double sigma = 0.0;
  for (int m = m0; m < m1; ++m) sigma += w[m];
  sigma /= (m1 - m0);
  // T - sigma I loaded by the whole warp (one serial lane would wait on every
  // global load in turn), then factored by lane 0
  for (int i = ln; i < l; i += 32) {
    dg[i] = d[i] - sigma;
    if (i + 1 < l) { dl[i] = e[i]; du[i] = e[i]; }
    du2[i] = 0.0;
    piv[i] = 0;
  }
  __syncwarp();
  if (ln == 0) {
    // dgttrf with the running pivot row (g = dg[i], u = du[i] as updated so
    // far) carried in registers: the dependence chain stays out of shared memory
    double g = dg[0], u = l > 1 ? du[0] : 0.0;
    for (int i = 0; i + 1 < l; ++i) {
      const double lo = dl[i], gn = dg[i + 1], un = i + 2 < l ? du[i + 1] : 0.0;
      if (fabs(g) >= fabs(lo)) {
        double gnew = gn;
        if (g != 0.0) {
          const double f = lo / g;
          dl[i] = f;
          gnew = gn - f * u;
        }
        dg[i] = g;
        du[i] = u;
        g = gnew;
        u = un;
      } else {
        const double f = g / lo;
        dg[i] = lo;
        dl[i] = f;
        du[i] = gn;
        g = u - f * gn;
        if (i + 2 < l) du2[i] = un;
        u = -f * un;
        piv[i] = 1;
      }
    }
    dg[l - 1] = g;
  }
  __syncwarp();
  for (int i = ln; i < l; i += 32) {
    double gi = dg[i];
    if (fabs(gi) < tiny) gi = gi < 0 ? -tiny : tiny;
    dg[i] = 1.0 / gi;  // the solves multiply by the reciprocal pivots
  }
  __syncwarp();
  if (m1 - m0 == 1) {
    // isolated eigenvalue (the common case): the vector lives in shared
    // memory (after the LU factors), lane 0 runs the substitutions
    int8_t *piv_end = reinterpret_cast<int8_t *>(ivs + (int64_t)IVW * 4 * l) + ((IVW * l + 7) & ~7);
    double *x = reinterpret_cast<double *>(piv_end) + (int64_t)wib * l;
    for (int i = ln; i < l; i += 32) {
      U4 r = philox4x32_10(U4{(uint32_t)i, (uint32_t)m0, 0x494E5649u, 0u}, seed, 0x5EEDu);
      x[i] = ((double)r.x + 0.5) * 2.3283064365386963e-10 - 0.5;
    }
    __syncwarp();
    for (int it = 0; it < 3; ++it) {
      if (ln == 0) {
        // the substitutions carry the running entries in registers, so the
        // dependence chain is one FMA per step (no shared-memory round trip)
        double cur = x[0];
        for (int i = 0; i + 1 < l; ++i) {
          const double nxt = x[i + 1];
          if (!piv[i]) {
            x[i] = cur;
            cur = nxt - dl[i] * cur;
          } else {
            x[i] = nxt;
            cur = cur - dl[i] * nxt;
          }
        }
        double x1 = cur * dg[l - 1], x2 = 0.0;  // x[i+1], x[i+2]
        x[l - 1] = x1;
        for (int i = l - 2; i >= 0; --i) {
          const double xi = (x[i] - du[i] * x1 - (i + 2 < l ? du2[i] * x2 : 0.0)) * dg[i];
          x[i] = xi;
          x2 = x1;
          x1 = xi;
        }
      }
      __syncwarp();
      double nrm = 0.0;
      for (int i = ln; i < l; i += 32) nrm += x[i] * x[i];
      nrm = sqrt(warp_sum(nrm));
      const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      for (int i = ln; i < l; i += 32) x[i] *= inv;
      __syncwarp();
    }
    for (int i = ln; i < l; i += 32) Zt[(int64_t)m0 * l + i] = x[i];
    return;
  }
  // deterministic random starts in the output rows
  for (int m = m0; m < m1; ++m)
    for (int i = ln; i < l; i += 32) {
      U4 r = philox4x32_10(U4{(uint32_t)i, (uint32_t)m, 0x494E5649u, 0u}, seed, 0x5EEDu);
      Zt[(int64_t)m * l + i] = ((double)r.x + 0.5) * 2.3283064365386963e-10 - 0.5;
    }
  __syncwarp();
  for (int it = 0; it < 3; ++it) {
    // solve (T - sigma I) x = x for every vector of the cluster, one lane each
    for (int m = m0 + ln; m < m1; m += 32) {
      double *x = Zt + (int64_t)m * l;
      for (int i = 0; i + 1 < l; ++i) {
        if (!piv[i]) {
          x[i + 1] -= dl[i] * x[i];
        } else {
          double t = x[i];
          x[i] = x[i + 1];
          x[i + 1] = t - dl[i] * x[i];
        }
      }
      x[l - 1] *= dg[l - 1];
      if (l > 1) x[l - 2] = (x[l - 2] - du[l - 2] * x[l - 1]) * dg[l - 2];
      for (int i = l - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) * dg[i];
    }
    __syncwarp();
    // modified Gram-Schmidt over the cluster
    for (int m = m0; m < m1; ++m) {
      double *x = Zt + (int64_t)m * l;
      for (int q = m0; q < m; ++q) {
        const double *zq = Zt + (int64_t)q * l;
        double s = 0.0;
        for (int i = ln; i < l; i += 32) s += zq[i] * x[i];
        s = warp_sum(s);
        for (int i = ln; i < l; i += 32) x[i] -= s * zq[i];
        __syncwarp();
      }
      double nrm = 0.0;
      for (int i = ln; i < l; i += 32) nrm += x[i] * x[i];
      nrm = sqrt(warp_sum(nrm));
      const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      for (int i = ln; i < l; i += 32) x[i] *= inv;
      __syncwarp();
    }
  }
}

// cluster starts: consecutive eigenvalues closer than ortol = 1e-9 ||T||
__global__ void k_clusters(const double *__restrict__ w, const double *__restrict__ d,
                           const double *__restrict__ e, int l, int *__restrict__ cstart, int *ncl) {
  grid_dep_enter();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double tnorm = 0.0;
  for (int i = 0; i < l; ++i)
    tnorm = fmax(tnorm, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < l ? fabs(e[i]) : 0.0));
  const double ortol = 1e-9 * tnorm;
  int c = 0;
  cstart[c++] = 0;
  for (int m = 1; m < l; ++m)
    if (w[m] - w[m - 1] > ortol) cstart[c++] = m;
  cstart[c] = l;
  *ncl = c;
}

// eigenvectors of S: x <- H_0 (H_1 (… H_{l-3} z)); one warp per eigenvector,
// held in registers (lane owns entries ln + 32 i); the reflectors two steps
// ahead are in flight while the current one is applied (Hv rows are zero at
// k <= j, so no masking below the reflector's support)
constexpr int BT_NR = 15;  // l <= 480
constexpr int BT_T = 64;  // 2 warps per block: the l eigenvectors spread over every SM
__global__ void __launch_bounds__(BT_T) k_backtransform(const double *__restrict__ Hv, const double *__restrict__ hbeta,
                                                       int l, double *__restrict__ Zt) {
  grid_dep_enter();
  const int m = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int ln = threadIdx.x % 32;
  if (m >= l) return;
  double *xg = Zt + (int64_t)m * l;
  double x[BT_NR];
#pragma unroll
  for (int i = 0; i < BT_NR; ++i) {
    const int k = ln + 32 * i;
    x[i] = k < l ? xg[k] : 0.0;
  }
  auto load = [&](double *dst, int j) {
    const double *v = Hv + (int64_t)j * l;
#pragma unroll
    for (int i = 0; i < BT_NR; ++i) {
      const int k = ln + 32 * i;
      dst[i] = k < l ? __ldg(v + k) : 0.0;
    }
  };
  auto apply = [&](const double *v, double b) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;  // three short chains instead of one of BT_NR
#pragma unroll
    for (int i = 0; i < BT_NR; i += 3) {
      s0 = fma(v[i], x[i], s0);
      if (i + 1 < BT_NR) s1 = fma(v[i + 1], x[i + 1], s1);
      if (i + 2 < BT_NR) s2 = fma(v[i + 2], x[i + 2], s2);
    }
    const double sacc = warp_sum((s0 + s1) + s2) * b;
#pragma unroll
    for (int i = 0; i < BT_NR; ++i) x[i] = fma(-sacc, v[i], x[i]);
  };
  // reflectors j = l-3 .. 0, two in flight: the loads of reflector j-2 are
  // issued before reflector j is applied (one step of prefetch left each
  // step waiting on an L2 round trip)
  double va[BT_NR], vb[BT_NR], v[BT_NR];
  double ba = 0.0, bb = 0.0;
  if (l >= 3) {
    load(va, l - 3);
    ba = __ldg(hbeta + l - 3);
  }
  if (l >= 4) {
    load(vb, l - 4);
    bb = __ldg(hbeta + l - 4);
  }
  for (int j = l - 3; j >= 0; j -= 2) {
#pragma unroll
    for (int i = 0; i < BT_NR; ++i) v[i] = va[i];
    double b = ba;
    if (j >= 2) {
      load(va, j - 2);
      ba = __ldg(hbeta + j - 2);
    }
    apply(v, b);
    if (j == 0) break;
#pragma unroll
    for (int i = 0; i < BT_NR; ++i) v[i] = vb[i];
    b = bb;
    if (j >= 3) {
      load(vb, j - 3);
      bb = __ldg(hbeta + j - 3);
    }
    apply(v, b);
  }
#pragma unroll
  for (int i = 0; i < BT_NR; ++i) {
    const int k = ln + 32 * i;
    if (k < l) xg[k] = x[i];
  }
}

// order by desc |λ| (ties: desc λ) or desc λ; V[r][c] = Zt[perm[c]][r]
__global__ void k_eig_sort(const double *__restrict__ w, const double *__restrict__ Zt, int l,
                           bool abs_order, double *__restrict__ lam, double *__restrict__ V) {
  grid_dep_enter();
  const int i = blockIdx.x;  // one block per eigenpair
  const double wi = w[i];
  __shared__ int rank_s;
  if (threadIdx.x == 0) rank_s = 0;
  __syncthreads();
  int cnt = 0;
  for (int j = threadIdx.x; j < l; j += blockDim.x) {
    const double wj = w[j];
    bool before;
    if (abs_order) {
      const double ai = fabs(wi), aj = fabs(wj);
      before = (aj > ai) || (aj == ai && (wj > wi || (wj == wi && j < i)));
    } else {
      before = (wj > wi) || (wj == wi && j < i);
    }
    cnt += before;
  }
  atomicAdd(&rank_s, cnt);
  __syncthreads();
  const int r = rank_s;
  if (threadIdx.x == 0) lam[r] = wi;
  for (int k = threadIdx.x; k < l; k += blockDim.x) V[(int64_t)k * l + r] = Zt[(int64_t)i * l + k];
}

void sym_eig(Ctx &c, double *S, int64_t l64, double *lam, double *V, bool abs_order) {
  const int l = (int)l64;
  NM_REQUIRE(l >= 1, "sym_eig: l >= 1");
  cudaStream_t s = c.stream;
  DBuf<double> d(l, s), e(l, s), Hv((size_t)l * l, s), hb(l, s), w(l, s), Zt((size_t)l * l, s);
  NM_CUDA(cudaMemsetAsync(Hv.p, 0, (size_t)l * l * 8, s));
  NM_CUDA(cudaMemsetAsync(hb.p, 0, (size_t)l * 8, s));
  NM_CUDA(cudaMemsetAsync(e.p, 0, (size_t)l * 8, s));
  const int nloc = (l + TDC - 1) / TDC;
  size_t smem = ((size_t)nloc * l + 4 * l + 40 + 32 * TDC + 8) * sizeof(double);
  NM_REQUIRE(smem <= 227 * 1024 && l <= 32 * BT_NR, "sym_eig: l too large for the 8-CTA cluster (l <= ~470)");
  smem_attr(k_tridiag, 227 * 1024);
  if (TDC > 8) func_attr(reinterpret_cast<const void *>(k_tridiag), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  NM_LAUNCH(c, "tridiag", launch_pdl(s, k_tridiag, TDC, TDT, smem, S, l, d, e, Hv, hb));
  NM_LAUNCH(c, "multisect", launch_pdl(s, k_multisect, l, MSW * 32, (size_t)2 * l * sizeof(double), d, e, l, w));
  DBuf<int> cst(l + 1, s), ncl(1, s);
  NM_LAUNCH(c, "clusters", launch_pdl(s, k_clusters, 1, 32, 0, w, d, e, l, cst, ncl));
  const size_t ivsm = (size_t)IVW * 4 * l * sizeof(double) + (size_t)IVW * l + 16 + (size_t)IVW * l * sizeof(double);
  smem_attr(k_invit, 200 * 1024);
  NM_LAUNCH(c, "invit", launch_pdl(s, k_invit, ceil_div(l, IVW), IVW * 32, ivsm, d, e, l, w, cst, ncl, Zt, 0x1234567u));
  NM_LAUNCH(c, "backtransform", launch_pdl(s, k_backtransform, ceil_div((int64_t)l * 32, BT_T), BT_T, 0, Hv, hb, l, Zt));
  NM_LAUNCH(c, "eig_sort", launch_pdl(s, k_eig_sort, l, 128, 0, w, Zt, l, abs_order, lam, V));
}

}  // namespace netmfp
