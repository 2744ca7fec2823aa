// dense.cu — tall-skinny dense kernels on n×c fp32 blocks:
//   gram:       G = Aᵀ W B (fp64 result) — CholeskyQR Gram, Rayleigh–Ritz
//               S = Pᵀ(AP), Eq. 3's K = Uᵀ D^(-1+2α) U
//   gemm_tall:  C = diag(rs) · A · Bs — Q = Y R⁻¹, U = Q Û, F·C, E = Q Û √Σ
//   gaussian_block: Ω = randn (Alg. 2 step 2, Philox [R1])
// Blocks of >= 128 rows run the tcgen05 kernels of tc_gemm.cu; the CUDA-core
// kernels here serve only blocks shorter than one tensor-core M tile.
#include "common.cuh"
#include "kernels.cuh"

#include <cstdlib>

namespace netmfp {

__device__ __forceinline__ float dpow_scale(const int32_t *deg, int64_t i, float e) {
  if (!deg) return 1.f;
  int d = deg[i];
  if (d <= 0) return 0.f;
  if (e == 0.f) return 1.f;
  if (e == 0.5f) return rsqrtf((float)d);
  if (e == 1.f) return 1.f / (float)d;
  return powf((float)d, -e);
}

// ---------------------------------------------------------------------------
// Gram: per-slab fp32 partial tiles → fp64 reduction over slabs (deterministic)
// ---------------------------------------------------------------------------
constexpr int GT = 64;   // output tile
constexpr int GK = 32;   // rows per smem stage

__global__ void __launch_bounds__(256) k_gram_partial(Mat A, Mat B, const int32_t *__restrict__ deg,
                                                      float wexp, int64_t slab_rows, bool sym,
                                                      float *__restrict__ part, int64_t a_pad,
                                                      int64_t b_pad) {
  grid_dep_enter();
  const int tb = blockIdx.x, ta = blockIdx.y, slab = blockIdx.z;
  if (sym && ta > tb) return;
  __shared__ __align__(16) float As[GK][GT];
  __shared__ __align__(16) float Bs[GK][GT];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t r0 = (int64_t)slab * slab_rows;
  const int64_t r1 = min(r0 + slab_rows, A.rows);
  const int a0 = ta * GT, b0 = tb * GT;
  float acc[4][4] = {};
  for (int64_t rr = r0; rr < r1; rr += GK) {
    // load GK rows × 64 cols of A (weighted) and B: 512 float4 each, 2 per thread
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      int idx = threadIdx.x + it * 256;
      int r = idx / 16, c4 = (idx % 16) * 4;
      int64_t row = rr + r;
      float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
      if (row < r1) {
        if (a0 + c4 < A.cols) va = *reinterpret_cast<const float4 *>(A.p + row * A.ld + a0 + c4);
        if (b0 + c4 < B.cols) vb = *reinterpret_cast<const float4 *>(B.p + row * B.ld + b0 + c4);
        float w = dpow_scale(deg, row, wexp);
        va.x *= w; va.y *= w; va.z *= w; va.w *= w;
      }
      // mask columns beyond cols (ld padding may hold data of a wider view)
      if (a0 + c4 + 4 > A.cols) {
        int nv = (int)(A.cols - (a0 + c4));
        if (nv < 4) va.w = 0.f;
        if (nv < 3) va.z = 0.f;
        if (nv < 2) va.y = 0.f;
        if (nv < 1) va.x = 0.f;
      }
      if (b0 + c4 + 4 > B.cols) {
        int nv = (int)(B.cols - (b0 + c4));
        if (nv < 4) vb.w = 0.f;
        if (nv < 3) vb.z = 0.f;
        if (nv < 2) vb.y = 0.f;
        if (nv < 1) vb.x = 0.f;
      }
      *reinterpret_cast<float4 *>(&As[r][c4]) = va;
      *reinterpret_cast<float4 *>(&Bs[r][c4]) = vb;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GK; ++kk) {
      float4 a = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
      float4 b = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
      float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float *dst = part + (size_t)slab * a_pad * b_pad;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t r = a0 + ty * 4 + i;
    *reinterpret_cast<float4 *>(dst + r * b_pad + b0 + tx * 4) =
        make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
  }
}

__global__ void k_gram_reduce(const float *__restrict__ part, int nslab, int64_t a, int64_t b,
                              int64_t a_pad, int64_t b_pad, bool sym, double *__restrict__ G,
                              int64_t ldg) {
  grid_dep_enter();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= a * b) return;
  int64_t i = idx / b, j = idx % b;
  int64_t si = i, sj = j;
  if (sym && (i / GT) > (j / GT)) { si = j; sj = i; }  // lower tile: mirror
  double s = 0.0;
  for (int t = 0; t < nslab; ++t) s += (double)part[(size_t)t * a_pad * b_pad + si * b_pad + sj];
  G[i * ldg + j] = s;
}

// Blocks of >= 128 rows (one tensor-core M tile) take the tcgen05 kernels of
// tc_gemm.cu, whatever their width; only blocks with fewer rows than one M
// tile (tiny graphs) use the CUDA-core kernels below.  There is no switch.
constexpr int64_t kTcMinRows = 128;

void gram(Ctx &c, const Mat &A, const Mat &B, const int32_t *deg, float wexp, double *G, int64_t ldg, bool exact,
          bool sym_result) {
  NM_REQUIRE(A.rows == B.rows, "gram: row mismatch");
  if (A.rows >= kTcMinRows) {
    tc_gram(c, A, B, deg, wexp, G, ldg, exact, sym_result && A.cols == B.cols);
    return;
  }
  const int64_t n = A.rows;
  if (n == 0 || A.cols == 0 || B.cols == 0) {
    if (A.cols > 0 && B.cols > 0) NM_CUDA(cudaMemset2DAsync(G, ldg * 8, 0, B.cols * 8, A.cols, c.stream));
    return;
  }
  const bool sym = (A.p == B.p && A.cols == B.cols && A.ld == B.ld);
  const int ta = (int)ceil_div(A.cols, GT), tb = (int)ceil_div(B.cols, GT);
  const int tiles = sym ? ta * (ta + 1) / 2 : ta * tb;
  int nslab = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 512),
                                                           ceil_div((int64_t)c.num_sms * 6, tiles)));
  int64_t slab_rows = (int64_t)ceil_div(n, nslab);
  slab_rows = (slab_rows + GK - 1) / GK * GK;
  nslab = (int)ceil_div(n, slab_rows);
  const int64_t a_pad = (int64_t)ta * GT, b_pad = (int64_t)tb * GT;
  DBuf<float> part((size_t)nslab * a_pad * b_pad, c.stream);
  dim3 grid(tb, ta, nslab);
  NM_LAUNCH(c, "gram_partial", launch_pdl(c.stream, k_gram_partial, grid, 256, 0, A, B, deg, wexp, slab_rows, sym, part, a_pad, b_pad));
  NM_LAUNCH(c, "gram_reduce", launch_pdl(c.stream, k_gram_reduce, ceil_div(A.cols * B.cols, 256), 256, 0, part, nslab, A.cols, B.cols,
                                                                      a_pad, b_pad, sym, G, ldg));
}

// ---------------------------------------------------------------------------
// C = rs · A · Bs   (A n×a fp32, Bs a×b fp64 small, C n×b fp32)
// ---------------------------------------------------------------------------
constexpr int TM = 128, TN = 64, TK = 32;

__global__ void __launch_bounds__(256) k_gemm_tall(Mat A, const double *__restrict__ Bs, int64_t ldb,
                                                   int64_t bcols, const int32_t *__restrict__ deg,
                                                   float rexp, Mat C) {
  grid_dep_enter();
  __shared__ __align__(16) float As[TK][TM + 4];
  __shared__ __align__(16) float Bsh[TK][TN];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.x * TM;
  const int n0 = blockIdx.y * TN;
  const int64_t K = A.cols;
  float acc[8][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += TK) {
    // A tile: 128 rows × 32 k -> As[k][m]
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      int idx = threadIdx.x + it * 256;
      int m = idx / 8, k4 = (idx % 8) * 4;
      int64_t row = m0 + m;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < A.rows && k0 + k4 < K) {
        v = *reinterpret_cast<const float4 *>(A.p + row * A.ld + k0 + k4);
        int64_t nv = K - (k0 + k4);
        if (nv < 4) v.w = 0.f;
        if (nv < 3) v.z = 0.f;
        if (nv < 2) v.y = 0.f;
      }
      As[k4 + 0][m] = v.x;
      As[k4 + 1][m] = v.y;
      As[k4 + 2][m] = v.z;
      As[k4 + 3][m] = v.w;
    }
    // B tile: 32 × 64 from fp64
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int idx = threadIdx.x + it * 256;
      int k = idx / TN, nn = idx % TN;
      double v = 0.0;
      if (k0 + k < K && n0 + nn < bcols) v = Bs[(k0 + k) * ldb + n0 + nn];
      Bsh[k][nn] = (float)v;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < TK; ++kk) {
      float4 a0 = *reinterpret_cast<const float4 *>(&As[kk][ty * 8]);
      float4 a1 = *reinterpret_cast<const float4 *>(&As[kk][ty * 8 + 4]);
      float4 b = *reinterpret_cast<const float4 *>(&Bsh[kk][tx * 4]);
      float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int cbase = n0 + tx * 4;
  if (cbase >= C.cols) return;
  const int nv = (int)(C.cols - cbase < 4 ? C.cols - cbase : 4);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int64_t row = m0 + ty * 8 + i;
    if (row >= C.rows) break;
    float s = dpow_scale(deg, row, rexp);
    float *dst = C.p + row * C.ld + cbase;
    if (nv == 4) {
      *reinterpret_cast<float4 *>(dst) = make_float4(s * acc[i][0], s * acc[i][1], s * acc[i][2], s * acc[i][3]);
    } else {
      for (int j = 0; j < nv; ++j) dst[j] = s * acc[i][j];
    }
  }
}

void gemm_tall(Ctx &c, const Mat &A, const double *Bs, int64_t ldb, int64_t bcols, const int32_t *deg,
               float rexp, const Mat &C) {
  NM_REQUIRE(A.rows == C.rows && C.cols == bcols, "gemm_tall: shape mismatch");
  NM_REQUIRE(C.p != A.p, "gemm_tall: in-place not supported");
  if (A.rows >= kTcMinRows) {
    tc_gemm_tall(c, A, Bs, ldb, bcols, deg, rexp, C);
    return;
  }
  if (A.rows == 0) return;
  dim3 grid(ceil_div(A.rows, TM), ceil_div(bcols, TN));
  NM_LAUNCH(c, "gemm_tall", launch_pdl(c.stream, k_gemm_tall, grid, 256, 0, A, Bs, ldb, bcols, deg, rexp, C));
}

void gemm_tall_tri(Ctx &c, const Mat &A, const double *Rinv, int64_t ldb, const int32_t *deg, float rexp,
                   const Mat &C, bool exact) {
  if (A.rows >= kTcMinRows) {
    tc_gemm_tall_tri(c, A, Rinv, ldb, A.cols, deg, rexp, C, exact);
    return;
  }
  gemm_tall(c, A, Rinv, ldb, A.cols, deg, rexp, C);
}

// ---------------------------------------------------------------------------
// Ω = randn(n, l) (Alg. 2 step 2) with Philox4x32-10 [R1], optional row scale
// ---------------------------------------------------------------------------
// A warp per row (grid-stride over rows), lane t over entries 4q..4q+3 for
// q = t, t + 32, ...: one Philox call per 4 entries (Box–Muller with both
// outputs of each word pair, R1) and one 16-B store; the row's id
// and scale d^-e are computed once per row, not per element.
__global__ void __launch_bounds__(256) k_gaussian(Mat O, uint32_t k0, uint32_t k1, const int32_t *__restrict__ deg,
                                                  float rexp, int64_t row0, const int32_t *__restrict__ ids) {
  grid_dep_enter();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool vec = (O.ld % 4) == 0 && ((uintptr_t)O.p & 15) == 0;
  const int64_t nq = (O.cols + 3) / 4;
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < O.rows; i += nw) {
    // global row: every rank (or compacted graph) draws its own rows of the same Ω
    const int64_t gi = ids ? (int64_t)ids[i] : i + row0;
    const float sc = dpow_scale(deg, i, rexp);
    float *orow = O.p + i * O.ld;
    // two counters per iteration: independent Philox chains interleave (ILP)
    for (int64_t q0 = lane; q0 < nq; q0 += 64) {
      U4 w[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t q = q0 + 32 * u;
        w[u] = philox4x32_10(U4{(uint32_t)q, (uint32_t)(gi & 0xFFFFFFFF), (uint32_t)((uint64_t)gi >> 32), kTagOmega},
                             k0, k1);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t q = q0 + 32 * u;
        if (q >= nq) break;
        // Box–Muller in fp32 (the block is fp32; |error| ~1e-7 relative to the fp64 oracle)
        const float u0 = ((float)w[u].x + 0.5f) * 2.3283064365386963e-10f;  // 2^-32
        const float u1 = ((float)w[u].y + 0.5f) * 2.3283064365386963e-10f;
        const float u2 = ((float)w[u].z + 0.5f) * 2.3283064365386963e-10f;
        const float u3 = ((float)w[u].w + 0.5f) * 2.3283064365386963e-10f;
        // MUFU log2 / sin / cos (abs. error ~1e-6 on a N(0,1) draw; the oracle
        // draws in fp64): (cos, sin)(2π u) = -(cos, sin)(2π (u - 1/2)), argument in [-π, π)
        const float r0 = -sqrtf(-1.3862943611198906f * __log2f(u0)) * sc;
        const float r2 = -sqrtf(-1.3862943611198906f * __log2f(u2)) * sc;
        float s1, c1, s3, c3;
        __sincosf(6.283185307179586f * (u1 - 0.5f), &s1, &c1);
        __sincosf(6.283185307179586f * (u3 - 0.5f), &s3, &c3);
        const float4 g = make_float4(r0 * c1, r0 * s1, r2 * c3, r2 * s3);
        const int64_t j = 4 * q;
        if (vec && j + 3 < O.cols) {
          *reinterpret_cast<float4 *>(orow + j) = g;
        } else {
          orow[j] = g.x;
          if (j + 1 < O.cols) orow[j + 1] = g.y;
          if (j + 2 < O.cols) orow[j + 2] = g.z;
          if (j + 3 < O.cols) orow[j + 3] = g.w;
        }
      }
    }
  }
}

void gaussian_block(Ctx &c, const Mat &O, uint64_t seed, const int32_t *deg, float rexp, int64_t row0,
                    const int32_t *ids) {
  if (O.rows * O.cols == 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(O.rows, 8), (int64_t)c.num_sms * 16);
  NM_LAUNCH(c, "gaussian", launch_pdl(c.stream, k_gaussian, blocks, 256, 0, O, (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32), deg, rexp, row0, ids));
}

__global__ void k_row_scale(Mat Y, const int32_t *__restrict__ deg, float rexp) {
  grid_dep_enter();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= Y.rows * Y.cols) return;
  int64_t i = idx / Y.cols, j = idx % Y.cols;
  Y.p[i * Y.ld + j] *= dpow_scale(deg, i, rexp);
}

// Dst[i, :] = d_i^-e · Src[i, :]  (float4; lds, ldd, cols multiples of 4 or tail handled)
__global__ void k_scale_copy(Mat Src, Mat Dst, const int32_t *__restrict__ deg, float rexp) {
  grid_dep_enter();
  const int64_t c4 = (Src.cols + 3) / 4;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= Src.rows * c4) return;
  const int64_t i = idx / c4, j = (idx % c4) * 4;
  const float sc = dpow_scale(deg, i, rexp);
  const float *src = Src.p + i * Src.ld + j;
  float *dst = Dst.p + i * Dst.ld + j;
  if (j + 4 <= Src.cols) {
    const float4 v = *reinterpret_cast<const float4 *>(src);
    *reinterpret_cast<float4 *>(dst) = make_float4(sc * v.x, sc * v.y, sc * v.z, sc * v.w);
  } else {
    for (int64_t t = j; t < Src.cols; ++t) dst[t - j] = sc * src[t - j];
  }
}

void scale_copy_block(Ctx &c, const Mat &Src, const Mat &Dst, const int32_t *deg, float rexp) {
  NM_REQUIRE(Src.ld % 4 == 0 && Dst.ld % 4 == 0, "scale_copy: ld % 4 == 0");
  const int64_t tot = Src.rows * ((Src.cols + 3) / 4);
  NM_LAUNCH(c, "scale_copy", launch_pdl(c.stream, k_scale_copy, ceil_div(tot, 256), 256, 0, Src, Dst, deg, rexp));
}

void row_scale_block(Ctx &c, const Mat &Y, const int32_t *deg, float rexp) {
  NM_LAUNCH(c, "row_scale", launch_pdl(c.stream, k_row_scale, ceil_div(Y.rows * Y.cols, 256), 256, 0, Y, deg, rexp));
}

void copy_block(Ctx &c, const float *src, int64_t lds, float *dst, int64_t ldd, int64_t rows,
                int64_t cols) {
  NM_CUDA(cudaMemcpy2DAsync(dst, ldd * 4, src, lds * 4, cols * 4, rows, cudaMemcpyDefault, c.stream));
}

// Dst[i, :] = Src[comp[i] - sub, :], or 0 where comp[i] < 0 (compacted rows
// back to all rows; every element of Dst written once).  A warp per row.
__global__ void __launch_bounds__(256) k_scatter_rows(Mat Src, const int32_t *__restrict__ comp, Mat Dst, bool vec4,
                                                      int64_t sub) {
  grid_dep_enter();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < Dst.rows; i += nw) {
    const int64_t r = comp[i] < 0 ? -1 : comp[i] - sub;
    float *d = Dst.p + i * Dst.ld;
    const float *src = Src.p + (int64_t)(r < 0 ? 0 : r) * Src.ld;
    if (vec4) {
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t j = 4 * lane; j < Dst.cols; j += 128)
        *reinterpret_cast<float4 *>(d + j) = r >= 0 ? *reinterpret_cast<const float4 *>(src + j) : z;
    } else {
      for (int64_t j = lane; j < Dst.cols; j += 32) d[j] = r >= 0 ? src[j] : 0.f;
    }
  }
}

void scatter_rows(Ctx &c, const Mat &Src, const int32_t *comp, const Mat &Dst, int64_t sub) {
  if (Dst.rows * Dst.cols == 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(Dst.rows, 8), (int64_t)c.num_sms * 16);
  const bool vec4 = Dst.cols % 4 == 0 && Dst.ld % 4 == 0 && Src.ld % 4 == 0 && ((uintptr_t)Dst.p & 15) == 0 &&
                    ((uintptr_t)Src.p & 15) == 0;
  NM_LAUNCH(c, "scatter_rows", launch_pdl(c.stream, k_scatter_rows, blocks, 256, 0, Src, comp, Dst, vec4, sub));
}

// Dst[ids[j], :] = Src[j, :] for every row j of Src (the other rows of Dst
// untouched); Dst may be mapped host memory.  A warp per row.
__global__ void __launch_bounds__(256) k_write_rows(Mat Src, const int32_t *__restrict__ ids, Mat Dst, bool vec4) {
  grid_dep_enter();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); j < Src.rows; j += nw) {
    float *d = Dst.p + (int64_t)ids[j] * Dst.ld;
    const float *src = Src.p + j * Src.ld;
    if (vec4) {
      for (int64_t c = 4 * lane; c < Src.cols; c += 128)
        *reinterpret_cast<float4 *>(d + c) = *reinterpret_cast<const float4 *>(src + c);
    } else {
      for (int64_t c = lane; c < Src.cols; c += 32) d[c] = src[c];
    }
  }
}

void write_rows(Ctx &c, const Mat &Src, const int32_t *ids, const Mat &Dst) {
  if (Src.rows * Src.cols == 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(Src.rows, 8), (int64_t)c.num_sms * 16);
  const bool vec4 = Src.cols % 4 == 0 && Dst.ld % 4 == 0 && Src.ld % 4 == 0 && ((uintptr_t)Dst.p & 15) == 0 &&
                    ((uintptr_t)Src.p & 15) == 0;
  NM_LAUNCH(c, "write_rows", launch_pdl(c.stream, k_write_rows, blocks, 256, 0, Src, ids, Dst, vec4));
}

}  // namespace netmfp
