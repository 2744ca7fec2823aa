// sketch.cu — rows a5-a7: sparse-sign matrices (Alg. 3) and the sketches of
// Alg. 4 without materialising M̂' (Eq. 5):
//   Y = f(scale · A B(p,:)ᵀ) Ψ(p,:)   computed tile by tile: a GEMM tile of
//   G = A B(p,:)ᵀ stays in registers, f = trunc_log/log1p is applied in the
//   epilogue and each entry is scattered with its sign into a shared-memory Y
//   tile (the "signed gather" of §4.4, "for each column of Ψ ... z nonzeros");
//   Y rows are written once.  Wide sketches (Π, d+s3 columns) go through an
//   explicit f(G) block and a row scatter.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace netmfp {

// ---------------------------------------------------------------------------
// Alg. 3: column j draws z distinct rows by sequential rejection from the
// Philox stream (j, r, 0, tag); sign = +1 if w1 even [R1]
// ---------------------------------------------------------------------------
constexpr int kMaxZ = 64;

__global__ void k_ss_gen(int64_t n, int64_t h, int z, uint32_t k0, uint32_t k1, uint32_t tag,
                         int32_t *__restrict__ rows, float *__restrict__ signs,
                         int32_t *__restrict__ keys, int32_t *__restrict__ vals) {
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
    float sg = (w.y & 1u) ? -1.f : 1.f;
    rows[j * z + cnt] = row;
    signs[j * z + cnt] = sg;
    keys[j * z + cnt] = row;
    vals[j * z + cnt] = (int32_t)(j * 2 + (sg < 0.f ? 1 : 0));
    ++cnt;
  }
}

__global__ void k_ss_unpack(const int32_t *__restrict__ vals, int64_t cnt, int32_t *__restrict__ pcol,
                            float *__restrict__ psign) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  int32_t v = vals[i];
  pcol[i] = v >> 1;
  psign[i] = (v & 1) ? -1.f : 1.f;
}

void gen_sparse_sign(Ctx &c, int64_t n, int64_t h, int64_t z, uint64_t seed, uint32_t tag, SparseSign &S) {
  NM_REQUIRE(z >= 2 && z <= n && z <= kMaxZ, "sparse-sign: need 2 <= z <= min(n, 64)");
  NM_REQUIRE(h >= 1, "sparse-sign: h >= 1");
  cudaStream_t s = c.stream;
  const int64_t cnt = h * z;
  S.n = n; S.h = h; S.z = z;
  S.rows.alloc(cnt, s);
  S.signs.alloc(cnt, s);
  DBuf<int32_t> keys(cnt, s), vals(cnt, s), keys2(cnt, s), vals2(cnt, s);
  NM_LAUNCH(c, "ss_gen", k_ss_gen<<<ceil_div(h, 128), 128, 0, s>>>(n, h, (int)z, (uint32_t)(seed & 0xFFFFFFFFu),
                                            (uint32_t)(seed >> 32), tag, S.rows, S.signs, keys, vals));
  size_t tb = 0;
  NM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys2.p, vals.p, vals2.p, cnt, 0, 32, s));
  DBuf<char> tmp(tb, s);
  NM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys2.p, vals.p, vals2.p, cnt, 0, 32, s));
  c.launches += 4;
  // run-length encode sorted rows -> unique p and counts
  DBuf<int32_t> uniq(cnt, s), counts(cnt, s), nruns(1, s);
  size_t tb2 = 0;
  NM_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb2, keys2.p, uniq.p, counts.p, nruns.p, cnt, s));
  DBuf<char> tmp2(tb2, s);
  NM_CUDA(cub::DeviceRunLengthEncode::Encode(tmp2.p, tb2, keys2.p, uniq.p, counts.p, nruns.p, cnt, s));
  c.launches += 2;
  int32_t v = 0;
  NM_CUDA(cudaMemcpyAsync(&v, nruns.p, 4, cudaMemcpyDeviceToHost, s));
  NM_CUDA(cudaStreamSynchronize(s));
  S.v = v;
  S.p.alloc(v, s);
  NM_CUDA(cudaMemcpyAsync(S.p.p, uniq.p, (size_t)v * 4, cudaMemcpyDeviceToDevice, s));
  S.pptr.alloc(v + 1, s);
  {
    // exclusive scan of counts[0..v] (counts[v] = 0)
    DBuf<int32_t> cz(v + 1, s);
    NM_CUDA(cudaMemcpyAsync(cz.p, counts.p, (size_t)v * 4, cudaMemcpyDeviceToDevice, s));
    NM_CUDA(cudaMemsetAsync(cz.p + v, 0, 4, s));
    size_t tb3 = 0;
    NM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb3, cz.p, S.pptr.p, v + 1, s));
    DBuf<char> tmp3(tb3, s);
    NM_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.p, tb3, cz.p, S.pptr.p, v + 1, s));
    c.launches += 1;
  }
  S.pcol.alloc(cnt, s);
  S.psign.alloc(cnt, s);
  NM_LAUNCH(c, "ss_unpack", k_ss_unpack<<<ceil_div(cnt, 256), 256, 0, s>>>(vals2, cnt, S.pcol, S.psign));
}

__device__ __forceinline__ float apply_log(float x, int logmode) {
  // trunc_log(x) = max(0, log x) = log(max(x, 1)); log1p(max(x, 0))   [R4]
  return logmode == 0 ? logf(fmaxf(x, 1.f)) : log1pf(fmaxf(x, 0.f));
}

// ---------------------------------------------------------------------------
// GEMM core: 64 (rows of A) × 64 (p-columns) tile, K = k, 256 threads, 4×4 each.
// A row-major (ld), B rows gathered through pidx.
// ---------------------------------------------------------------------------
constexpr int SM_ = 64, SN_ = 64, SK_ = 32;

struct GemmTile {
  float acc[4][4];
};

__device__ __forceinline__ void gemm_tile_abt(const Mat &A, int64_t r0, const float *__restrict__ Bp,
                                              int64_t ldb, const int32_t *__restrict__ pidx, int64_t v,
                                              int64_t j0, int64_t K, float (*As)[SM_ + 4],
                                              float (*Bs)[SN_ + 4], GemmTile &t) {
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) t.acc[i][j] = 0.f;
  for (int64_t k0 = 0; k0 < K; k0 += SK_) {
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      int idx = threadIdx.x + it * 256;  // 0..511 -> 64 rows × 8 float4
      int m = idx / 8, k4 = (idx % 8) * 4;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      int64_t row = r0 + m;
      if (k0 + k4 < K) {
        if (row < A.rows) a = *reinterpret_cast<const float4 *>(A.p + row * A.ld + k0 + k4);
        int64_t jj = j0 + m;
        if (jj < v) {
          int64_t br = pidx ? pidx[jj] : jj;
          b = *reinterpret_cast<const float4 *>(Bp + br * ldb + k0 + k4);
        }
        int64_t nv = K - (k0 + k4);
        if (nv < 4) { a.w = 0.f; b.w = 0.f; }
        if (nv < 3) { a.z = 0.f; b.z = 0.f; }
        if (nv < 2) { a.y = 0.f; b.y = 0.f; }
      }
      As[k4 + 0][m] = a.x; As[k4 + 1][m] = a.y; As[k4 + 2][m] = a.z; As[k4 + 3][m] = a.w;
      Bs[k4 + 0][m] = b.x; Bs[k4 + 1][m] = b.y; Bs[k4 + 2][m] = b.z; Bs[k4 + 3][m] = b.w;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < SK_; ++kk) {
      float4 a = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
      float4 b = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
      float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) t.acc[i][j] = fmaf(av[i], bv[j], t.acc[i][j]);
    }
    __syncthreads();
  }
}

// fused: Y[r0:r0+64, :h] = Σ_p-tiles scatter(f(scale G_tile))
constexpr int kFusedMaxH = 256;

__global__ void __launch_bounds__(256) k_sketch_fused(Mat A, const float *__restrict__ B, int64_t ldb,
                                                      const int32_t *__restrict__ p,
                                                      const int32_t *__restrict__ pptr,
                                                      const int32_t *__restrict__ pcol,
                                                      const float *__restrict__ psign, int64_t v,
                                                      int64_t K, float scale, int logmode, Mat Y) {
  extern __shared__ __align__(16) float smem[];
  float(*As)[SM_ + 4] = reinterpret_cast<float(*)[SM_ + 4]>(smem);
  float(*Bs)[SN_ + 4] = reinterpret_cast<float(*)[SN_ + 4]>(smem + SK_ * (SM_ + 4));
  float *Yt = smem + 2 * SK_ * (SM_ + 4);  // 64 × hp
  const int hp = (int)Y.cols + 1;          // pad against bank conflicts
  const int64_t r0 = (int64_t)blockIdx.x * SM_;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  for (int i = threadIdx.x; i < SM_ * hp; i += 256) Yt[i] = 0.f;
  __syncthreads();
  GemmTile t;
  for (int64_t j0 = 0; j0 < v; j0 += SN_) {
    gemm_tile_abt(A, r0, B, ldb, p, v, j0, K, As, Bs, t);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t jj = j0 + tx * 4 + j;
      if (jj >= v) break;
      const int e0 = pptr[jj], e1 = pptr[jj + 1];
      for (int e = e0; e < e1; ++e) {
        const int cc = pcol[e];
        const float sg = psign[e];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float g = apply_log(scale * t.acc[i][j], logmode);
          atomicAdd(&Yt[(ty * 4 + i) * hp + cc], sg * g);
        }
      }
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < SM_ * Y.cols; idx += 256) {
    int i = idx / (int)Y.cols, cc = idx % (int)Y.cols;
    int64_t row = r0 + i;
    if (row < Y.rows) Y.p[row * Y.ld + cc] = Yt[i * hp + cc];
  }
}

// unfused: Gf[rows × v] = f(scale A B(p,:)ᵀ)
__global__ void __launch_bounds__(256) k_gemm_abt_f(Mat A, const float *__restrict__ B, int64_t ldb,
                                                    const int32_t *__restrict__ p, int64_t v, int64_t K,
                                                    float scale, int logmode, float *__restrict__ Gf,
                                                    int64_t ldg) {
  __shared__ __align__(16) float As[SK_][SM_ + 4];
  __shared__ __align__(16) float Bs[SK_][SN_ + 4];
  const int64_t r0 = (int64_t)blockIdx.y * SM_, j0 = (int64_t)blockIdx.x * SN_;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  GemmTile t;
  gemm_tile_abt(A, r0, B, ldb, p, v, j0, K, As, Bs, t);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t row = r0 + ty * 4 + i;
    if (row >= A.rows) break;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t jj = j0 + tx * 4 + j;
      if (jj < v) Gf[row * ldg + jj] = apply_log(scale * t.acc[i][j], logmode);
    }
  }
}

// Y[i, :] = Σ_jj Gf[i, jj] Ψrow(jj): 16 rows per CTA, Y rows in shared memory
__global__ void __launch_bounds__(256) k_scatter_rows(const float *__restrict__ Gf, int64_t ldg,
                                                      int64_t rows, int64_t v,
                                                      const int32_t *__restrict__ pptr,
                                                      const int32_t *__restrict__ pcol,
                                                      const float *__restrict__ psign, Mat Y) {
  extern __shared__ float Ys[];  // 16 × Y.cols
  const int R = 16;
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const int h = (int)Y.cols;
  for (int i = threadIdx.x; i < R * h; i += blockDim.x) Ys[i] = 0.f;
  __syncthreads();
  const int w = threadIdx.x / 32, ln = threadIdx.x % 32;
  for (int rr = w; rr < R; rr += blockDim.x / 32) {
    int64_t row = r0 + rr;
    if (row >= rows) break;
    const float *g = Gf + row * ldg;
    for (int64_t jj = ln; jj < v; jj += 32) {
      float x = g[jj];
      if (x == 0.f) continue;
      for (int e = pptr[jj]; e < pptr[jj + 1]; ++e) atomicAdd(&Ys[rr * h + pcol[e]], psign[e] * x);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < R * h; i += blockDim.x) {
    int64_t row = r0 + i / h;
    if (row < rows) Y.p[row * Y.ld + i % h] = Ys[i];
  }
}

void sketch_apply(Ctx &c, const Mat &A, const Mat &B, const SparseSign &S, float scale, int logmode,
                  const Mat &Y) {
  NM_REQUIRE(A.cols == B.cols && Y.cols == S.h && Y.rows == A.rows, "sketch: shape mismatch");
  cudaStream_t s = c.stream;
  if (Y.cols <= kFusedMaxH) {
    size_t smem = (size_t)(2 * SK_ * (SM_ + 4) + SM_ * (Y.cols + 1)) * sizeof(float);
    static bool attr = false;
    if (!attr) {
      NM_CUDA(cudaFuncSetAttribute(k_sketch_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    NM_LAUNCH(c, "sketch_fused", k_sketch_fused<<<ceil_div(A.rows, SM_), 256, smem, s>>>(A, B.p, B.ld, S.p, S.pptr, S.pcol, S.psign,
                                                            S.v, A.cols, scale, logmode, Y));
  } else {
    int64_t ldg = pad4(S.v);
    DBuf<float> Gf((size_t)A.rows * ldg, s);
    dim3 grid(ceil_div(S.v, SN_), ceil_div(A.rows, SM_));
    NM_LAUNCH(c, "gemm_abt_f", k_gemm_abt_f<<<grid, 256, 0, s>>>(A, B.p, B.ld, S.p, S.v, A.cols, scale, logmode, Gf, ldg));
    size_t smem = (size_t)16 * Y.cols * sizeof(float);
    static bool attr2 = false;
    if (!attr2) {
      NM_CUDA(cudaFuncSetAttribute(k_scatter_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr2 = true;
    }
    NM_REQUIRE(smem <= 200 * 1024, "sketch: h too large");
    NM_LAUNCH(c, "scatter_rows", k_scatter_rows<<<ceil_div(A.rows, 16), 256, smem, s>>>(Gf, ldg, A.rows, S.v, S.pptr, S.pcol, S.psign, Y));
  }
}

// Out[j, :] = Σ_t sign[j,t] X[rows[j,t], :]  (fp64 accumulate)
__global__ void k_sign_gather(const int32_t *__restrict__ rows, const float *__restrict__ signs, int64_t h,
                              int z, Mat X, const int32_t *__restrict__ p, int64_t v,
                              double *__restrict__ Out, int64_t ldo) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= h * X.cols) return;
  int64_t j = idx / X.cols, cc = idx % X.cols;
  double s = 0.0;
  for (int t = 0; t < z; ++t) {
    int64_t r = rows[j * z + t];
    if (p) {  // map row id -> position in p (sorted)
      int64_t lo = 0, hi = v - 1;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (p[mid] < r) lo = mid + 1; else hi = mid;
      }
      r = lo;
    }
    s += (double)signs[j * z + t] * (double)X.p[r * X.ld + cc];
  }
  Out[j * ldo + cc] = s;
}

void sign_gather_T(Ctx &c, const SparseSign &S, const Mat &X, double *Out, int64_t ldo) {
  NM_LAUNCH(c, "sign_gather", k_sign_gather<<<ceil_div(S.h * X.cols, 256), 256, 0, c.stream>>>(S.rows, S.signs, S.h, (int)S.z, X,
                                                                   nullptr, 0, Out, ldo));
}

void sign_gather_T_p(Ctx &c, const SparseSign &S, const Mat &Xp, double *Out, int64_t ldo) {
  NM_LAUNCH(c, "sign_gather_p", k_sign_gather<<<ceil_div(S.h * Xp.cols, 256), 256, 0, c.stream>>>(S.rows, S.signs, S.h, (int)S.z, Xp,
                                                                    S.p, S.v, Out, ldo));
}

__global__ void k_gather_rows(Mat X, const int32_t *__restrict__ idx, int64_t cnt, Mat Out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= cnt * Out.cols) return;
  int64_t r = t / Out.cols, cc = t % Out.cols;
  Out.p[r * Out.ld + cc] = X.p[(int64_t)idx[r] * X.ld + cc];
}

void gather_rows(Ctx &c, const Mat &X, const int32_t *idx, int64_t cnt, const Mat &Out) {
  NM_LAUNCH(c, "gather_rows", k_gather_rows<<<ceil_div(cnt * Out.cols, 256), 256, 0, c.stream>>>(X, idx, cnt, Out));
}

}  // namespace netmfp
