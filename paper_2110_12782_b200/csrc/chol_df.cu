// chol_df.cu — CholeskyQR's small factorisation on many SMs:
//   G = Rᵀ R (R upper, G l×l SPD fp64),  Rinv = R⁻¹.
// The lower triangle is cut into 32×32 tiles; one CTA owns one tile (I, J),
// I >= J, and the tiles run as a dataflow graph synchronised through
// per-tile ready flags in global memory (release/acquire at gpu scope), so
// the critical path is ~2·nb tile steps instead of l column steps on one SM:
//   Cholesky (L = Rᵀ, right-looking by dependencies):
//     S_IJ = G_IJ − Σ_{K<J} L_IK L_JKᵀ      (waits for L_IK, L_JK)
//     L_JJ = chol(S_JJ), X_JJ = L_JJ⁻¹       (one warp, rows in registers)
//     L_IJ = S_IJ X_JJᵀ                      (waits for L_JJ, X_JJ; a tile GEMM)
//   inverse X = L⁻¹ (lower), pipelined behind the factorisation in the same attempt:
//     X_IJ = −X_II Σ_{K=J}^{I−1} L_IK X_KJ    (waits for L_IK, X_KJ, X_II)
//   Rinv = Xᵀ.
// A breakdown (pivot <= 1e-12 × original diagonal, or non-finite) raises a
// global fail word; every CTA notices it, the grid synchronises and all tiles
// restart from G (never written: L has its own buffer) with a diagonal shift
// (shifted CholeskyQR), as the
// single-CTA kernels in small.cu do.  Launched cooperatively (co-residency of
// the ≤ nb(nb+1)/2 CTAs is required by the spin waits).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

#ifdef CDF_PROF
__device__ unsigned long long g_cdf_t[64 * 16];
#define CDF_MARK(i)                                                                 \
  do {                                                                              \
    if (threadIdx.x == 0) {                                                         \
      unsigned long long _t;                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                        \
      g_cdf_t[blockIdx.x * 16 + (i)] = _t;                                           \
    }                                                                               \
  } while (0)
#else
#define CDF_MARK(i)
#endif
namespace netmfp {
namespace cdf {

constexpr int T = 256;
constexpr int TL = 33;  // smem tile row stride (doubles)

__device__ __forceinline__ int ld_relaxed(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct DfP {
  const double *G;  // l×l (ld), read only
  int64_t ld;
  int l, nb;
  double *L;   // l×l (ld = l): L in the lower tiles
  double *Rinv;  // l×l (ld = l); holds X = L⁻¹ (lower) before the final transpose
  int *lflag, *xflag;  // nb×nb ready flags (value = attempt + 1)
  int *fail;           // 0 = ok, else attempt+1 of the failing attempt
  int *flag;           // caller's status word (shift counter, 1<<30 on failure)
  double drop_tol;     // > 0: a pivot below drop_tol × its diagonal marks a dependent column
  int *dropped;        // l: attempt+1 of the attempt that dropped column j (else 0)
};

// wait until *f >= want (or the attempt failed); returns false on failure
__device__ bool wait_flag(const DfP &p, const int *f, int want, int attempt) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    // relaxed polls, one acquire fence once the flag is seen (an acquire
    // load at gpu scope invalidates the SM's L1 on every poll)
    int r = 1;
    while (ld_relaxed(f) < want) {
      if (ld_relaxed(p.fail) == attempt + 1) {
        r = 0;
        break;
      }
      __nanosleep(64);
    }
    asm volatile("fence.acquire.gpu;" ::: "memory");
    ok = r;
  }
  __syncthreads();
  const bool r = ok != 0;
  __syncthreads();
  return r;
}

__device__ void publish(int *f, int v) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(f, v);  // cumulative: the CTA's writes ordered by the barrier
}

// load a 32×32 tile (rows r0.., cols c0.., valid ib×jb, zero padded) bypassing L1
__device__ void load_tile(double *dst, const double *src, int64_t ld, int r0, int c0, int ib, int jb) {
  for (int i = threadIdx.x; i < 32 * 32; i += T) {
    const int r = i >> 5, c = i & 31;
    dst[r * TL + c] = (r < ib && c < jb) ? __ldcg(src + (int64_t)(r0 + r) * ld + c0 + c) : 0.0;
  }
}
__device__ void store_tile(double *dst, int64_t ld, const double *src, int r0, int c0, int ib, int jb) {
  for (int i = threadIdx.x; i < 32 * 32; i += T) {
    const int r = i >> 5, c = i & 31;
    if (r < ib && c < jb) __stcg(dst + (int64_t)(r0 + r) * ld + c0 + c, src[r * TL + c]);
  }
}

// S -= A · Bᵀ  (32×32 tiles in smem); thread owns 4 outputs (rows r, r+8, r+16, r+24)
__device__ void tile_sub_abt(double *S, const double *A, const double *B) {
  const int c = threadIdx.x & 31, r0 = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int t = 0; t < 32; ++t) {
    const double b = B[c * TL + t];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += A[(r0 + 8 * i) * TL + t] * b;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) S[(r0 + 8 * i) * TL + c] -= acc[i];
}
// S += A · B  (A, B, S 32×32 smem)
__device__ void tile_add_ab(double *S, const double *A, const double *B) {
  const int c = threadIdx.x & 31, r0 = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int t = 0; t < 32; ++t) {
    const double b = B[t * TL + c];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += A[(r0 + 8 * i) * TL + t] * b;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) S[(r0 + 8 * i) * TL + c] += acc[i];
}

// OUT = A · Bᵀ  (32×32 smem tiles)
__device__ void tile_mul_abt(double *OUT, const double *A, const double *B) {
  const int c = threadIdx.x & 31, r0 = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int t = 0; t < 32; ++t) {
    const double b = B[c * TL + t];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += A[(r0 + 8 * i) * TL + t] * b;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) OUT[(r0 + 8 * i) * TL + c] = acc[i];
}

// Warps 0 and 1: S (32×32, rows >= ib identity) -> L = chol(S) (lower, in S)
// and X = L⁻¹ (lower, in X).  Warp 0 factors right-looking with its row in
// registers, column j of L broadcast through shared memory, and publishes its
// progress after every column; warp 1 inverts one step behind (inverse step k
// needs only column k of L and 1/L[k][k]), so the inverse overlaps the factor
// instead of following it.  The inverse's register window shifts by one row
// per step (w[m] = row k + m), so one rolled loop body serves every step with
// register operands (the code runs once per tile from a cold instruction
// cache).  Returns (warp 0) true on breakdown (pivot <= 1e-12 × piv[j] or
// non-finite).
__device__ bool warp_chol_inv(double *S, double *X, double *rinv, const double *piv, int ib, volatile int *prog,
                              double drop_tol, int *dropped, int want) {
  const int r = threadIdx.x & 31;
  double w[32];
  if (threadIdx.x < 32) {
    CDF_MARK(10);
#pragma unroll
    for (int c = 0; c < 32; ++c) w[c] = S[r * TL + c];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      double d = __shfl_sync(0xffffffffu, w[j], j);  // S[j][j]
      // a (numerically) dependent column of an orthonormalising pass: its
      // Schur pivot is rounding noise; identity pivot, and its column of R⁻¹
      // is zeroed at the end (that column of Q comes out exactly zero, the
      // pseudo-inverse semantics of orth on range(Y) [R10])
      const bool drop = drop_tol > 0.0 && j < ib && isfinite(d) && d < drop_tol * piv[j];
      if (drop) {
        d = 1.0;
        if (r == 0) dropped[j] = want;
      }
      bad |= j < ib && !drop && (!(d > 1e-12 * piv[j]) || !isfinite(d));
      const double inv = rsqrt(fmax(d, 1e-300));
      const double l = r >= j ? w[j] * inv : 0.0;  // L[r][j]
      S[r * TL + j] = l;
      if (r == j) rinv[j] = inv;  // 1 / L[j][j]
      __threadfence_block();
      __syncwarp();
      if (r == 0) *prog = j + 1;  // column j and rinv[j] are final
#pragma unroll
      for (int c = j + 1; c < 32; ++c) w[c] -= l * S[c * TL + j];
    }
    __syncwarp();
    CDF_MARK(12);
    return bad;
  }
  // X = L⁻¹, lane r owning column r: x_k = acc_k / L[k][k], then the later
  // rows' partial sums (w[m] = row k + m)
#pragma unroll
  for (int i = 0; i < 32; ++i) w[i] = i == r ? 1.0 : 0.0;
#pragma unroll 1
  for (int k = 0; k < 32; ++k) {
    while (*prog <= k) {
    }
    __threadfence_block();
    const double xk = w[0] * rinv[k];
    X[k * TL + r] = xk;
#pragma unroll
    for (int m = 1; m < 32; ++m) w[m - 1] = w[m] - S[((k + m) & 31) * TL + k] * xk;
  }
  __syncwarp();
  CDF_MARK(14);
  return false;
}

__global__ void __launch_bounds__(T) k_chol_df(DfP p) {
  grid_dep_enter();
  cg::grid_group grid = cg::this_grid();
  __shared__ double S[32 * TL], A[32 * TL], B[32 * TL], D[32 * TL], E[32 * TL];
  __shared__ int bad;
  __shared__ double piv[32], rinv[32];
  __shared__ int prog;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // tile of this CTA: block 0 -> (0, 0); then the strictly lower tiles
  // (I, J), I > J, column-major.  The sub-diagonal CTA (J+1, J) also owns the
  // diagonal tile J+1 (accumulates its updates, factors it right after its own
  // L_{J+1,J}): one flag hop per block step on the critical path, not two.
  int I = 0, J = 0;
  if (blockIdx.x > 0) {
    int t = blockIdx.x - 1;
    while (t >= p.nb - 1 - J) {
      t -= p.nb - 1 - J;
      ++J;
    }
    I = J + 1 + t;
  }
  const bool owns_diag = (I == J) || (I == J + 1);  // (0,0) or a sub-diagonal tile
  const int ib = min(32, p.l - 32 * I), jb = min(32, p.l - 32 * J);
  CDF_MARK(0);
  // G stays intact (L goes to its own buffer), so a shifted retry restarts from it
  CDF_MARK(1);
  __shared__ double red[T / 32];
  double maxdiag = 0.0;
  for (int i = threadIdx.x; i < p.l; i += T) maxdiag = fmax(maxdiag, __ldcg(p.G + (int64_t)i * p.ld + i));
  for (int o = 16; o > 0; o >>= 1) maxdiag = fmax(maxdiag, __shfl_xor_sync(0xffffffffu, maxdiag, o));
  if (lane == 0) red[warp] = maxdiag;
  __syncthreads();
  maxdiag = 0.0;
  for (int w = 0; w < T / 32; ++w) maxdiag = fmax(maxdiag, red[w]);
  int attempt = 0;
  for (; attempt < 6; ++attempt) {
    const double shift = attempt == 0 ? 0.0 : maxdiag * 1e-7 * pow(100.0, (double)(attempt - 1));
    const int want = attempt + 1;
    bool alive = true;
    // S = G_IJ (+ shift on the diagonal); a sub-diagonal CTA also keeps the
    // diagonal tile I in E
    CDF_MARK(8);
    load_tile(S, p.G, p.ld, 32 * I, 32 * J, ib, jb);
    if (I == J + 1) load_tile(E, p.G, p.ld, 32 * I, 32 * I, ib, ib);
    __syncthreads();
    CDF_MARK(9);
    if (I == J)
      for (int i = threadIdx.x; i < ib; i += T) S[i * TL + i] += shift;
    if (I == J + 1)
      for (int i = threadIdx.x; i < ib; i += T) E[i * TL + i] += shift;
    // left-looking updates
    for (int K = 0; K < J && alive; ++K) {
      alive = wait_flag(p, p.lflag + I * p.nb + K, want, attempt) &&
              wait_flag(p, p.lflag + J * p.nb + K, want, attempt);
      if (!alive) break;
      load_tile(A, p.L, p.l, 32 * I, 32 * K, ib, 32);
      load_tile(B, p.L, p.l, 32 * J, 32 * K, jb, 32);
      __syncthreads();
      tile_sub_abt(S, A, B);
      if (I == J + 1) tile_sub_abt(E, A, A);  // diagonal I: - L_IK L_IKᵀ
      __syncthreads();
    }
    CDF_MARK(4);
    if (alive && I != J) {
      // L_IJ = S_IJ X_JJᵀ once the diagonal J is factored
      alive = wait_flag(p, p.lflag + J * p.nb + J, want, attempt);
      if (alive) {
        load_tile(D, p.Rinv, p.l, 32 * J, 32 * J, jb, jb);  // X_JJ
        __syncthreads();
        tile_mul_abt(A, S, D);  // L_IJ
        __syncthreads();
        store_tile(p.L, p.l, A, 32 * I, 32 * J, ib, jb);
        publish(p.lflag + I * p.nb + J, want);
        CDF_MARK(7);
        if (I == J + 1) {  // the diagonal I gets its last update from this CTA's own tile
          tile_sub_abt(E, A, A);
          __syncthreads();
          for (int i = threadIdx.x; i < 32 * TL; i += T) S[i] = E[i];
          __syncthreads();
        }
      }
    }
    if (alive && owns_diag) {
      // factor and invert the diagonal tile I (warp 0); rows beyond ib are identity padding
      if (threadIdx.x < 32) {
        for (int cc = 0; cc < 32; ++cc)
          if ((int)threadIdx.x >= ib) S[threadIdx.x * TL + cc] = (cc == (int)threadIdx.x) ? 1.0 : 0.0;
        const double g0 = (int)threadIdx.x < ib
                              ? __ldcg(p.G + (int64_t)(32 * I + threadIdx.x) * p.ld + 32 * I + threadIdx.x)
                              : 1.0;
        // an exactly-zero column of the Gram's input (zero row and column of
        // G, so of S): identity pivot — that column of Y R⁻¹ stays zero and
        // the others are untouched, i.e. orth on range(Y) [R10]
        if ((int)threadIdx.x < ib && g0 == 0.0) S[threadIdx.x * TL + threadIdx.x] = 1.0;
        piv[threadIdx.x] = (int)threadIdx.x < ib ? (g0 == 0.0 ? 1.0 : g0 + shift) : 1.0;
        if (threadIdx.x == 0) prog = 0;
      }
      __syncthreads();
      if (threadIdx.x < 64) {
        const bool b = warp_chol_inv(S, D, rinv, piv, ib, &prog, p.drop_tol, p.dropped + 32 * I, want);
        if (threadIdx.x == 0) bad = b;
      }
      __syncthreads();
      CDF_MARK(11);
      if (bad) {
        if (threadIdx.x == 0) atomicMax(p.fail, want);
        alive = false;
      } else {
        store_tile(p.L, p.l, S, 32 * I, 32 * I, ib, ib);
        store_tile(p.Rinv, p.l, D, 32 * I, 32 * I, ib, ib);  // X_II for the L_JI GEMMs and the inverse
        CDF_MARK(13);
        publish(p.lflag + I * p.nb + I, want);
        publish(p.xflag + I * p.nb + I, want);
        CDF_MARK(7);
      }
    }
    // inverse X = L⁻¹ of this tile, pipelined behind the factorisation:
    // X_IJ = -X_II Σ_{K=J}^{I-1} L_IK X_KJ as its inputs appear (flags of this attempt)
    if (alive && I != J) {
      for (int i = threadIdx.x; i < 32 * TL; i += T) S[i] = 0.0;
      __syncthreads();
      for (int K = J; K < I && alive; ++K) {
        alive = (K == J || wait_flag(p, p.lflag + I * p.nb + K, want, attempt)) &&
                wait_flag(p, p.xflag + K * p.nb + J, want, attempt);
        if (!alive) break;
        load_tile(A, p.L, p.l, 32 * I, 32 * K, ib, 32);    // L_IK
        load_tile(B, p.Rinv, p.l, 32 * K, 32 * J, 32, jb);  // X_KJ
        __syncthreads();
        tile_add_ab(S, A, B);
        __syncthreads();
      }
      if (alive) alive = wait_flag(p, p.xflag + I * p.nb + I, want, attempt);
      if (alive) {
        load_tile(A, p.Rinv, p.l, 32 * I, 32 * I, ib, ib);  // X_II
        for (int i = threadIdx.x; i < 32 * TL; i += T) D[i] = 0.0;
        __syncthreads();
        tile_add_ab(D, A, S);  // D = X_II · S
        __syncthreads();
        for (int i = threadIdx.x; i < 32 * TL; i += T) D[i] = -D[i];
        __syncthreads();
        store_tile(p.Rinv, p.l, D, 32 * I, 32 * J, ib, jb);
        publish(p.xflag + I * p.nb + J, want);
      }
    }
    CDF_MARK(2);
    grid.sync();
    CDF_MARK(3);
    if (__ldcg(p.fail) != want) break;  // this attempt succeeded
  }
  if (attempt >= 6) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(p.flag, 1 << 30);
    return;
  }
  if (attempt > 0 && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(p.flag, 1);
  CDF_MARK(4);
  CDF_MARK(5);
  // ---- Rinv = Xᵀ: this CTA transposes its own tile pair (and its diagonal)
  if (owns_diag) {
    load_tile(A, p.Rinv, p.l, 32 * I, 32 * I, ib, ib);
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 32; i += T) {
      const int r = i >> 5, c = i & 31;
      const bool dz = p.drop_tol > 0.0 && c < ib && __ldcg(p.dropped + 32 * I + c) == attempt + 1;
      if (r < ib && c < ib) p.Rinv[(int64_t)(32 * I + r) * p.l + 32 * I + c] = (c >= r && !dz) ? A[c * TL + r] : 0.0;
    }
    __syncthreads();
  }
  if (I != J) {
    load_tile(A, p.Rinv, p.l, 32 * I, 32 * J, ib, jb);
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 32; i += T) {
      const int r = i >> 5, c = i & 31;
      const bool dz = p.drop_tol > 0.0 && c < ib && __ldcg(p.dropped + 32 * I + c) == attempt + 1;
      if (r < jb && c < ib) p.Rinv[(int64_t)(32 * J + r) * p.l + 32 * I + c] = dz ? 0.0 : A[c * TL + r];
      if (r < ib && c < jb) p.Rinv[(int64_t)(32 * I + r) * p.l + 32 * J + c] = 0.0;
    }
  }
  CDF_MARK(6);
}

}  // namespace cdf

// G = RᵀR → Rinv = R⁻¹ on 1 + nb(nb-1)/2 co-resident CTAs (cooperative launch)
void chol_inv_df(Ctx &c, double *G, int64_t l, int64_t ld, double *Rinv, int *flag, double drop_tol) {
  using namespace cdf;
  const int nb = (int)ceil_div(l, 32);
  const int tiles = 1 + nb * (nb - 1) / 2;  // (0,0) and the strictly lower tiles
  DBuf<double> L((size_t)l * l, c.stream);
  DBuf<int> flags((size_t)2 * nb * nb + 1 + 32 * nb, c.stream);
  NM_CUDA(cudaMemsetAsync(flags.p, 0, flags.n * sizeof(int), c.stream));
  DfP p{};
  p.G = G;
  p.ld = ld;
  p.l = (int)l;
  p.nb = nb;
  p.L = L.p;
  p.Rinv = Rinv;
  p.lflag = flags.p;
  p.xflag = flags.p + nb * nb;
  p.fail = flags.p + 2 * nb * nb;
  p.flag = flag;
  p.drop_tol = drop_tol;
  p.dropped = flags.p + 2 * nb * nb + 1;
  void *args[] = {&p};
  NM_LAUNCH(c, "chol_df", NM_CUDA(cudaLaunchCooperativeKernel((void *)k_chol_df, dim3(tiles), dim3(T), args, 0,
                                                                c.stream)));
}

}  // namespace netmfp
