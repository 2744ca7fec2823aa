// pipeline.cu — the NetMF+ stages of Alg. 5 on device blocks.
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "pipeline.cuh"

namespace netmfp {

// Alg. 2 / Alg. 4 orthonormalisations must succeed (shifted retries
// included); the failure bit is checked once, at the end of the ABI call
// (api.cu finish), instead of draining the stream here.
static void check_flag(Ctx &c, const char *what) { c.flag_checks.push_back(what); }

// CholeskyQR (north_star; [R7]): Gram G = YᵀY (fp64), G = RᵀR, out = rs · Y R⁻¹.
// passes = 2 gives CholeskyQR2 (second pass on the materialised Y R1⁻¹ in tmp).
// orthonormal = false (a power iteration's intermediate basis, which the next
// iteration re-orthonormalises; only its span matters) and every pass but the
// last of a CholeskyQR2: the Gram is a single tf32 product and the basis
// change uses R⁻¹ rounded to tf32 (any invertible R keeps the span; the
// columns come out orthonormal to ~1e-3), 1 and 2 tensor-core products
// instead of 3.
void cholqr(Ctx &c, const Mat &Y, const Mat &out, const int32_t *deg, float rexp, int passes,
            const Mat *tmp, bool orthonormal) {
  NM_STAGE(c, "stage_cholqr");
  const int64_t l = Y.cols;
  cudaStream_t s = c.stream;
  DBuf<double> G((size_t)l * l, s), Rinv((size_t)l * l, s);
  Mat cur = Y;
  for (int ps = 0; ps < passes; ++ps) {
    // the Gram of a pass whose output is only an intermediate basis (not the
    // last pass of an orthonormal CholeskyQR) need not be fp32-accurate
    gram(c, cur, cur, nullptr, 0.f, G, l, orthonormal && ps + 1 == passes);
    dist_allreduce(c, G, (size_t)l * l, DType::F64);  // Gram over all ranks' rows
    // the pass whose output must be orthonormal drops numerically dependent
    // columns (pivot < 1e-8 of the column's own diagonal): after a first pass
    // such a column is rounding noise inside span(Y) [R10]
    chol_inv_upper(c, G, l, l, Rinv, c.d_flags, orthonormal && ps + 1 == passes && passes > 1 ? 1e-8 : 0.0);
    const bool last = (ps + 1 == passes);
    if (last) {
      gemm_tall_tri(c, cur, Rinv, l, deg, rexp, out, orthonormal);
    } else {
      NM_REQUIRE(tmp && tmp->p != cur.p, "cholqr2: needs a scratch block");
      gemm_tall_tri(c, cur, Rinv, l, nullptr, 0.f, *tmp, false);
      cur = *tmp;
    }
  }
}

// Alg. 2 freigs(D^-α A D^-α, k, s1, q) with the basis kept pre-scaled
// (P = D^-α Q) so that every SpMM is an unweighted gather with a row scale:
//   X Q = D^-α A P;  X X Q = D^-α A (D^-2α A P);  S = Qᵀ X Q = Pᵀ (A P);  U = D^α P Û.
void freigs(Ctx &c, const Graph &g, double alpha, int k, int s1, int q, uint64_t seed, const Mat &U,
            double *lam_dev, bool out_F) {
  const int64_t n = g.n, l = (int64_t)k + s1;
  NM_REQUIRE(k >= 1 && s1 >= 0 && q >= 0, "eig: need k >= 1, s1 >= 0, q >= 0");
  NM_REQUIRE(l <= g.n_global, "eig: k + s1 must not exceed n (Alg. 2)");
  NM_REQUIRE(alpha > 0.0 && alpha <= 0.5, "eig: alpha in (0, 0.5] (PAPER.md:217)");
  cudaStream_t s = c.stream;
  const float a = (float)alpha;
  Block P(n, l, s), T(n, l, s), Y(n, l, s);
  DBuf<float> xfull;  // all ranks' rows of the SpMM input (multi-GPU only)
  // step 2: Ω = randn(n, l), Y = X Ω
  gaussian_block(c, P.m, seed, g.deg, a, g.row0, g.orig_id.p);  // P = D^-α Ω (this rank's rows)
  SpmmArgs sp;
  sp.cols = l;
  sp.Y = Y.m.p; sp.ldy = Y.m.ld; sp.a = a;
  dist_spmm(c, g, P.m, sp, xfull);
  // step 3: Q = orth(Y)
  cholqr(c, Y.m, P.m, g.deg, a, q == 0 ? 2 : 1, &T.m, q == 0);
  // steps 4-6: Q = orth(X X Q)
  for (int it = 0; it < q; ++it) {
    SpmmArgs s1a;
    s1a.cols = l;
    s1a.Y = T.m.p; s1a.ldy = T.m.ld; s1a.a = 2.f * a;
    dist_spmm(c, g, P.m, s1a, xfull);  // T = D^-2α A P = D^-α (X Q)
    SpmmArgs s2a;
    s2a.cols = l;
    s2a.Y = Y.m.p; s2a.ldy = Y.m.ld; s2a.a = a;
    dist_spmm(c, g, T.m, s2a, xfull);  // Y = D^-α A T = X X Q
    cholqr(c, Y.m, P.m, g.deg, a, it + 1 == q ? 2 : 1, &T.m, it + 1 == q);
  }
  check_flag(c, "freigs orthonormalisation");
  // step 7: S = Qᵀ X Q = Pᵀ A P
  SpmmArgs s3;
  s3.cols = l;
  s3.Y = T.m.p; s3.ldy = T.m.ld; s3.a = 0.f;
  dist_spmm(c, g, P.m, s3, xfull);
  xfull.release();
  DBuf<double> S((size_t)l * l, s), lam(l, s), V((size_t)l * l, s);
  gram(c, P.m, T.m, nullptr, 0.f, S, l, true, true);  // S = Pᵀ (A P) is symmetric: upper tiles only
  dist_allreduce(c, S, (size_t)l * l, DType::F64);
  symmetrize64(c, S, l, l);
  // step 8: [Û, Λ] = eig(S), ordered by |λ| [R3]
  {
    NM_STAGE(c, "stage_sym_eig");
    sym_eig(c, S, l, lam, V, true);
  }
  // step 9-10: U = Q Û(:, 1:k) = D^α P Û(:, 1:k)
  // U = D^α P Û, or (out_F) directly F = D^(-1+α) U = D^(-1+2α) P Û (Eq. 3)
  gemm_tall(c, P.m, V, l, k, g.deg, out_F ? (float)(1.0 - 2.0 * alpha) : -a, U);
  NM_CUDA(cudaMemcpyAsync(lam_dev, lam.p, (size_t)k * 8, cudaMemcpyDeviceToDevice, s));
}

// Eq. 3 / Alg. 5 steps 2-3
void factor_pair(Ctx &c, const Graph &g, double alpha, int T, const Mat &U, const double *lam, int k,
                 const Mat &F, double *C, bool u_is_F) {
  NM_REQUIRE(T >= 1, "factor_pair: T >= 1");
  cudaStream_t s = c.stream;
  DBuf<double> K((size_t)k * k, s), Pw((size_t)k * k, s), Pn((size_t)k * k, s), acc((size_t)k * k, s);
  // K = Uᵀ D^(-1+2α) U Λ  (= Fᵀ D F Λ with F = D^(-1+α) U)
  if (u_is_F)
    gram(c, U, U, g.deg, -1.f, K, k);
  else
    gram(c, U, U, g.deg, (float)(1.0 - 2.0 * alpha), K, k);
  dist_allreduce(c, K, (size_t)k * k, DType::F64);
  scale_cols64(c, K, k, k, k, lam, 0);
  // Σ_{r=1}^T K^(r-1) = S_T with S_m = Σ_{r<m} K^r, P_m = K^m, by the bits of T
  // from the top: S_{2m} = S_m + P_m S_m, P_{2m} = P_m²; S_{m+1} = S_m + P_m,
  // P_{m+1} = P_m K  (T = 10: 5 k×k GEMMs instead of 9)
  DBuf<double> Tm((size_t)k * k, s);
  set_identity64(c, acc, k, k);                                                  // S_1 = I
  NM_CUDA(cudaMemcpyAsync(Pw.p, K.p, (size_t)k * k * 8, cudaMemcpyDeviceToDevice, s));  // P_1 = K
  int top = 0;
  while ((T >> (top + 1)) != 0) ++top;
  int m = 1;
  for (int b = top - 1; b >= 0; --b) {
    const bool inc = (T >> b) & 1;
    const bool last = b == 0;
    // double: S = S + P S (P = K, S = I at m = 1: S = I + K), P = P P
    if (m == 1) {
      axpy64(c, (int64_t)k * k, 1.0, Pw, acc);
    } else {
      gemm64(c, false, false, k, k, k, 1.0, Pw, k, acc, k, 0.0, Tm, k);
      axpy64(c, (int64_t)k * k, 1.0, Tm, acc);
    }
    m *= 2;
    if (!(last && !inc)) {  // P_{2m} only if used later
      gemm64(c, false, false, k, k, k, 1.0, Pw, k, Pw, k, 0.0, Pn, k);
      std::swap(Pw.p, Pn.p);
    }
    if (inc) {  // S = S + P, P = P K
      axpy64(c, (int64_t)k * k, 1.0, Pw, acc);
      m += 1;
      if (!last) {
        gemm64(c, false, false, k, k, k, 1.0, Pw, k, K, k, 0.0, Pn, k);
        std::swap(Pw.p, Pn.p);
      }
    }
  }
  // C = Λ · acc
  NM_CUDA(cudaMemcpyAsync(C, acc.p, (size_t)k * k * 8, cudaMemcpyDeviceToDevice, s));
  scale_cols64(c, C, k, k, k, lam, 1);
  // F = D^(-1+α) U
  if (!u_is_F) scale_copy_block(c, U, F, g.deg, (float)(1.0 - alpha));
}

__global__ void k_sqrt_abs(const double *lam, int d, double *out) {
  grid_dep_enter();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) out[i] = sqrt(fabs(lam[i]));
}
__global__ void k_abs(const double *lam, int d, double *out) {
  grid_dep_enter();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) out[i] = fabs(lam[i]);
}

// Side stream (one GPU): side_fork() makes c.stream the side stream, ordered
// after everything queued so far on the main one; side_join_point() records
// where it ends and switches back; the main stream waits on c.ev_join where it
// needs the side's results.  NETMFP_SIDE_STREAM=0 keeps everything on the main
// stream (A/B measurements).
bool side_fork(Ctx &c) {
  static const bool side_on = [] {
    const char *v = getenv("NETMFP_SIDE_STREAM");
    return !(v && atoi(v) == 0);
  }();
  if (!side_on || c.nranks != 1 || c.comm || c.ops_on) return false;
  if (!c.side) {
    NM_CUDA(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
    NM_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    NM_CUDA(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
  }
  NM_CUDA(cudaEventRecord(c.ev_fork, c.stream));
  NM_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
  c.stream = c.side;
  return true;
}
void side_join_point(Ctx &c, cudaStream_t main) {
  NM_CUDA(cudaEventRecord(c.ev_join, c.side));
  c.stream = main;
}

// Alg. 4
void sketch_svd(Ctx &c, const Mat &F, const double *C, int k, double scale, int d, int s2, int s3, int z,
                uint64_t seed, int logmode, const Mat *Uout, double *sigma_dev, const Mat *Eout,
                const Mat *Yout, double *Zout, int64_t row0, int64_t n_global, const int32_t *comp_id,
                const SketchA *preA) {
  const int64_t n = F.rows;  // this rank's rows [row0, row0 + n) of n_global
  if (n_global < 0) n_global = n;
  // comp_id (compacted graph): Ψ and Π are drawn over the n_global original
  // vertices and their rows mapped to compact rows (-1: isolated, zero terms)
  const int64_t h2 = (int64_t)d + s2, h3 = (int64_t)d + s3;
  NM_REQUIRE(d >= 1 && s2 >= 0 && s3 >= 0, "sketch_svd: need d >= 1, s2, s3 >= 0");
  NM_REQUIRE(h2 <= n_global && h3 <= n_global * (int64_t)z, "sketch_svd: d + s2 must not exceed n");
  NM_REQUIRE(h3 >= h2, "sketch_svd: need s3 >= s2 (PAPER.md:413)");
  cudaStream_t s = c.stream;
  const float fs = (float)scale;
  // step 2: Ψ
  SparseSign Psi;
  {
    NM_STAGE(c, "stage_gen_sparse_sign");
    gen_sparse_sign(c, n_global, h2, z, seed, kTagPsi, Psi);
    if (comp_id) remap_rows(c, Psi.rows, h2 * z, comp_id);
  }
  // step 3: Y = f(scale F C F(p,:)ᵀ) Ψ  (Eq. 5, column group by column group of Ψ)
  Block Y(n, h2, s), Qb(n, h2, s), Tb(n, h2, s);
  {
    NM_STAGE(c, "stage_sketch_y");
    tc_sketch_y(c, F, C, k, Psi.rows, Psi.signs, h2, z, fs, logmode, Y.m, row0, preA);
  }
  if (Yout) copy_block(c, Y.m.p, Y.m.ld, Yout->p, Yout->ld, n, h2);
  // steps 5-6 need F, C and Π only, not Q: on one GPU they run on the side
  // stream while step 4 (CholeskyQR2 of Y, whose Cholesky factors occupy 37
  // SMs on a latency-bound chain) runs on the main one; joined before step 7
  const bool fork = side_fork(c);
  DBuf<double> Z((size_t)h3 * h3, s), PtQ((size_t)h3 * h2, s);
  SparseSign Pi;
  try {
    // step 5: Π
    {
      NM_STAGE(c, "stage_gen_sparse_sign");
      gen_sparse_sign(c, n_global, h3, z, seed, kTagPi, Pi);
      if (comp_id) remap_rows(c, Pi.rows, h3 * z, comp_id);
    }
    // step 6: Z = Πᵀ f(scale F(p,:) C F(p,:)ᵀ) Π  (both sides restricted to Π's coordinates)
    NM_STAGE(c, "stage_sketch_z");
    DBuf<float> Zf((size_t)h3 * h3, c.stream);
    tc_sketch_z(c, F, C, k, Pi.rows, Pi.signs, h3, z, fs, logmode, Zf, h3, row0);
    f32_to_f64(c, Zf, h3, Z, h3, h3, h3);
  } catch (...) {
    c.stream = s;
    throw;
  }
  if (fork) {
    side_join_point(c, s);
    Pi.rows.s = s;  // freed after their last use on the main stream
    Pi.signs.s = s;
  }
  // step 4: Q = orth(Y)   (CholeskyQR2 [R7])
  cholqr(c, Y.m, Qb.m, nullptr, 0.f, 2, &Tb.m);
  check_flag(c, "single-pass SVD orth(Y)");
  if (fork) NM_CUDA(cudaStreamWaitEvent(s, c.ev_join, 0));
  NM_STAGE(c, "stage_sketch_z_core");
  if (Zout) NM_CUDA(cudaMemcpyAsync(Zout, Z.p, (size_t)h3 * h3 * 8, cudaMemcpyDeviceToDevice, s));
  // step 7: S = (ΠᵀQ)† Z (QᵀΠ)†  via the normal equations in fp64
  sign_gather_T(c, Pi, Qb.m, PtQ, h2, row0);
  dist_allreduce(c, PtQ, (size_t)h3 * h2, DType::F64);
  DBuf<double> N((size_t)h2 * h2, s), Ninv((size_t)h2 * h2, s), Rinv((size_t)h2 * h2, s);
  DBuf<double> W((size_t)h2 * h3, s), WZ((size_t)h2 * h3, s), S((size_t)h2 * h2, s);
  gemm64(c, true, false, h2, h2, h3, 1.0, PtQ, h2, PtQ, h2, 0.0, N, h2);  // N = AᵀA
  chol_inv_upper(c, N, h2, h2, Rinv, c.d_flags);
  gemm64(c, false, true, h2, h2, h2, 1.0, Rinv, h2, Rinv, h2, 0.0, Ninv, h2);  // (AᵀA)⁻¹
  gemm64(c, false, true, h2, h3, h2, 1.0, Ninv, h2, PtQ, h2, 0.0, W, h3);      // A† = (AᵀA)⁻¹Aᵀ
  gemm64(c, false, false, h2, h3, h3, 1.0, W, h3, Z, h3, 0.0, WZ, h3);
  gemm64(c, false, true, h2, h2, h3, 1.0, WZ, h3, W, h3, 0.0, S, h2);
  symmetrize64(c, S, h2, h2);
  check_flag(c, "single-pass SVD core solve");
  // step 8: svd(S) of the symmetric core = eig with |λ| ordering
  DBuf<double> lam(h2, s), V((size_t)h2 * h2, s), sq(d, s);
  {
    NM_STAGE(c, "stage_sym_eig");
    sym_eig(c, S, h2, lam, V, true);
  }
  if (sigma_dev) {
    NM_LAUNCH(c, "abs", launch_pdl(s, k_abs, ceil_div(d, 128), 128, 0, lam, d, sigma_dev));
  }
  // step 9: U = Q Û(:, 1:d);  Alg. 5 step 5: E = U √Σ
  if (Uout) gemm_tall(c, Qb.m, V, h2, d, nullptr, 0.f, *Uout);
  if (Eout) {
    NM_LAUNCH(c, "sqrt_abs", launch_pdl(s, k_sqrt_abs, ceil_div(d, 128), 128, 0, lam, d, sq));
    DBuf<double> Vs((size_t)h2 * d, s);
    NM_CUDA(cudaMemcpy2DAsync(Vs.p, d * 8, V.p, h2 * 8, d * 8, h2, cudaMemcpyDeviceToDevice, s));
    scale_cols64(c, Vs, h2, d, d, sq, 0);
    gemm_tall(c, Qb.m, Vs, d, d, nullptr, 0.f, *Eout);
  }
}

// Chebyshev coefficients of the band-pass kernel [R6] (host, fp64)
void cheb_coeffs(int order, double mu, double theta, double *c) {
  const int N = 256;
  const double PI = 3.14159265358979323846;
  for (int r = 0; r <= order; ++r) {
    double sacc = 0.0;
    for (int j = 0; j < N; ++j) {
      double t = PI * (j + 0.5) / N;
      double x = std::cos(t);
      double lam = x + 1.0;
      double g = std::exp(-0.5 * ((lam - mu) * (lam - mu) - 1.0) * theta);
      sacc += g * std::cos(r * t);
    }
    c[r] = 2.0 / N * sacc;
  }
  c[0] *= 0.5;
  const double c0 = c[0];
  for (int r = 0; r <= order; ++r) c[r] /= c0;
}

// E <- Σ_{r=0}^{N} c_r T_r(L~) E, L~ = -D^-1 A (Chebyshev filter [R6]),
// evaluated by Clenshaw's recurrence (the same polynomial):
//   b_{N+1} = b_{N+2} = 0,  b_r = c_r E + 2 L~ b_{r+1} - b_{r+2} (r = N..1),
//   result = c_0 E + L~ b_1 - b_2.
// N SpMMs as the three-term forward recurrence, but each step streams two
// blocks and writes one (gathered b_{r+1}; b_{r+2} and E read; b_r written
// over b_{r+2} by the thread that read it) instead of streaming two and
// writing two; b_N = c_N E is never materialised (folded into the next two
// steps' multiple of E), and the last step writes the result into E.
void propagate(Ctx &c, const Graph &g, const Mat &E, int order, double mu, double theta) {
  if (order <= 0) return;
  NM_REQUIRE(order <= 64, "propagate: order <= 64");
  const int N = order;
  std::vector<double> cf(N + 1);
  cheb_coeffs(N, mu, theta, cf.data());
  cudaStream_t s = c.stream;
  const int64_t n = E.rows, d = E.cols;
  Block B0(n, d, s), B1(n, d, s);
  DBuf<float> xfull;  // all ranks' rows of the SpMM input (multi-GPU only)
  // one fused step: out = sE·E + coef·D^-1 A X (+ beta·prev)
  auto step = [&](const Mat &X, double coef, const Mat *prev, double beta, double sE, const Mat &out) {
    SpmmArgs a;
    a.cols = d;

    a.Y = nullptr;
    a.a = 1.f;
    a.coef = (float)coef;
    if (prev) {
      a.prev = prev->p;
      a.ldp = prev->ld;
      a.beta = (float)beta;
    }
    a.acc_in = E.p;
    a.ldai = E.ld;
    a.acc_scale = (float)sE;
    a.gamma = 1.f;
    a.acc_out = out.p;
    a.ldacc = out.ld;
    dist_spmm(c, g, X, a, xfull);
  };
  if (N == 1) {  // c0 E + c1 L~ E: E is gathered, so the result goes through a scratch block
    step(E, -cf[1], nullptr, 0.0, cf[0], B0.m);
    copy_block(c, B0.m.p, B0.m.ld, E.p, E.ld, n, d);
    return;
  }
  // b_{N-1} = c_{N-1} E + 2 L~ (c_N E)
  Mat bnext = B0.m, bcur = B1.m;  // b_{r+1}, and the buffer b_r will overwrite (b_{r+2})
  step(E, -2.0 * cf[N], nullptr, 0.0, cf[N - 1], bnext);
  // b_{N-2} = c_{N-2} E + 2 L~ b_{N-1} - c_N E   (b_N not materialised)
  // ... b_r = c_r E + 2 L~ b_{r+1} - b_{r+2}, b_r over b_{r+2}
  for (int r = N - 2; r >= 1; --r) {
    if (r == N - 2)
      step(bnext, -2.0, nullptr, 0.0, cf[r] - cf[N], bcur);
    else
      step(bnext, -2.0, &bcur, -1.0, cf[r], bcur);
    std::swap(bnext, bcur);  // bnext = b_r, bcur = b_{r+1}
  }
  // result = c_0 E + L~ b_1 - b_2 into E (E read and written per element by
  // one thread, not gathered); N == 2: b_2 = c_2 E
  if (N == 2)
    step(bnext, -1.0, nullptr, 0.0, cf[0] - cf[2], E);
  else
    step(bnext, -1.0, &bcur, -1.0, cf[0], E);
}

}  // namespace netmfp
