// kernels.cuh — internal interfaces between the .cu translation units.
#pragma once
#include "common.cuh"

namespace netmfp {

// ---- build_csr.cu
// CSR of rows [row0, row1) (default: all rows) with global column ids; the
// edge list must contain every edge incident to those rows.
// nullptr if nothing to drop; degall = every vertex's degree (g.deg for one rank)
Graph *compact_graph(Ctx &c, const Graph &g, const int32_t *degall);
void remap_rows(Ctx &c, int32_t *rows, int64_t m, const int32_t *comp);
Graph *build_csr_device(Ctx &c, int64_t n, const int32_t *src, const int32_t *dst, int64_t m, int64_t row0 = 0,
                        int64_t row1 = -1);

// ---- dist.cu
enum class DType { F32, F64, I64, I32, U8 };
void dist_unique_id(void *out);
void dist_init(Ctx &c, const void *id, int nranks, int rank);
void dist_destroy(Ctx &c);
void dist_init_ops(Ctx &c, const netmfp_comm_ops &ops, int nranks, int rank);
void dist_allreduce(Ctx &c, void *buf, size_t count, DType t);  // in place, sum
// out[0, n_global) = every rank's local int32 vector (rank r's at bounds[r])
void dist_allgather_i32(Ctx &c, const int32_t *local, const std::vector<int64_t> &bounds, int32_t *out);
// full n_global × local.ld block gathered from every rank's rows (identity for one rank)
const float *dist_gather_rows(Ctx &c, const Graph &g, const Mat &local, DBuf<float> &scratch);

// ---- spmm.cu
struct SpmmArgs {
  const float *X = nullptr;
  int64_t ldx = 0;
  float *Y = nullptr;  // may be null (only acc_out written)
  int64_t ldy = 0;
  int64_t cols = 0;
  float a = 0.f;                 // row scale d_u^-a (computed from rowptr)
  const float *s_col = nullptr;  // optional column scale vector (n), e.g. d_v^-b
  float coef = 1.f;              // y = coef * rs * sum + beta * prev
  const float *prev = nullptr;
  int64_t ldp = 0;
  float beta = 0.f;
  const float *acc_in = nullptr;  // acc_out = acc_scale * acc_in + gamma * y
  int64_t ldai = 0;
  float *acc_out = nullptr;
  int64_t ldacc = 0;
  float acc_scale = 0.f;
  float gamma = 0.f;
  int light_cap = kLightCapDefault;  // filled from the graph by spmm()
  int heavy_seg = kHeavySegDefault;
};
void spmm(Ctx &c, const Graph &g, const SpmmArgs &p);
// SpMM of a row-partitioned block: `local` is this rank's rows of X; the
// input rows of every rank are all-gathered (NCCL: by column slices on the
// communicator's stream, each slice's SpMM pass starting as soon as its rows
// arrived, overlapping the next slice's transfer).  One rank: spmm on local.
void dist_spmm(Ctx &c, const Graph &g, const Mat &local, const SpmmArgs &p, DBuf<float> &scratch);
void deg_pow(Ctx &c, const Graph &g, float e, float *out);  // out[i] = d_i^-e (0 if d_i = 0)

// ---- dense.cu (tall-skinny fp32 blocks, fp64 small results)
// G[a×b] (fp64, row-major ldg) = Σ_i w_i A[i,:a]ᵀ B[i,:b]; w optional (row weight
// d_i^-e when wexp != 0, computed from deg).  If A == B and a == b only the
// upper triangle is computed and mirrored.
// exact = false: tf32 products only (~1e-3 relative; for CholeskyQR passes
// whose output only needs to be a well-conditioned basis of the same span)
// sym_result: AᵀWB is known to be symmetric (e.g. Pᵀ(A P) with A symmetric):
// only the upper block-triangle is computed and mirrored.
void gram(Ctx &c, const Mat &A, const Mat &B, const int32_t *deg, float wexp, double *G, int64_t ldg,
          bool exact = true, bool sym_result = false);
// C[n×b] = rs_i · (A[n×a] · Bs[a×b]) with Bs fp64 small (converted to fp32),
// rs_i = d_i^-e (e = rexp, deg != null) else 1.
void gemm_tall(Ctx &c, const Mat &A, const double *Bs, int64_t ldb, int64_t bcols, const int32_t *deg,
               float rexp, const Mat &C);
// tensor-core (tcgen05, 3xTF32) versions (any width: outputs in column groups of <= 288)
void tc_gemm_tall(Ctx &c, const Mat &A, const double *Bs, int64_t ldb, int64_t bcols, const int32_t *deg,
                  float rexp, const Mat &C);
void tc_gram(Ctx &c, const Mat &A, const Mat &B, const int32_t *deg, float wexp, double *G, int64_t ldg,
             bool exact = true, bool sym_result = false);
void tc_gemm_tall_tri(Ctx &c, const Mat &A, const double *Rinv, int64_t ldb, int64_t bcols, const int32_t *deg,
                      float rexp, const Mat &C, bool exact = true);
// C = rs · A · Rinv with Rinv (a×a) upper triangular (CholeskyQR's Y R⁻¹).  exact =
// false: Rinv rounded to tf32 (the product is exact for that R̃⁻¹: same span,
// orthonormal to ~1e-3 — for CholeskyQR passes another pass follows)
void gemm_tall_tri(Ctx &c, const Mat &A, const double *Rinv, int64_t ldb, const int32_t *deg, float rexp,
                   const Mat &C, bool exact = true);
// Ω = randn(n, l) from Philox [R1], row-scaled by d_i^-e (deg != null)
void gaussian_block(Ctx &c, const Mat &O, uint64_t seed, const int32_t *deg, float rexp, int64_t row0 = 0,
                    const int32_t *ids = nullptr);  // ids: global row id per row (compacted graphs)
// Dst[i, :] = d_i^-e Src[i, :]
void scale_copy_block(Ctx &c, const Mat &Src, const Mat &Dst, const int32_t *deg, float rexp);
// Y[i, :] *= d_i^-e
void row_scale_block(Ctx &c, const Mat &Y, const int32_t *deg, float rexp);
// Dst[i, :] = Src[comp[i], :] (0 where comp[i] < 0)
void scatter_rows(Ctx &c, const Mat &Src, const int32_t *comp, const Mat &Dst, int64_t sub = 0);
// Dst[ids[j], :] = Src[j, :] (other Dst rows untouched; Dst may be mapped host memory)
void write_rows(Ctx &c, const Mat &Src, const int32_t *ids, const Mat &Dst);
// copy with ld conversion (device-to-device)
void copy_block(Ctx &c, const float *src, int64_t lds, float *dst, int64_t ldd, int64_t rows,
                int64_t cols);

// ---- small.cu (fp64 small dense, row-major, single-CTA or few-CTA kernels)
// In place upper Cholesky: G = Rᵀ R (R in the upper triangle, lower zeroed).
// On breakdown retries with a diagonal shift (shifted CholeskyQR); increments
// *flag when a shift was needed and sets *flag |= 1<<30 on failure.
void cholesky_upper(Ctx &c, double *G, int64_t l, int64_t ld, int *flag);
// G = RᵀR (l×l, ld) → Rinv = R⁻¹ (l×l upper, ld = l); G is overwritten.
// Shifted retry and *flag protocol as cholesky_upper.
// drop_tol > 0 (orthonormalising passes): a Schur pivot below drop_tol × its
// diagonal marks a numerically dependent column, whose column of R⁻¹ is zero [R10]
void chol_inv_upper(Ctx &c, double *G, int64_t l, int64_t ld, double *Rinv, int *flag, double drop_tol = 0.0);
// the same on nb(nb+1)/2 cooperative CTAs (chol_df.cu), nb = ceil(l/32)
void chol_inv_df(Ctx &c, double *G, int64_t l, int64_t ld, double *Rinv, int *flag, double drop_tol = 0.0);
// Rinv = R^-1 for upper triangular R (l×l)
void tri_inv_upper(Ctx &c, const double *R, int64_t ld, double *Rinv, int64_t l);
// symmetric eigendecomposition (cyclic Jacobi), S overwritten; V (l×l) gets
// eigenvectors as columns, lam the eigenvalues, both sorted by desc |λ| when
// abs_order, else by desc λ.
void sym_eig(Ctx &c, double *S, int64_t l, double *lam, double *V, bool abs_order);
// C = alpha op(A) op(B) + beta C (fp64 small), op = transpose if flag
void gemm64(Ctx &c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
            int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc);
void symmetrize64(Ctx &c, double *S, int64_t l, int64_t ld);
void scale_cols64(Ctx &c, double *A, int64_t rows, int64_t cols, int64_t ld, const double *s, int mode);
void set_identity64(Ctx &c, double *A, int64_t l, int64_t ld);
void axpy64(Ctx &c, int64_t n, double alpha, const double *x, double *y);

// ---- sketch.cu / sketch_tc.cu
// Alg. 3 sparse-sign matrix n×h with z nonzeros per column: column j's entries
// are (rows[j*z + t], signs[j*z + t]), t < z, distinct rows.
struct SparseSign {
  int64_t n = 0, h = 0, z = 0;
  DBuf<int32_t> rows;  // h*z
  DBuf<float> signs;   // h*z (±1)
};
void gen_sparse_sign(Ctx &c, int64_t n, int64_t h, int64_t z, uint64_t seed, uint32_t tag, SparseSign &S);
// Y[n×h] = f(scale · F C F(rows)ᵀ) Ψ  (Eq. 5 sketch), tensor cores
// (F holds this rank's rows [row0, row0 + F.rows); the gathered rows are
// summed over ranks)
// A operand of the fp16-split Y sketch: F split once into hi / lo fp16 planes
// with per-row power-of-two scales (depends on F only, so embed prepares it
// on the side stream while Eq. 3 runs)
struct SketchA {
  int64_t n = 0;
  int k = 0, kp = 0;
  DBuf<uint16_t> hi, lo;  // n × kp fp16 bit patterns
  DBuf<float> rinv;       // per-row 2^-e
  void set_stream(cudaStream_t s) { hi.s = s; lo.s = s; rinv.s = s; }
};
bool sketch_uses_split();  // the fp16-split path is on (NETMFP_SKETCH_F16)
void sketch_split_a(Ctx &c, const Mat &F, SketchA &A);
void tc_sketch_y(Ctx &c, const Mat &F, const double *C, int64_t ldc, const int32_t *rows, const float *signs,
                 int64_t h, int z, float scale, int logmode, const Mat &Y, int64_t row0 = 0,
                 const SketchA *pre = nullptr);
// Zf[h×h] (fp32, ldz) = Πᵀ f(scale · F C Fᵀ restricted to Π's rows) Π  (Alg. 4 step 6)
void tc_sketch_z(Ctx &c, const Mat &F, const double *C, int64_t ldc, const int32_t *rows, const float *signs,
                 int64_t h, int z, float scale, int logmode, float *Zf, int64_t ldz, int64_t row0 = 0);
// Out[h×cols] (fp64) = Ψᵀ X  (sign-gather of rows of X; X fp32 n×cols)
// (X holds rows [row0, row0 + X.rows); rows elsewhere contribute 0)
void sign_gather_T(Ctx &c, const SparseSign &S, const Mat &X, double *Out, int64_t ldo, int64_t row0 = 0);
// fp32 -> fp64 copy of an r×c matrix
void f32_to_f64(Ctx &c, const float *src, int64_t lds, double *dst, int64_t ldd, int64_t rows, int64_t cols);

}  // namespace netmfp
