/*
 * netmfp.h — C ABI of the B200-native NetMF+ hot path (libnetmfp.so).
 *
 * Paper: PAPER.md = arxiv 2110.12782, "NetMF+: Network Embedding Based on
 * Fast and Effective Single-Pass Randomized Matrix Factorization".
 * "PAPER.md:L" cites a line of that text; [R#] cites a reading in DESIGN.md §3.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Return value: NETMFP_OK (0) or an error code below; a human-readable
 *    message for the calling thread is available from netmfp_last_error().
 *    On error, outputs are unspecified; inputs are never modified.
 *  - Dense n×c matrices are fp32, ROW-MAJOR with leading dimension ld
 *    (elements, ld >= c, ld % 4 == 0, base pointer 16-byte aligned).
 *    Element (i, j) is at ptr[i*ld + j].  Small matrices (k×k, d vectors)
 *    are fp64 unless stated.  Padding columns [c, ld) are never written.
 *  - mem = NETMFP_MEM_DEVICE: every pointer argument is device memory on the
 *    context's device; mem = NETMFP_MEM_HOST: every pointer argument is host
 *    memory (pinned or pageable) and the call copies inputs in / outputs out
 *    itself (the end-to-end path).
 *  - All work is enqueued on the context's stream; every call returns only
 *    after that work completed (it synchronises the stream once at the end),
 *    so outputs are ready on return.
 *  - Ownership: the library owns netmfp_ctx and netmfp_graph objects and their
 *    device memory; callers own every buffer they pass in.
 *  - There is no CPU fallback: without a CUDA device every call that computes
 *    returns NETMFP_ERR_CUDA.
 */
#ifndef NETMFP_H
#define NETMFP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NETMFP_OK 0
#define NETMFP_ERR_ARG 1      /* invalid argument (sizes, alignment, ranges)            */
#define NETMFP_ERR_CUDA 2     /* CUDA runtime error / no device                          */
#define NETMFP_ERR_NUMERIC 3  /* e.g. Gram matrix not positive definite after shifting   */
#define NETMFP_ERR_OOM 4      /* device allocation failed                                */
#define NETMFP_ERR_NCCL 5     /* collective failed (multi-GPU)                           */

#define NETMFP_DIST_ID_BYTES 128  /* size of the communicator id (ncclUniqueId) */

#define NETMFP_MEM_DEVICE 0
#define NETMFP_MEM_HOST 1

#define NETMFP_LOG_TRUNC 0    /* trunc_log(x) = max(0, log x), PAPER.md:158  [R4] */
#define NETMFP_LOG_LOG1P 1    /* log1p(max(x, 0)),           PAPER.md:158  [R4] */

typedef struct netmfp_ctx netmfp_ctx;
typedef struct netmfp_graph netmfp_graph;

/* Parameters of Alg. 5 ("Input: ... α; k, s1, q; s2, s3, z; p; d")
 * plus the window T and negative samples b of Eq. 1. */
typedef struct netmfp_params {
  double alpha;        /* modified Laplacian exponent, (0, 0.5]            */
  int32_t k;           /* eigen rank                              (Alg. 2, BASELINE "h")    */
  int32_t s1;          /* eigen oversampling                      (Alg. 2)                  */
  int32_t q;           /* power iterations                        (Alg. 2 steps 4-6)        */
  int32_t T;           /* context window                          (Eq. 1)                   */
  double b;            /* negative samples                        (Eq. 1)                   */
  int32_t d;           /* embedding dimension                                               */
  int32_t s2, s3;      /* sketch oversampling of Psi / Pi         (Alg. 4)                  */
  int32_t z;           /* sparse-sign column sparsity, 2 <= z <= n (Alg. 3)                 */
  int32_t prop_order;  /* Chebyshev order p (0 = no propagation)  (Alg. 5 step 6)          */
  double mu, theta;    /* band-pass kernel of the propagation     [R6]                      */
  uint64_t seed;       /* Philox4x32-10 key for Omega, Psi, Pi    [R1]                      */
  int32_t logmode;     /* NETMFP_LOG_TRUNC or NETMFP_LOG_LOG1P                              */
} netmfp_params;

/* ---- context -------------------------------------------------------------- */

/* Create a context on CUDA device `device`, enqueueing on `stream`
 * (a cudaStream_t owned by the caller; NULL = the legacy default stream). */
int netmfp_ctx_create(int device, void *stream, netmfp_ctx **out);
int netmfp_ctx_destroy(netmfp_ctx *ctx);
/* Number of kernels this context launched since creation (launch accounting). */
int64_t netmfp_ctx_launches(const netmfp_ctx *ctx);
/* Per-kernel timing with CUDA events recorded around every launch whose
 * kernel name starts with one of the comma-separated prefixes in `filter`
 * (NULL or "" = all kernels).  enable = 0 turns it off and clears the stats. */
int netmfp_ctx_profile(netmfp_ctx *ctx, int enable, const char *filter);
/* Write "name count total_ms\n" lines of the intervals collected since the
 * last read into buf (NUL-terminated) and reset the statistics. */
int netmfp_ctx_profile_read(netmfp_ctx *ctx, char *buf, size_t len);
const char *netmfp_last_error(void);
const char *netmfp_version(void);

/* ---- a1: graph ------------------------------------------------------------- */

/* Build the CSR of the undirected simple graph G = (V, E, A) (PAPER.md:124,
 * :151): the m_in input pairs (src[e], dst[e]), 0 <= src,dst < n, are
 * symmetrised, self-loops dropped, duplicates collapsed (A is 0/1), neighbour
 * lists sorted ascending.  Isolated vertices are kept with degree 0 [R2].
 * Result: rowptr int64[n+1], col int32[nnz], deg int32[n], vol(G) = nnz = 2m.
 * n < 2^31.  src/dst in `mem`.  *out is owned by the library (netmfp_graph_free). */
int netmfp_build_csr(netmfp_ctx *ctx, int64_t n, const int32_t *src, const int32_t *dst,
                     int64_t m_in, int mem, netmfp_graph **out);
/* n, nnz (= vol(G)), number of heavy rows (degree > the light-kernel cap). */
int netmfp_graph_info(const netmfp_graph *g, int64_t *n, int64_t *nnz, int64_t *n_heavy);
/* Copy the CSR out (any pointer may be NULL to skip it). */
int netmfp_graph_export(netmfp_ctx *ctx, const netmfp_graph *g, int64_t *rowptr, int32_t *col,
                        int32_t *deg, int mem);
int netmfp_graph_free(netmfp_graph *g);
/* Split rows into `parts` contiguous ranges of near-equal nnz + rows cost
 * (north_star: "the CSR is row-partitioned"); bounds int64[parts+1], host. */
int netmfp_partition_rows(const int64_t *rowptr_host, int64_t n, int32_t parts, int64_t *bounds);

/* ---- multi-GPU: row-partitioned CSR (north_star) ------------------------------
 * One process per GPU.  Rank r owns rows [bounds[r], bounds[r+1]) of the graph
 * and of every n×c block; each SpMM all-gathers its input block (NCCL
 * broadcasts from every rank into one n×c buffer, over NVLink), Gram
 * matrices and the sketch's gathered rows are all-reduced, the small fp64
 * problems are replicated, and Ω, Ψ, Π are counter-based (every rank draws its
 * own rows).  With one rank (the default) no collective is issued.  NCCL is
 * loaded at run time (libnccl.so.2); failures return NETMFP_ERR_NCCL. */
/* Write a fresh communicator id (NETMFP_DIST_ID_BYTES bytes, host) on one rank. */
int netmfp_dist_unique_id(void *id);
/* Join the communicator (collective over all ranks; the context's device). */
int netmfp_dist_init(netmfp_ctx *ctx, const void *id, int32_t nranks, int32_t rank);
/* Host-staged communicator (instead of NCCL): the library synchronises its
 * stream, copies the operand to host memory, calls the callback and copies
 * the result back.  Callbacks return 0 on success (else NETMFP_ERR_NCCL is
 * reported) and must be collective over all ranks in call order, like the
 * NCCL calls they replace:
 *   allreduce_sum(user, buf, count, dtype): buf[0..count) = Σ_ranks buf, in place;
 *   broadcast(user, buf, count, dtype, root): buf[0..count) = root's buf.
 * dtype: NETMFP_DT_F32 / _F64 / _I64 / _I32 / _U8.  Used to execute the
 * multi-rank schedule where NCCL cannot run (several ranks on one GPU in
 * tests, CPU-side process groups); the NVLink path is netmfp_dist_init. */
#define NETMFP_DT_F32 0
#define NETMFP_DT_F64 1
#define NETMFP_DT_I64 2
#define NETMFP_DT_I32 3
#define NETMFP_DT_U8 4
typedef struct netmfp_comm_ops {
  void *user;
  int (*allreduce_sum)(void *user, void *buf, int64_t count, int32_t dtype);
  int (*broadcast)(void *user, void *buf, int64_t count, int32_t dtype, int32_t root);
} netmfp_comm_ops;
int netmfp_dist_init_ops(netmfp_ctx *ctx, const netmfp_comm_ops *ops, int32_t nranks, int32_t rank);
/* Bytes this rank received in collectives since the last call (all-gathers:
 * the other ranks' rows; all-reduces: the reduced payload), and how many
 * collectives were issued; both counters are reset. */
int netmfp_dist_stats(netmfp_ctx *ctx, int64_t *bytes, int64_t *collectives);
/* Build this rank's CSR rows [bounds[rank], bounds[rank+1]) (bounds: nranks+1
 * host int64, strictly increasing from 0 to n — every rank owns >= 1 row; NULL = equal row counts; netmfp_partition_rows gives an
 * nnz-balanced split) with global column ids.  src/dst must contain every
 * (undirected) edge incident to those rows (the full list is fine: only the
 * rank's own edges are sorted, so device memory is O(m/nranks) beyond the
 * input).  Collective (vol(G) is all-reduced).  Then netmfp_embed /
 * netmfp_eig / netmfp_propagate on this graph take and return this rank's rows
 * of every n×c block; netmfp_embed drops isolated vertices from the blocks
 * (every rank learns all degrees by one all-gather) and returns
 * zero rows for them [R2]. */
int netmfp_dist_build_csr(netmfp_ctx *ctx, int64_t n, const int32_t *src, const int32_t *dst, int64_t m_in,
                          const int64_t *bounds, int mem, netmfp_graph **out);
/* CSR of rows [row0, row1) only (global column ids; no communicator; vol(G)
 * reported is the local nnz).  netmfp_spmm on such a graph takes the FULL n×c
 * input block and writes the row1−row0 output rows — one rank's SpMM. */
int netmfp_build_csr_rows(netmfp_ctx *ctx, int64_t n, const int32_t *src, const int32_t *dst, int64_t m_in,
                          int64_t row0, int64_t row1, int mem, netmfp_graph **out);
/* First global row, n, vol(G) of a (possibly partitioned) graph. */
int netmfp_graph_rows(const netmfp_graph *g, int64_t *row0, int64_t *n_global, int64_t *nnz_global);

/* ---- a2: the normalized SpMM (the hot operator) --------------------------- */

/* Y = D^-a A D^-b X on cols columns (PAPER.md:217 modified Laplacian: a = b = α;
 * PAPER.md:171 D^-1 A: a = 1, b = 0), d^e := 0 for d = 0 [R2]. */
int netmfp_spmm(netmfp_ctx *ctx, const netmfp_graph *g, double a, double b, const float *X,
                int64_t ldx, float *Y, int64_t ldy, int64_t cols, int mem);

/* ---- dense steps of Alg. 2 / Alg. 4 (exposed for step-wise parity) ---------- */

/* Omega = randn(n, l) of Alg. 2 step 2: entries (i, 4q..4q+3)
 * from Philox4x32-10 on counter (q, i mod 2^32, i >> 32, tag Omega) with key
 * (seed mod 2^32, seed >> 32) and Box-Muller on both word pairs [R1] -- the
 * draw netmfp_eig / netmfp_embed use (before their degree row scale).
 * Omega: n×l fp32, row-major, ld >= l (device: ld % 4 == 0, 16-B aligned),
 * caller-owned.  Errors: NETMFP_ERR_ARG for l < 1, n < 0 or ld < l. */
int netmfp_gaussian(netmfp_ctx *ctx, int64_t n, int64_t l, uint64_t seed, float *Omega, int64_t ld, int mem);

/* G = Aᵀ B over the n rows (fp64 result, row-major a×b).  A: n×a fp32 (lda),
 * B: n×b fp32 (ldb).  The Gram matrix of eigSVD/CholeskyQR. */
int netmfp_gram(netmfp_ctx *ctx, int64_t n, const float *A, int64_t lda, int64_t a, const float *B,
                int64_t ldb, int64_t b, double *G, int mem);
/* Q = orth(Y): CholeskyQR (passes = 1) or CholeskyQR2 (passes = 2), the
 * "orth"/"eigSVD" step of Alg. 2 steps 3, 5 and Alg. 4 step 4 [R7].
 * Y, Q: n×c fp32 (ldy, ldq); requires n >= c.  An exactly-zero column of Y
 * gives a zero column of Q; with passes >= 2 a numerically dependent column
 * (Schur pivot below 1e-8 of its diagonal in the second pass) does too, so Q
 * spans range(Y) [R10].  NETMFP_ERR_NUMERIC if the factorisation still fails
 * after shifted retries. */
int netmfp_orthonormalize(netmfp_ctx *ctx, int64_t n, int64_t c, const float *Y, int64_t ldy, float *Q,
                          int64_t ldq, int32_t passes, int mem);
/* [V, Λ] = eig(S) of a symmetric l×l fp64 matrix (row-major): Alg. 2 step 8,
 * and svd(S) of the symmetric core in Alg. 4 step 8.  lam: l eigenvalues
 * ordered by descending |λ| (abs_order = 1, [R3]) or descending λ; V: l×l,
 * column j = unit eigenvector of lam[j].  l <= 460. */
int netmfp_sym_eig(netmfp_ctx *ctx, const double *S, int64_t l, double *lam, double *V, int32_t abs_order,
                   int mem);

/* ---- a3: Alg. 2 freigs ------------------------------------------------------ */

/* [U_k, Λ_k] = freigs(D^-α A D^-α, k, s1, q): Ω = randn(n,
 * k+s1) from Philox(seed) [R1], q power iterations, Rayleigh–Ritz, eigenpairs
 * ordered by descending |λ| [R3].  U: n×k fp32 (ldu), lambda: k fp64.
 * Requires k + s1 <= n.  Orthonormalisation by CholeskyQR [R7]. */
int netmfp_eig(netmfp_ctx *ctx, const netmfp_graph *g, double alpha, int32_t k, int32_t s1,
               int32_t q, uint64_t seed, float *U, int64_t ldu, double *lambda, int mem);

/* ---- a4: Eq. 3 factor pair -------------------------------------------------- */

/* K = Uᵀ D^(-1+2α) U Λ, F = D^(-1+α) U, C = Λ Σ_{r=1}^T K^(r-1) (PAPER.md:233-235,
 * Alg. 5 steps 2-3).  U: n×k fp32 (ldu); lambda: k fp64; F: n×k fp32 (ldf);
 * C: k×k fp64 row-major. */
int netmfp_factor_pair(netmfp_ctx *ctx, const netmfp_graph *g, double alpha, int32_t T,
                       const float *U, int64_t ldu, const double *lambda, int32_t k, float *F,
                       int64_t ldf, double *C, int mem);

/* ---- a5-a7: Alg. 4 sparse-sign randomized single-pass SVD ------------------- */

/* [U, Σ, ~] = sparse_sign_rand_single_pass_SVD(F, C, d, s2, s3, z) of
 * M̂' = f(scale · F C Fᵀ), scale = vol(G)/(bT) (Eq. 4-5):
 * Y = f(scale F C F(p,:)ᵀ)Ψ (Eq. 5), Q = orth(Y), Z = Πᵀ f(scale F(p,:) C F(p,:)ᵀ) Π,
 * S = (ΠᵀQ)† Z (QᵀΠ)†, svd(S).  F: n×k fp32 (ldf); C: k×k fp64.
 * Outputs (any may be NULL): U n×d fp32 (ldu), sigma d fp64, and the raw
 * embedding E = U √Σ (Alg. 5 step 5) n×d fp32 (lde).  orth(Y) spans range(Y)
 * (zero / dependent columns of Y are dropped [R10]); when rank(Y) < d the
 * trailing singular values are zero.
 * Optional sketch outputs for parity tests (NULL to skip): Ysk n×(d+s2) fp32
 * (ldy) and Zsk (d+s3)×(d+s3) fp64. */
int netmfp_sketch_svd(netmfp_ctx *ctx, int64_t n, const float *F, int64_t ldf, const double *C,
                      int32_t k, double scale, int32_t d, int32_t s2, int32_t s3, int32_t z,
                      uint64_t seed, int32_t logmode, float *U, int64_t ldu, double *sigma,
                      float *E, int64_t lde, float *Ysk, int64_t ldy, double *Zsk, int mem);

/* ---- a8: spectral propagation ----------------------------------------------- */

/* E <- Σ_{r=0}^{p} c_r T_r(L - I) E, L = I - D^-1 A (Alg. 5 step 6),
 * c_r = Chebyshev coefficients of the band-pass kernel [R6], evaluated by
 * Clenshaw's recurrence (p SpMMs).  In place on E n×d fp32 (lde).  p = 0
 * leaves E unchanged. */
int netmfp_propagate(netmfp_ctx *ctx, const netmfp_graph *g, float *E, int64_t lde, int32_t d,
                     int32_t order, double mu, double theta, int mem);
/* The c_0..c_order used by netmfp_propagate (host output, order+1 doubles). */
int netmfp_cheb_coeffs(int32_t order, double mu, double theta, double *c);

/* ---- Alg. 5 end to end -------------------------------------------------------- */

/* E = NetMF+(G) on a built graph: freigs → K, F, C →
 * single-pass SVD → E = U√Σ → propagation.  E: n×d fp32 (lde); sigma (d fp64)
 * and lambda (k fp64) optional (NULL).  `mem` applies to E, sigma, lambda.
 * Isolated vertices are dropped from the computation (their rows of E are 0).
 * With mem = HOST and E in pinned (page-locked, mapped) memory the device
 * writes E's non-isolated rows directly while host threads zero the rest. */
int netmfp_embed(netmfp_ctx *ctx, const netmfp_graph *g, const netmfp_params *p, float *E,
                 int64_t lde, double *sigma, double *lambda, int mem);

/* Alg. 5 from an edge list: netmfp_build_csr + netmfp_embed in one call
 * (src/dst/E in `mem`; with NETMFP_MEM_HOST this is the end-to-end path). */
int netmfp_embed_edges(netmfp_ctx *ctx, int64_t n, const int32_t *src, const int32_t *dst,
                       int64_t m_in, const netmfp_params *p, float *E, int64_t lde,
                       double *sigma, int mem);

#ifdef __cplusplus
}
#endif
#endif /* NETMFP_H */
