// api.cu — the C ABI of include/netmfp.h: argument checking, host/device
// marshalling, error codes.  All compute is in the other translation units.
#include <algorithm>
#include <chrono>
#include <exception>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "pipeline.cuh"

struct netmfp_ctx {
  netmfp::Ctx c;
};
struct netmfp_graph {
  netmfp::Graph *g;
};

namespace netmfp {

static thread_local std::string g_last_error;
void set_last_error(const std::string &m) { g_last_error = m; }

template <class F>
static int guarded(F &&f) {
  try {
    f();
    set_last_error("");
    return NETMFP_OK;
  } catch (const Error &e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return NETMFP_ERR_CUDA;
  }
}

// Wrap a caller n×cols fp32 matrix: device pointers are used in place; host
// pointers are staged through a padded device block.
struct InMat {
  Block staged;
  Mat m;
  InMat(Ctx &c, const float *p, int64_t rows, int64_t cols, int64_t ld, int mem, bool copy_in) {
    NM_REQUIRE(ld >= cols && cols > 0, "matrix: need ld >= cols > 0");
    if (mem == NETMFP_MEM_DEVICE) {
      NM_REQUIRE(ld % 4 == 0 && ((uintptr_t)p & 15) == 0,
                 "device matrix: ld % 4 == 0 and 16-byte aligned base required");
      m.p = const_cast<float *>(p);
      m.rows = rows;
      m.cols = cols;
      m.ld = ld;
    } else {
      staged.alloc(rows, cols, c.stream);
      m = staged.m;
      if (copy_in)
        NM_CUDA(cudaMemcpy2DAsync(m.p, m.ld * 4, p, ld * 4, cols * 4, rows, cudaMemcpyHostToDevice, c.stream));
    }
  }
  void copy_out(Ctx &c, float *p, int64_t ld, int mem) {
    if (mem == NETMFP_MEM_HOST)
      NM_CUDA(cudaMemcpy2DAsync(p, ld * 4, m.p, m.ld * 4, m.cols * 4, m.rows, cudaMemcpyDeviceToHost, c.stream));
  }
};

template <class T>
struct InVec {
  DBuf<T> staged;
  T *p = nullptr;
  InVec(Ctx &c, const T *src, int64_t n, int mem, bool copy_in) {
    if (mem == NETMFP_MEM_DEVICE || !src) {
      p = const_cast<T *>(src);
    } else {
      staged.alloc(n, c.stream);
      p = staged.p;
      if (copy_in) NM_CUDA(cudaMemcpyAsync(p, src, n * sizeof(T), cudaMemcpyHostToDevice, c.stream));
    }
  }
  void copy_out(Ctx &c, T *dst, int64_t n, int mem) {
    if (mem == NETMFP_MEM_HOST && dst)
      NM_CUDA(cudaMemcpyAsync(dst, p, n * sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  }
};

static void check_mem(int mem) {
  NM_REQUIRE(mem == NETMFP_MEM_DEVICE || mem == NETMFP_MEM_HOST, "mem must be NETMFP_MEM_DEVICE or _HOST");
}

// Every entry point runs on its context's device (the caller's current
// device is restored on return).  If the call throws, pending deferred numeric
// checks and the device status flags are dropped so that the next call does
// not report this call's failure.
struct DevScope {
  Ctx &c;
  int prev = -1;
  int unwinding0;
  explicit DevScope(Ctx &cc) : c(cc), unwinding0(std::uncaught_exceptions()) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != c.device) NM_CUDA(cudaSetDevice(c.device));
  }
  ~DevScope() {
    if (std::uncaught_exceptions() > unwinding0) {
      if (c.side) cudaStreamSynchronize(c.side);  // side-stream work may still use freed buffers
      cudaStreamSynchronize(c.stream);
      cudaGetLastError();
      c.flag_checks.clear();
      if (c.d_flags) cudaMemsetAsync(c.d_flags, 0, 16, c.stream);
      cudaStreamSynchronize(c.stream);
      c.pending.clear();
    }
    if (prev >= 0 && prev != c.device) cudaSetDevice(prev);
  }
  DevScope(const DevScope &) = delete;
  DevScope &operator=(const DevScope &) = delete;
};

// All netmfp_params fields, checked before any work is queued (Alg. 5's
// inputs; the stages re-check what they use).
static void check_params(const netmfp_params &p, int64_t n) {
  NM_REQUIRE(p.alpha > 0.0 && p.alpha <= 0.5, "params: alpha in (0, 0.5] (PAPER.md:217)");
  NM_REQUIRE(p.k >= 1 && p.s1 >= 0 && p.q >= 0, "params: need k >= 1, s1 >= 0, q >= 0");
  NM_REQUIRE((int64_t)p.k + p.s1 <= n, "params: k + s1 must not exceed n (Alg. 2)");
  NM_REQUIRE(p.T >= 1 && p.b > 0.0, "params: need T >= 1, b > 0 (Eq. 1)");
  NM_REQUIRE(p.d >= 1 && p.s2 >= 0 && p.s3 >= p.s2, "params: need d >= 1, 0 <= s2 <= s3 (PAPER.md:413)");
  NM_REQUIRE((int64_t)p.d + p.s2 <= n, "params: d + s2 must not exceed n (Alg. 4)");
  NM_REQUIRE(p.z >= 2 && p.z <= 64 && p.z <= n, "params: need 2 <= z <= min(n, 64) (Alg. 3)");
  NM_REQUIRE(p.prop_order >= 0 && p.prop_order <= 64, "params: prop_order in [0, 64]");
  NM_REQUIRE(p.logmode == NETMFP_LOG_TRUNC || p.logmode == NETMFP_LOG_LOG1P, "params: bad logmode");
}

static void finish(Ctx &c) {
  static const bool dbg = getenv("NETMFP_DEBUG_ENQUEUE") != nullptr;
  if (dbg) {  // host time to enqueue the call vs its device time (is the host the bottleneck?)
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c.stream);
    const auto t0 = std::chrono::steady_clock::now();
    cudaEventSynchronize(e);
    const double wait_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "netmfp: host waited %.3f ms for the device after enqueueing\n", wait_ms);
    cudaEventDestroy(e);
  }
  int h = 0;
  if (!c.flag_checks.empty())
    NM_CUDA(cudaMemcpyAsync(&h, c.d_flags, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  NM_CUDA(cudaStreamSynchronize(c.stream));
  prof_collect(c);
  if (!c.flag_checks.empty()) {
    const std::string what = c.flag_checks.front();
    c.flag_checks.clear();
    if (h & (1 << 30)) {
      NM_CUDA(cudaMemset(c.d_flags, 0, sizeof(int)));
      throw Error(NETMFP_ERR_NUMERIC, what +
                                          ": Gram matrix not positive definite even after shifting "
                                          "(input not of full column rank, PAPER.md:215)");
    }
  }
}

}  // namespace netmfp

using namespace netmfp;

extern "C" {

const char *netmfp_last_error(void) { return g_last_error.c_str(); }
const char *netmfp_version(void) { return "netmfp 0.1 (sm_100a)"; }

int netmfp_ctx_create(int device, void *stream, netmfp_ctx **out) {
  return guarded([&] {
    NM_REQUIRE(out, "ctx_create: out is NULL");
    int ndev = 0;
    NM_CUDA(cudaGetDeviceCount(&ndev));
    NM_REQUIRE(device >= 0 && device < ndev, "ctx_create: no such CUDA device");
    NM_CUDA(cudaSetDevice(device));
    auto *x = new netmfp_ctx();
    x->c.device = device;
    cudaDeviceProp prop;
    NM_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
      delete x;
      throw Error(NETMFP_ERR_CUDA, "ctx_create: libnetmfp is built for sm_100a (B200) only");
    }
    x->c.num_sms = prop.multiProcessorCount;
    x->c.stream = (cudaStream_t)stream;  // NULL = the legacy default stream
    NM_CUDA(cudaMalloc(&x->c.d_flags, 16));
    NM_CUDA(cudaMemsetAsync(x->c.d_flags, 0, 16, x->c.stream));
    // keep freed pool memory cached (stream-ordered allocator)
    cudaMemPool_t pool;
    NM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    NM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // reserve working memory up front (NETMFP_POOL_RESERVE_GB, default 24 GiB or
    // half the free memory) so that steps never grow the pool mid-stream
    {
      size_t fr = 0, tot = 0;
      NM_CUDA(cudaMemGetInfo(&fr, &tot));
      const char *ev = getenv("NETMFP_POOL_RESERVE_GB");
      size_t want = (size_t)(ev ? atof(ev) : 24.0) << 30;
      want = std::min(want, fr / 2);
      if (want > 0) {
        void *tmp = nullptr;
        if (cudaMallocAsync(&tmp, want, x->c.stream) == cudaSuccess) cudaFreeAsync(tmp, x->c.stream);
        cudaGetLastError();
        NM_CUDA(cudaStreamSynchronize(x->c.stream));
      }
    }
    *out = x;
  });
}

int netmfp_ctx_destroy(netmfp_ctx *ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->c.d_flags) cudaFree(ctx->c.d_flags);
    ctx->c.spmm_part.release();  // stream-ordered frees before the stream goes
    ctx->c.spmm_cnt.release();
    cudaStreamSynchronize(ctx->c.stream);
    try {
      dist_destroy(ctx->c);
    } catch (...) {
    }
    if (ctx->c.side) {
      cudaStreamSynchronize(ctx->c.side);
      cudaStreamDestroy(ctx->c.side);
      cudaEventDestroy(ctx->c.ev_fork);
      cudaEventDestroy(ctx->c.ev_join);
    }
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
    delete ctx;
  });
}

int64_t netmfp_ctx_launches(const netmfp_ctx *ctx) { return ctx ? ctx->c.launches : -1; }

int netmfp_ctx_profile(netmfp_ctx *ctx, int enable, const char *filter) {
  return guarded([&] {
    NM_REQUIRE(ctx, "ctx_profile: NULL ctx");
    ctx->c.prof = enable != 0;
    ctx->c.prof_filter = filter ? filter : "";
    if (!enable) ctx->c.stats.clear();
  });
}

int netmfp_ctx_profile_read(netmfp_ctx *ctx, char *buf, size_t len) {
  return guarded([&] {
    NM_REQUIRE(ctx && buf && len > 0, "ctx_profile_read: bad arguments");
    DevScope _dev(ctx->c);
    NM_CUDA(cudaStreamSynchronize(ctx->c.stream));
    prof_collect(ctx->c);
    std::string out;
    for (auto &s : ctx->c.stats)
      out += s.first + " " + std::to_string(s.second.first) + " " + std::to_string(s.second.second) + "\n";
    NM_REQUIRE(out.size() < len, "ctx_profile_read: buffer too small");
    std::memcpy(buf, out.c_str(), out.size() + 1);
    ctx->c.stats.clear();
  });
}

int netmfp_build_csr(netmfp_ctx *ctx, int64_t n, const int32_t *src, const int32_t *dst, int64_t m_in,
                     int mem, netmfp_graph **out) {
  return guarded([&] {
    NM_REQUIRE(ctx && out, "build_csr: NULL ctx/out");
    check_mem(mem);
    NM_REQUIRE(m_in == 0 || (src && dst), "build_csr: NULL edge arrays");
    Ctx &c = ctx->c;
    DevScope _dev(c);
    InVec<int32_t> s(c, src, m_in, mem, true), t(c, dst, m_in, mem, true);
    Graph *g = build_csr_device(c, n, s.p, t.p, m_in);
    finish(c);
    *out = new netmfp_graph{g};
  });
}

int netmfp_dist_unique_id(void *id) {
  return guarded([&] {
    NM_REQUIRE(id, "dist_unique_id: NULL");
    dist_unique_id(id);
  });
}

int netmfp_dist_init(netmfp_ctx *ctx, const void *id, int32_t nranks, int32_t rank) {
  return guarded([&] {
    NM_REQUIRE(ctx && (id || nranks == 1), "dist_init: NULL argument");
    DevScope _dev(ctx->c);
    dist_init(ctx->c, id, nranks, rank);
  });
}

int netmfp_dist_init_ops(netmfp_ctx *ctx, const netmfp_comm_ops *ops, int32_t nranks, int32_t rank) {
  return guarded([&] {
    NM_REQUIRE(ctx && ops, "dist_init_ops: NULL argument");
    DevScope _dev(ctx->c);
    dist_init_ops(ctx->c, *ops, nranks, rank);
  });
}

int netmfp_dist_stats(netmfp_ctx *ctx, int64_t *bytes, int64_t *collectives) {
  return guarded([&] {
    NM_REQUIRE(ctx, "dist_stats: NULL ctx");
    if (bytes) *bytes = ctx->c.comm_bytes;
    if (collectives) *collectives = ctx->c.collectives;
    ctx->c.comm_bytes = 0;
    ctx->c.collectives = 0;
  });
}

int netmfp_dist_build_csr(netmfp_ctx *ctx, int64_t n, const int32_t *src, const int32_t *dst, int64_t m_in,
                          const int64_t *bounds, int mem, netmfp_graph **out) {
  return guarded([&] {
    NM_REQUIRE(ctx && out, "dist_build_csr: NULL ctx/out");
    check_mem(mem);
    NM_REQUIRE(m_in == 0 || (src && dst), "dist_build_csr: NULL edge arrays");
    Ctx &c = ctx->c;
    DevScope _dev(c);
    std::vector<int64_t> b(c.nranks + 1);
    for (int r = 0; r <= c.nranks; ++r) b[r] = bounds ? bounds[r] : n * r / c.nranks;
    NM_REQUIRE(b[0] == 0 && b[c.nranks] == n, "dist_build_csr: bounds must start at 0 and end at n");
    for (int r = 0; r < c.nranks; ++r) NM_REQUIRE(b[r] < b[r + 1], "dist_build_csr: every rank needs >= 1 row (bounds strictly increasing)");
    InVec<int32_t> s(c, src, m_in, mem, true), t(c, dst, m_in, mem, true);
    std::unique_ptr<Graph> g(build_csr_device(c, n, s.p, t.p, m_in, b[c.rank], b[c.rank + 1]));
    g->bounds = b;
    // vol(G) = Σ_ranks local nnz
    DBuf<int64_t> v(1, c.stream);
    NM_CUDA(cudaMemcpyAsync(v.p, &g->nnz, 8, cudaMemcpyHostToDevice, c.stream));
    dist_allreduce(c, v.p, 1, DType::I64);
    NM_CUDA(cudaMemcpyAsync(&g->nnz_global, v.p, 8, cudaMemcpyDeviceToHost, c.stream));
    finish(c);
    *out = new netmfp_graph{g.release()};
  });
}

int netmfp_build_csr_rows(netmfp_ctx *ctx, int64_t n, const int32_t *src, const int32_t *dst, int64_t m_in,
                          int64_t row0, int64_t row1, int mem, netmfp_graph **out) {
  return guarded([&] {
    NM_REQUIRE(ctx && out, "build_csr_rows: NULL ctx/out");
    check_mem(mem);
    NM_REQUIRE(m_in == 0 || (src && dst), "build_csr_rows: NULL edge arrays");
    Ctx &c = ctx->c;
    DevScope _dev(c);
    InVec<int32_t> s(c, src, m_in, mem, true), t(c, dst, m_in, mem, true);
    Graph *g = build_csr_device(c, n, s.p, t.p, m_in, row0, row1);
    finish(c);
    *out = new netmfp_graph{g};
  });
}

int netmfp_graph_rows(const netmfp_graph *g, int64_t *row0, int64_t *n_global, int64_t *nnz_global) {
  return guarded([&] {
    NM_REQUIRE(g, "graph_rows: NULL graph");
    if (row0) *row0 = g->g->row0;
    if (n_global) *n_global = g->g->n_global;
    if (nnz_global) *nnz_global = g->g->nnz_global;
  });
}

int netmfp_graph_info(const netmfp_graph *g, int64_t *n, int64_t *nnz, int64_t *n_heavy) {
  return guarded([&] {
    NM_REQUIRE(g, "graph_info: NULL graph");
    if (n) *n = g->g->n;
    if (nnz) *nnz = g->g->nnz;
    if (n_heavy) *n_heavy = g->g->n_heavy;
  });
}

int netmfp_graph_export(netmfp_ctx *ctx, const netmfp_graph *gr, int64_t *rowptr, int32_t *col,
                        int32_t *deg, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && gr, "graph_export: NULL");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    const Graph &g = *gr->g;
    auto kind = mem == NETMFP_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (rowptr) NM_CUDA(cudaMemcpyAsync(rowptr, g.rowptr.p, (g.n + 1) * 8, kind, c.stream));
    if (col && g.nnz) NM_CUDA(cudaMemcpyAsync(col, g.col.p, g.nnz * 4, kind, c.stream));
    if (deg) NM_CUDA(cudaMemcpyAsync(deg, g.deg.p, g.n * 4, kind, c.stream));
    finish(c);
  });
}

int netmfp_graph_free(netmfp_graph *g) {
  return guarded([&] {
    if (!g) return;
    // free on the legacy default stream: the creating context (and its
    // stream) may already be gone
    Graph *gg = g->g;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(gg->device);
    gg->detach_streams();
    delete gg;
    delete g;
    if (prev >= 0) cudaSetDevice(prev);
  });
}

int netmfp_partition_rows(const int64_t *rowptr, int64_t n, int32_t parts, int64_t *bounds) {
  return guarded([&] {
    NM_REQUIRE(rowptr && bounds && parts >= 1 && n >= 0, "partition_rows: bad arguments");
    // cost(row) = nnz + 1 (the gather work plus the row's output write);
    // bounds[r] = first row whose prefix cost reaches r/parts of the total.
    const int64_t total = rowptr[n] + n;
    bounds[0] = 0;
    int64_t row = 0;
    for (int32_t r = 1; r < parts; ++r) {
      const long double target = (long double)total * r / parts;
      while (row < n && (long double)(rowptr[row] + row) < target) ++row;
      bounds[r] = row;
    }
    bounds[parts] = n;
  });
}

int netmfp_spmm(netmfp_ctx *ctx, const netmfp_graph *gr, double a, double b, const float *X, int64_t ldx,
                float *Y, int64_t ldy, int64_t cols, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && gr && X && Y, "spmm: NULL argument");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    const Graph &g = *gr->g;
    // X: all n_global rows (the columns of A); Y: this graph's rows
    InMat xi(c, X, g.n_global, cols, ldx, mem, true), yo(c, Y, g.n, cols, ldy, mem, false);
    NM_REQUIRE(b == 0.0 || g.n == g.n_global, "spmm: column scaling (b != 0) needs the unpartitioned graph");
    DBuf<float> scol;
    SpmmArgs p;
    p.X = xi.m.p; p.ldx = xi.m.ld; p.Y = yo.m.p; p.ldy = yo.m.ld; p.cols = cols; p.a = (float)a;
    if (b != 0.0) {
      scol.alloc(g.n, c.stream);
      deg_pow(c, g, (float)b, scol.p);
      p.s_col = scol.p;
    }
    spmm(c, g, p);
    yo.copy_out(c, Y, ldy, mem);
    finish(c);
  });
}

int netmfp_gaussian(netmfp_ctx *ctx, int64_t n, int64_t l, uint64_t seed, float *Omega, int64_t ld, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && Omega, "gaussian: NULL argument");
    NM_REQUIRE(n >= 0 && l >= 1 && ld >= l, "gaussian: need n >= 0, l >= 1, ld >= l");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    if (n == 0) return;
    InMat out(c, Omega, n, l, ld, mem, false);
    gaussian_block(c, out.m, seed, nullptr, 0.f, 0, nullptr);  // Alg. 2 step 2, no row scale
    out.copy_out(c, Omega, ld, mem);
    finish(c);
  });
}

int netmfp_gram(netmfp_ctx *ctx, int64_t n, const float *A, int64_t lda, int64_t a, const float *B,
                int64_t ldb, int64_t b, double *G, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && A && B && G, "gram: NULL argument");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    InMat ai(c, A, n, a, lda, mem, true);
    std::unique_ptr<InMat> bi;
    Mat bm = ai.m;
    if (B != A || b != a || ldb != lda) {
      bi.reset(new InMat(c, B, n, b, ldb, mem, true));
      bm = bi->m;
    }
    InVec<double> go(c, G, a * b, mem, false);
    gram(c, ai.m, bm, nullptr, 0.f, go.p, b);
    go.copy_out(c, G, a * b, mem);
    finish(c);
  });
}

int netmfp_orthonormalize(netmfp_ctx *ctx, int64_t n, int64_t cc, const float *Y, int64_t ldy, float *Q,
                          int64_t ldq, int32_t passes, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && Y && Q && passes >= 1 && passes <= 3 && n >= cc, "orthonormalize: bad arguments");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    InMat yi(c, Y, n, cc, ldy, mem, true), qo(c, Q, n, cc, ldq, mem, false);
    Block tmp(n, cc, c.stream);
    cholqr(c, yi.m, qo.m, nullptr, 0.f, passes, &tmp.m);
    NM_CUDA(cudaStreamSynchronize(c.stream));
    int h = 0;
    NM_CUDA(cudaMemcpy(&h, c.d_flags, sizeof(int), cudaMemcpyDeviceToHost));
    if (h & (1 << 30)) {
      NM_CUDA(cudaMemset(c.d_flags, 0, sizeof(int)));
      throw Error(NETMFP_ERR_NUMERIC, "orthonormalize: Y not of full column rank");
    }
    qo.copy_out(c, Q, ldq, mem);
    finish(c);
  });
}

int netmfp_sym_eig(netmfp_ctx *ctx, const double *S, int64_t l, double *lam, double *V, int32_t abs_order,
                   int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && S && lam && V && l >= 1, "sym_eig: bad arguments");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    InVec<double> si(c, S, l * l, mem, true), lo(c, lam, l, mem, false), vo(c, V, l * l, mem, false);
    DBuf<double> work(l * l, c.stream);  // sym_eig overwrites its input
    NM_CUDA(cudaMemcpyAsync(work.p, si.p, l * l * 8, cudaMemcpyDeviceToDevice, c.stream));
    sym_eig(c, work, l, lo.p, vo.p, abs_order != 0);
    lo.copy_out(c, lam, l, mem);
    vo.copy_out(c, V, l * l, mem);
    finish(c);
  });
}

int netmfp_eig(netmfp_ctx *ctx, const netmfp_graph *gr, double alpha, int32_t k, int32_t s1, int32_t q,
               uint64_t seed, float *U, int64_t ldu, double *lambda, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && gr && U && lambda, "eig: NULL argument");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    const Graph &g = *gr->g;
    InMat uo(c, U, g.n, k, ldu, mem, false);
    InVec<double> lo(c, lambda, k, mem, false);
    freigs(c, g, alpha, k, s1, q, seed, uo.m, lo.p);
    uo.copy_out(c, U, ldu, mem);
    lo.copy_out(c, lambda, k, mem);
    finish(c);
  });
}

int netmfp_factor_pair(netmfp_ctx *ctx, const netmfp_graph *gr, double alpha, int32_t T, const float *U,
                       int64_t ldu, const double *lambda, int32_t k, float *F, int64_t ldf, double *C,
                       int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && gr && U && lambda && F && C, "factor_pair: NULL argument");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    const Graph &g = *gr->g;
    InMat ui(c, U, g.n, k, ldu, mem, true), fo(c, F, g.n, k, ldf, mem, false);
    InVec<double> li(c, lambda, k, mem, true), co(c, C, (int64_t)k * k, mem, false);
    factor_pair(c, g, alpha, T, ui.m, li.p, k, fo.m, co.p);
    fo.copy_out(c, F, ldf, mem);
    co.copy_out(c, C, (int64_t)k * k, mem);
    finish(c);
  });
}

int netmfp_sketch_svd(netmfp_ctx *ctx, int64_t n, const float *F, int64_t ldf, const double *C, int32_t k,
                      double scale, int32_t d, int32_t s2, int32_t s3, int32_t z, uint64_t seed,
                      int32_t logmode, float *U, int64_t ldu, double *sigma, float *E, int64_t lde,
                      float *Ysk, int64_t ldy, double *Zsk, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && F && C, "sketch_svd: NULL argument");
    NM_REQUIRE(logmode == NETMFP_LOG_TRUNC || logmode == NETMFP_LOG_LOG1P, "sketch_svd: bad logmode");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    InMat fi(c, F, n, k, ldf, mem, true);
    InVec<double> ci(c, C, (int64_t)k * k, mem, true);
    const int64_t h2 = (int64_t)d + s2, h3 = (int64_t)d + s3;
    InVec<double> sg(c, sigma, d, mem, false), zo(c, Zsk, h3 * h3, mem, false);
    std::unique_ptr<InMat> uo, eo, yo;
    if (U) uo.reset(new InMat(c, U, n, d, ldu, mem, false));
    if (E) eo.reset(new InMat(c, E, n, d, lde, mem, false));
    if (Ysk) yo.reset(new InMat(c, Ysk, n, h2, ldy, mem, false));
    sketch_svd(c, fi.m, ci.p, k, scale, d, s2, s3, z, seed, logmode, uo ? &uo->m : nullptr, sg.p,
               eo ? &eo->m : nullptr, yo ? &yo->m : nullptr, zo.p);
    if (uo) uo->copy_out(c, U, ldu, mem);
    if (eo) eo->copy_out(c, E, lde, mem);
    if (yo) yo->copy_out(c, Ysk, ldy, mem);
    sg.copy_out(c, sigma, d, mem);
    zo.copy_out(c, Zsk, h3 * h3, mem);
    finish(c);
  });
}

int netmfp_cheb_coeffs(int32_t order, double mu, double theta, double *cc) {
  return guarded([&] {
    NM_REQUIRE(cc && order >= 0 && order <= 64, "cheb_coeffs: bad arguments");
    cheb_coeffs(order, mu, theta, cc);
  });
}

int netmfp_propagate(netmfp_ctx *ctx, const netmfp_graph *gr, float *E, int64_t lde, int32_t d,
                     int32_t order, double mu, double theta, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && gr && E, "propagate: NULL argument");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    const Graph &g = *gr->g;
    InMat ei(c, E, g.n, d, lde, mem, true);
    propagate(c, g, ei.m, order, mu, theta);
    ei.copy_out(c, E, lde, mem);
    finish(c);
  });
}

// The compacted copy of g without its isolated vertices, when embed may run
// on it: g is the whole graph (one rank) or one rank's rows of a
// graph partitioned for this communicator, not itself compacted, and enough
// vertices remain for the rank-(k+s1) basis.  Built once per graph and cached
// (under the graph's lock); a partitioned graph all-gathers the degrees.
static const Graph *embed_graph(Ctx &c, const Graph &g, const netmfp_params &p) {
  static const bool off = [] {
    const char *v = getenv("NETMFP_NO_COMPACT");
    return v && atoi(v);
  }();
  if (off || g.n_orig != 0) return &g;
  const bool whole = g.row0 == 0 && g.n == g.n_global;
  if (c.nranks == 1 && !c.comm && !whole) return &g;  // a row slice used without a communicator
  if ((c.nranks > 1 || c.comm) && (int)g.bounds.size() != c.nranks + 1) return &g;
  std::lock_guard<std::mutex> lk(g.compact_mu);
  if (!g.compact_checked) {
    NM_STAGE(c, "stage_compact");
    DBuf<int32_t> degall;
    const int32_t *da = g.deg.p;
    if (c.nranks > 1 || c.comm) {
      degall.alloc(g.n_global, c.stream);
      dist_allgather_i32(c, g.deg.p, g.bounds, degall.p);
      da = degall.p;
    }
    g.compact.reset(compact_graph(c, g, da));
    g.compact_checked = true;
  }
  if (!g.compact || g.compact->n_global < (int64_t)p.k + p.s1) return &g;
  return g.compact.get();
}

// Host-side zeroing of a pinned output while the GPU computes (see
// embed_host_pinned): worker threads memset E's rows, joined before the GPU
// writes the non-isolated rows.
struct HostZero {
  std::vector<std::thread> th;
  HostZero(float *E, int64_t n, int64_t d, int64_t lde) {
    const int T = (int)std::max<unsigned>(1, std::min<unsigned>(16, std::thread::hardware_concurrency()));
    for (int t = 0; t < T; ++t)
      th.emplace_back([=] {
        const int64_t r0 = n * t / T, r1 = n * (t + 1) / T;
        if (lde == d)
          memset(E + r0 * lde, 0, (size_t)(r1 - r0) * d * sizeof(float));
        else
          for (int64_t r = r0; r < r1; ++r) memset(E + r * lde, 0, (size_t)d * sizeof(float));
      });
  }
  void join() {
    for (auto &t : th)
      if (t.joinable()) t.join();
  }
  ~HostZero() { join(); }
};

// Device pointer through which the GPU can write a host buffer directly
// (pinned, mapped memory under unified addressing), or nullptr.
static float *mapped_device_ptr(float *E) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, E) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (a.type == cudaMemoryTypeHost && a.devicePointer) ? static_cast<float *>(a.devicePointer) : nullptr;
}

// Alg. 5 on graph g (compacted or not); E has g.n rows.
static void embed_core(Ctx &c, const Graph &g, const netmfp_params &p, const Mat &E, double *sigma_dev,
                       double *lambda_dev) {
  NM_REQUIRE(p.T >= 1 && p.b > 0, "embed: need T >= 1, b > 0");
  cudaStream_t s = c.stream;
  const bool compacted = g.n_orig != 0;
  const int64_t n = g.n;
  Block F(n, p.k, s);
  DBuf<double> lam(p.k, s), C((size_t)p.k * p.k, s);
  {
    NM_STAGE(c, "stage_freigs");
    freigs(c, g, p.alpha, p.k, p.s1, p.q, p.seed, F.m, lam, true);    // Alg. 5 step 1 (F = D^(-1+α) U)
  }
  if (lambda_dev) NM_CUDA(cudaMemcpyAsync(lambda_dev, lam.p, p.k * 8, cudaMemcpyDeviceToDevice, s));
  // the Y sketch's A operand (F split into fp16 planes) needs F only: on one
  // GPU it is prepared on the side stream while Eq. 3 runs on the main one
  SketchA preA;
  bool pre = false;
  if (sketch_uses_split() && side_fork(c)) {
    try {
      sketch_split_a(c, F.m, preA);
    } catch (...) {
      c.stream = s;
      throw;
    }
    side_join_point(c, s);
    preA.set_stream(s);
    pre = true;
  }
  {
    NM_STAGE(c, "stage_factor_pair");
    factor_pair(c, g, p.alpha, p.T, F.m, lam, p.k, F.m, C, true);      // steps 2-3
  }
  if (pre) NM_CUDA(cudaStreamWaitEvent(s, c.ev_join, 0));
  const double scale = (double)g.nnz_global / (p.b * p.T);           // vol(G)/(bT)
  {
    NM_STAGE(c, "stage_sketch_svd");
    sketch_svd(c, F.m, C, p.k, scale, p.d, p.s2, p.s3, p.z, p.seed, p.logmode, nullptr, sigma_dev, &E,
               nullptr, nullptr, g.row0, compacted ? g.n_orig : g.n_global,
               compacted ? g.comp_id.p : nullptr, pre ? &preA : nullptr);  // steps 4-5
  }
  F.buf.release();
  {
    NM_STAGE(c, "stage_propagate");
    propagate(c, g, E, p.prop_order, p.mu, p.theta);                   // step 6
  }
}

static void embed_impl(Ctx &c, const Graph &g_in, const netmfp_params &p, const Mat &E_out, double *sigma_dev,
                       double *lambda_dev) {
  const Graph &g = *embed_graph(c, g_in, p);
  if (&g == &g_in) {
    embed_core(c, g, p, E_out, sigma_dev, lambda_dev);
    return;
  }
  Block Ec(g.n, p.d, c.stream);
  embed_core(c, g, p, Ec.m, sigma_dev, lambda_dev);
  // this rank's original rows [g_in.row0, +g_in.n) from its compact rows
  // [g.row0, +g.n); isolated vertices: zero rows [R2]
  scatter_rows(c, Ec.m, g.comp_id.p + g_in.row0, E_out, g.row0);
}

// Host output, compacted graph, pinned E: the host zeroes E (threads, while
// the GPU computes) and the GPU then writes only the n' non-isolated rows
// straight into it — n' instead of n rows cross the host link.  Returns false
// (nothing done) when the path does not apply.
static bool embed_host_pinned(Ctx &c, const Graph &g_in, const netmfp_params &p, float *E, int64_t lde,
                              double *sigma_dev, double *lambda_dev) {
  if (c.nranks > 1 || c.comm) return false;  // partitioned: the staged copy of this rank's rows
  const Graph &g = *embed_graph(c, g_in, p);
  float *Edev = (&g != &g_in) ? mapped_device_ptr(E) : nullptr;
  if (!Edev) return false;
  HostZero zero(E, g_in.n, p.d, lde);
  Block Ec(g.n, p.d, c.stream);
  embed_core(c, g, p, Ec.m, sigma_dev, lambda_dev);
  zero.join();
  Mat Eh{Edev, g.n_orig, p.d, lde};
  write_rows(c, Ec.m, g.orig_id.p, Eh);
  return true;
}

int netmfp_embed(netmfp_ctx *ctx, const netmfp_graph *gr, const netmfp_params *p, float *E, int64_t lde,
                 double *sigma, double *lambda, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && gr && p && E, "embed: NULL argument");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    const Graph &g = *gr->g;
    check_params(*p, g.n_global);
    NM_REQUIRE(lde >= p->d, "embed: lde < d");
    InVec<double> so(c, sigma, p->d, mem, false), lo(c, lambda, p->k, mem, false);
    if (!(mem == NETMFP_MEM_HOST && embed_host_pinned(c, g, *p, E, lde, so.p, lo.p))) {
      InMat eo(c, E, g.n, p->d, lde, mem, false);
      embed_impl(c, g, *p, eo.m, so.p, lo.p);
      eo.copy_out(c, E, lde, mem);
    }
    so.copy_out(c, sigma, p->d, mem);
    lo.copy_out(c, lambda, p->k, mem);
    finish(c);
  });
}

int netmfp_embed_edges(netmfp_ctx *ctx, int64_t n, const int32_t *src, const int32_t *dst, int64_t m_in,
                       const netmfp_params *p, float *E, int64_t lde, double *sigma, int mem) {
  return guarded([&] {
    NM_REQUIRE(ctx && p && E, "embed_edges: NULL argument");
    check_mem(mem);
    Ctx &c = ctx->c;
    DevScope _dev(c);
    check_params(*p, n);
    InVec<int32_t> s(c, src, m_in, mem, true), t(c, dst, m_in, mem, true);
    std::unique_ptr<Graph> g;
    {
      NM_STAGE(c, "stage_build_csr");
      g.reset(build_csr_device(c, n, s.p, t.p, m_in));
    }
    NM_REQUIRE(lde >= p->d, "embed_edges: lde < d");
    InVec<double> so(c, sigma, p->d, mem, false);
    if (!(mem == NETMFP_MEM_HOST && embed_host_pinned(c, *g, *p, E, lde, so.p, nullptr))) {
      InMat eo(c, E, n, p->d, lde, mem, false);
      embed_impl(c, *g, *p, eo.m, so.p, nullptr);
      eo.copy_out(c, E, lde, mem);
    }
    so.copy_out(c, sigma, p->d, mem);
    finish(c);
  });
}

}  // extern "C"
