// dist.cu — row-partitioned multi-GPU plumbing (north_star: "the CSR is
// row-partitioned ... the dense block is all-gathered over NVLink with NCCL each
// iteration, and the k×k Gram matrices are allreduced").
//
// One process per GPU.  NCCL is loaded at run time (dlopen of libnccl.so.2 —
// the copy torch already mapped into the process, else the system one), so the
// single-GPU library has no link-time NCCL dependency.  With nranks == 1 every
// helper is a no-op / identity: the single-GPU path IS the distributed path
// with one rank.  A host-staged communicator (netmfp_comm_ops callbacks) can
// stand in for NCCL: same calls at the same points, operands staged through
// host memory — the multi-rank tests use it with several processes on one GPU
// (no kernel ever waits on another rank's kernel).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace netmfp {

namespace {
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char *(*errStr)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
  static NcclApi api;
  if (!api.h) {
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!api.h) api.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!api.h) throw Error(NETMFP_ERR_NCCL, std::string("dlopen libnccl.so.2 failed: ") + dlerror());
    auto sym = [&](const char *nm) {
      void *p = dlsym(api.h, nm);
      if (!p) throw Error(NETMFP_ERR_NCCL, std::string("NCCL symbol missing: ") + nm);
      return p;
    };
    api.getUniqueId = (decltype(api.getUniqueId))sym("ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))sym("ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))sym("ncclCommDestroy");
    api.allReduce = (decltype(api.allReduce))sym("ncclAllReduce");
    api.broadcast = (decltype(api.broadcast))sym("ncclBroadcast");
    api.groupStart = (decltype(api.groupStart))sym("ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))sym("ncclGroupEnd");
    api.errStr = (decltype(api.errStr))sym("ncclGetErrorString");
  }
  return api;
}

void nccl_check(ncclResult_t r, const char *what) {
  if (r != ncclSuccess) throw Error(NETMFP_ERR_NCCL, std::string(what) + ": " + nccl().errStr(r));
}
}  // namespace

void dist_unique_id(void *out) {
  static_assert(sizeof(ncclUniqueId) == NETMFP_DIST_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

void dist_init(Ctx &c, const void *id, int nranks, int rank) {
  NM_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "dist_init: bad rank / nranks");
  dist_destroy(c);
  c.nranks = nranks;
  c.rank = rank;
  // one rank: no communicator (every helper is the identity) unless
  // NETMFP_DIST_FORCE_COMM=1 — then the NCCL path runs with one rank (its
  // collectives are copies), which the single-GPU tests use to execute it
  const char *fc = getenv("NETMFP_DIST_FORCE_COMM");
  if (nranks == 1 && !(fc && atoi(fc))) return;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  NM_CUDA(cudaSetDevice(c.device));
  nccl_check(nccl().commInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  c.comm = comm;
  NM_CUDA(cudaStreamCreateWithFlags(&c.comm_stream, cudaStreamNonBlocking));
}

void dist_destroy(Ctx &c) {
  if (c.comm) nccl().commDestroy((ncclComm_t)c.comm);
  c.comm = nullptr;
  if (c.comm_stream) {
    cudaStreamSynchronize(c.comm_stream);
    cudaStreamDestroy(c.comm_stream);
  }
  c.comm_stream = nullptr;
  c.ops_on = false;
  c.nranks = 1;
  c.rank = 0;
}

static size_t dt_size(DType t) {
  return t == DType::F32 || t == DType::I32 ? 4 : t == DType::U8 ? 1 : 8;
}
static int32_t dt_code(DType t) {
  return t == DType::F32 ? NETMFP_DT_F32 : t == DType::F64 ? NETMFP_DT_F64 : t == DType::I64 ? NETMFP_DT_I64
                                                     : t == DType::I32 ? NETMFP_DT_I32 : NETMFP_DT_U8;
}
static ncclDataType_t nccl_dt(DType t) {
  return t == DType::F32 ? ncclFloat32 : t == DType::F64 ? ncclFloat64 : t == DType::I64 ? ncclInt64
                                                 : t == DType::I32 ? ncclInt32 : ncclUint8;
}

void dist_init_ops(Ctx &c, const netmfp_comm_ops &ops, int nranks, int rank) {
  NM_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "dist_init_ops: bad rank / nranks");
  NM_REQUIRE(nranks == 1 || (ops.allreduce_sum && ops.broadcast), "dist_init_ops: missing callbacks");
  dist_destroy(c);
  c.nranks = nranks;
  c.rank = rank;
  c.ops = ops;
  c.ops_on = nranks > 1;
}

static void ops_check(int rc, const char *what) {
  if (rc != 0) throw Error(NETMFP_ERR_NCCL, std::string(what) + ": communicator callback failed");
}

static bool dist_active(const Ctx &c) { return c.nranks > 1 || c.comm != nullptr; }

// Every NCCL call of a context goes to its communicator stream, in program
// order (one stream per communicator: no cross-stream ordering question for
// NCCL), fenced to the compute stream by events on both sides.
static void comm_after_compute(Ctx &c) {
  cudaEvent_t e;
  NM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  NM_CUDA(cudaEventRecord(e, c.stream));
  NM_CUDA(cudaStreamWaitEvent(c.comm_stream, e, 0));
  cudaEventDestroy(e);
}
static void compute_after_comm(Ctx &c) {
  cudaEvent_t e;
  NM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  NM_CUDA(cudaEventRecord(e, c.comm_stream));
  NM_CUDA(cudaStreamWaitEvent(c.stream, e, 0));
  cudaEventDestroy(e);
}

void dist_allreduce(Ctx &c, void *buf, size_t count, DType t) {
  if (!dist_active(c) || count == 0) return;
  NM_STAGE(c, "stage_comm_allreduce");
  const size_t bytes = count * dt_size(t);
  c.comm_bytes += (int64_t)bytes;
  c.collectives++;
  if (c.ops_on) {
    std::vector<char> h(bytes);
    NM_CUDA(cudaMemcpyAsync(h.data(), buf, bytes, cudaMemcpyDeviceToHost, c.stream));
    NM_CUDA(cudaStreamSynchronize(c.stream));
    ops_check(c.ops.allreduce_sum(c.ops.user, h.data(), (int64_t)count, dt_code(t)), "allreduce");
    NM_CUDA(cudaMemcpyAsync(buf, h.data(), bytes, cudaMemcpyHostToDevice, c.stream));
    NM_CUDA(cudaStreamSynchronize(c.stream));
    return;
  }
  comm_after_compute(c);
  nccl_check(nccl().allReduce(buf, buf, count, nccl_dt(t), ncclSum, (ncclComm_t)c.comm, c.comm_stream),
             "ncclAllReduce");
  compute_after_comm(c);
}

// all-gather-v of row blocks: rank r's `rows_r * row_elems` elements land at
// out + bounds[r] * row_elems (the local block is read from `local`)
static void gather_blocks(Ctx &c, const void *local, const std::vector<int64_t> &bounds, int64_t row_elems, DType t,
                          void *out) {
  const size_t es = dt_size(t);
  const int64_t n_all = bounds[c.nranks];
  const int64_t mine = bounds[c.rank + 1] - bounds[c.rank];
  c.comm_bytes += (int64_t)((n_all - mine) * row_elems * es);
  c.collectives++;
  if (c.ops_on) {
    std::vector<char> h((size_t)n_all * row_elems * es);
    if (mine > 0)
      NM_CUDA(cudaMemcpyAsync(h.data() + (size_t)bounds[c.rank] * row_elems * es, local, (size_t)mine * row_elems * es,
                              cudaMemcpyDeviceToHost, c.stream));
    NM_CUDA(cudaStreamSynchronize(c.stream));
    for (int r = 0; r < c.nranks; ++r) {
      const int64_t rows = bounds[r + 1] - bounds[r];
      if (rows == 0) continue;
      ops_check(c.ops.broadcast(c.ops.user, h.data() + (size_t)bounds[r] * row_elems * es, rows * row_elems,
                                dt_code(t), r),
                "broadcast");
    }
    NM_CUDA(cudaMemcpyAsync(out, h.data(), h.size(), cudaMemcpyHostToDevice, c.stream));
    NM_CUDA(cudaStreamSynchronize(c.stream));
    return;
  }
  comm_after_compute(c);
  nccl_check(nccl().groupStart(), "ncclGroupStart");
  for (int r = 0; r < c.nranks; ++r) {
    const int64_t rows = bounds[r + 1] - bounds[r];
    if (rows == 0) continue;
    nccl_check(nccl().broadcast(local, static_cast<char *>(out) + (size_t)bounds[r] * row_elems * es,
                                (size_t)(rows * row_elems), nccl_dt(t), r, (ncclComm_t)c.comm, c.comm_stream),
               "ncclBroadcast");
  }
  nccl_check(nccl().groupEnd(), "ncclGroupEnd");
  compute_after_comm(c);
}

const float *dist_gather_rows(Ctx &c, const Graph &g, const Mat &local, DBuf<float> &scratch) {
  if (!dist_active(c)) {
    NM_REQUIRE(g.n == g.n_global, "partitioned graph used without a communicator (netmfp_dist_init)");
    return local.p;
  }
  NM_REQUIRE((int)g.bounds.size() == c.nranks + 1, "gather: graph not partitioned for this communicator");
  NM_STAGE(c, "stage_comm_gather");
  const int64_t ld = local.ld;
  scratch.alloc((size_t)g.n_global * ld, c.stream);
  gather_blocks(c, local.p, g.bounds, ld, DType::F32, scratch.p);
  return scratch.p;
}

void dist_spmm(Ctx &c, const Graph &g, const Mat &local, const SpmmArgs &p, DBuf<float> &scratch) {
  if (!dist_active(c)) {
    NM_REQUIRE(g.n == g.n_global, "partitioned graph used without a communicator (netmfp_dist_init)");
    SpmmArgs q = p;
    q.X = local.p;
    q.ldx = local.ld;
    spmm(c, g, q);
    return;
  }
  NM_REQUIRE((int)g.bounds.size() == c.nranks + 1, "gather: graph not partitioned for this communicator");
  if (c.ops_on) {  // host-staged: whole block, then the SpMM
    SpmmArgs q = p;
    q.X = dist_gather_rows(c, g, local, scratch);
    q.ldx = local.ld;
    spmm(c, g, q);
    return;
  }
  // NCCL: column slices of <= 128 (the SpMM's pass width), each packed
  // contiguous (n_local x ld_j) and broadcast from every rank into its own
  // n_global x ld_j buffer on the communicator's stream; the compute stream
  // waits for slice j only before pass j, so slice j+1 crosses NVLink while
  // pass j gathers.
  const int64_t cols = p.cols, nl = g.n, ng = g.n_global;
  std::vector<int64_t> c0s, ws, lds, offs;
  int64_t tot = 0;
  for (int64_t c0 = 0; c0 < cols; c0 += 128) {
    const int64_t w = std::min<int64_t>(128, cols - c0), ldj = pad4(w);
    c0s.push_back(c0);
    ws.push_back(w);
    lds.push_back(ldj);
    offs.push_back(tot);
    tot += (ng + nl) * ldj;
  }
  const size_t nsl = c0s.size();
  scratch.alloc((size_t)tot, c.stream);
  for (size_t j = 0; j < nsl; ++j) {
    float *send = scratch.p + offs[j] + ng * lds[j];
    if (nl > 0)
      NM_CUDA(cudaMemcpy2DAsync(send, lds[j] * 4, local.p + c0s[j], local.ld * 4, ws[j] * 4, nl,
                                cudaMemcpyDeviceToDevice, c.stream));
  }
  cudaEvent_t packed;
  NM_CUDA(cudaEventCreateWithFlags(&packed, cudaEventDisableTiming));
  NM_CUDA(cudaEventRecord(packed, c.stream));
  NM_CUDA(cudaStreamWaitEvent(c.comm_stream, packed, 0));
  cudaEventDestroy(packed);
  std::vector<cudaEvent_t> arrived(nsl);
  const bool prof = c.prof && prof_match(c, "stage_comm_gather");
  for (size_t j = 0; j < nsl; ++j) {
    cudaEvent_t pa = nullptr, pb = nullptr;
    if (prof) {
      pa = prof_event(c);
      cudaEventRecord(pa, c.comm_stream);
    }
    const float *send = scratch.p + offs[j] + ng * lds[j];
    float *recv = scratch.p + offs[j];
    nccl_check(nccl().groupStart(), "ncclGroupStart");
    for (int r = 0; r < c.nranks; ++r) {
      const int64_t rows = g.bounds[r + 1] - g.bounds[r];
      if (rows == 0) continue;
      nccl_check(nccl().broadcast(send, recv + g.bounds[r] * lds[j], (size_t)(rows * lds[j]), ncclFloat32, r,
                                  (ncclComm_t)c.comm, c.comm_stream),
                 "ncclBroadcast");
    }
    nccl_check(nccl().groupEnd(), "ncclGroupEnd");
    if (prof) {
      pb = prof_event(c);
      cudaEventRecord(pb, c.comm_stream);
      c.pending.push_back({pa, pb, "stage_comm_gather"});
    }
    NM_CUDA(cudaEventCreateWithFlags(&arrived[j], cudaEventDisableTiming));
    NM_CUDA(cudaEventRecord(arrived[j], c.comm_stream));
    c.comm_bytes += (ng - nl) * lds[j] * 4;
    c.collectives++;
  }
  for (size_t j = 0; j < nsl; ++j) {
    NM_CUDA(cudaStreamWaitEvent(c.stream, arrived[j], 0));
    cudaEventDestroy(arrived[j]);
    SpmmArgs q = p;
    const int64_t c0 = c0s[j];
    q.X = scratch.p + offs[j];
    q.ldx = lds[j];
    q.cols = ws[j];
    if (q.Y) q.Y += c0;
    if (q.prev) q.prev += c0;
    if (q.acc_in) q.acc_in += c0;
    if (q.acc_out) q.acc_out += c0;
    spmm(c, g, q);
  }
}

void dist_allgather_i32(Ctx &c, const int32_t *local, const std::vector<int64_t> &bounds, int32_t *out) {
  if (!dist_active(c)) {
    if (bounds[1] > 0 && out != local)
      NM_CUDA(cudaMemcpyAsync(out, local, (size_t)bounds[1] * 4, cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  NM_STAGE(c, "stage_comm_gather");
  gather_blocks(c, local, bounds, 1, DType::I32, out);
}

}  // namespace netmfp
