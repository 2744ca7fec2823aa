// dist.cu — row-partitioned multi-GPU plumbing (north_star: "the CSR is
// row-partitioned ... the dense block is all-gathered over NVLink with NCCL each
// iteration, and the k×k Gram matrices are allreduced").
//
// One process per GPU.  NCCL is loaded at run time (dlopen of libnccl.so.2 —
// the copy torch already mapped into the process, else the system one), so the
// single-GPU library has no link-time NCCL dependency.  With nranks == 1 every
// helper is a no-op / identity: the single-GPU path IS the distributed path
// with one rank, which is how the GPU parity tests cover it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

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
  if (nranks == 1) return;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  NM_CUDA(cudaSetDevice(c.device));
  nccl_check(nccl().commInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  c.comm = comm;
}

void dist_destroy(Ctx &c) {
  if (c.comm) nccl().commDestroy((ncclComm_t)c.comm);
  c.comm = nullptr;
  c.nranks = 1;
  c.rank = 0;
}

void dist_allreduce(Ctx &c, void *buf, size_t count, DType t) {
  if (c.nranks == 1 || count == 0) return;
  const ncclDataType_t dt = t == DType::F32 ? ncclFloat32 : t == DType::F64 ? ncclFloat64 : ncclInt64;
  nccl_check(nccl().allReduce(buf, buf, count, dt, ncclSum, (ncclComm_t)c.comm, c.stream), "ncclAllReduce");
  c.collectives++;
}

const float *dist_gather_rows(Ctx &c, const Graph &g, const Mat &local, DBuf<float> &scratch) {
  if (c.nranks == 1) {
    NM_REQUIRE(g.n == g.n_global, "partitioned graph used without a communicator (netmfp_dist_init)");
    return local.p;
  }
  NM_REQUIRE((int)g.bounds.size() == c.nranks + 1, "gather: graph not partitioned for this communicator");
  const int64_t ld = local.ld;
  scratch.alloc((size_t)g.n_global * ld, c.stream);
  nccl_check(nccl().groupStart(), "ncclGroupStart");
  for (int r = 0; r < c.nranks; ++r) {
    const int64_t rows = g.bounds[r + 1] - g.bounds[r];
    if (rows == 0) continue;
    nccl_check(nccl().broadcast(local.p, scratch.p + g.bounds[r] * ld, (size_t)rows * ld, ncclFloat32, r,
                                (ncclComm_t)c.comm, c.stream),
               "ncclBroadcast");
  }
  nccl_check(nccl().groupEnd(), "ncclGroupEnd");
  c.collectives++;
  return scratch.p;
}

}  // namespace netmfp
