// common.cuh — shared plumbing of libnetmfp (context, errors, buffers, RNG).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <memory>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/netmfp.h"

namespace netmfp {

// ----------------------------------------------------------------------------
// errors: internal code throws netmfp::Error; the C ABI converts to codes.
// ----------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &msg);

#define NM_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) {                                                           \
      throw ::netmfp::Error(_e == cudaErrorMemoryAllocation ? NETMFP_ERR_OOM           \
                                                            : NETMFP_ERR_CUDA,         \
                            std::string(#call) + ": " + cudaGetErrorString(_e) +       \
                                " (" __FILE__ ":" + std::to_string(__LINE__) + ")");  \
    }                                                                                  \
  } while (0)

#define NM_REQUIRE(cond, msg)                                        \
  do {                                                               \
    if (!(cond)) throw ::netmfp::Error(NETMFP_ERR_ARG, (msg));       \
  } while (0)

// stream-ordered device buffer (cudaMallocAsync pool; freed on scope exit)
template <class T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) NM_CUDA(cudaMallocAsync((void **)&p, count * sizeof(T), st));
  }
  void zero() {
    if (n) NM_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T *get() const { return p; }
  operator T *() const { return p; }
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf &operator=(DBuf &&o) noexcept {
    release();
    p = o.p; n = o.n; s = o.s;
    o.p = nullptr; o.n = 0;
    return *this;
  }
  ~DBuf() { release(); }
};

// Kernel attributes are per (kernel, device): set an attribute on the current
// device unless this value (or, for the dynamic shared memory limit, a larger
// one) is already set there.  Thread-safe; replaces per-process static guards.
inline void func_attr(const void *kern, cudaFuncAttribute a, int v) {
  static std::mutex mu;
  static std::map<std::tuple<const void *, int, int>, int> done;
  int dev = 0;
  NM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(kern, dev, (int)a);
  auto it = done.find(key);
  if (it != done.end() && (it->second == v || (a == cudaFuncAttributeMaxDynamicSharedMemorySize && it->second >= v)))
    return;
  NM_CUDA(cudaFuncSetAttribute(kern, a, v));
  done[key] = v;
}
template <class K>
inline void smem_attr(K kern, size_t bytes) {
  func_attr(reinterpret_cast<const void *>(kern), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// ----------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int64_t launches = 0;
  int *d_flags = nullptr;  // device status flags (numeric breakdown counters)
  // per-kernel CUDA-event profiling (netmfp_ctx_profile): events around each
  // launch whose name matches one of the comma-separated filter prefixes
  bool prof = false;
  std::string prof_filter;
  struct PEv {
    cudaEvent_t a, b;
    const char *name;
  };
  std::vector<PEv> pending;
  std::vector<cudaEvent_t> evpool;
  cudaEvent_t cur_a = nullptr;
  const char *cur_name = nullptr;
  std::vector<std::pair<std::string, std::pair<int64_t, double>>> stats;
  // row-partitioned multi-GPU (dist.cu); nranks == 1: single GPU
  int nranks = 1, rank = 0;
  void *comm = nullptr;  // ncclComm_t
  cudaStream_t comm_stream = nullptr;  // NCCL stream (overlaps all-gathers with SpMM passes)
  // single-GPU side stream for work independent of the main chain (Alg. 4's
  // Z sketch beside orth(Y)), forked / joined by events; created on first use
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  netmfp_comm_ops ops{};  // host-staged communicator (netmfp_dist_init_ops) when ops_on
  bool ops_on = false;
  int64_t collectives = 0;
  int64_t comm_bytes = 0;  // bytes received in collectives (netmfp_dist_stats)
  // numeric checks deferred to the end of the ABI call (one synchronisation):
  // the stage whose Cholesky failure bit (d_flags & 1<<30) is reported
  std::vector<const char *> flag_checks;
  // SpMM heavy-row scratch owned by the context (one stream: launches on it
  // are ordered): per (column pass, heavy segment) partial sums, and per
  // (heavy row, column pass) arrival counters that every launch leaves zero
  DBuf<float> spmm_part;
  DBuf<int32_t> spmm_cnt;
};

inline bool prof_match(const Ctx &c, const char *name) {
  if (c.prof_filter.empty()) return true;
  size_t st = 0;
  const std::string n(name);
  while (st <= c.prof_filter.size()) {
    size_t e = c.prof_filter.find(',', st);
    if (e == std::string::npos) e = c.prof_filter.size();
    std::string tok = c.prof_filter.substr(st, e - st);
    if (!tok.empty() && n.compare(0, tok.size(), tok) == 0) return true;
    st = e + 1;
  }
  return false;
}

inline cudaEvent_t prof_event(Ctx &c) {
  if (c.evpool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = c.evpool.back();
  c.evpool.pop_back();
  return e;
}

inline void prof_begin(Ctx &c, const char *name) {
  c.cur_name = nullptr;
  if (!c.prof || !prof_match(c, name)) return;
  c.cur_a = prof_event(c);
  cudaEventRecord(c.cur_a, c.stream);
  c.cur_name = name;
}

// count + check a kernel launch (and close its profiling interval)
inline void launched(Ctx &c, const char *what) {
  c.launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(NETMFP_ERR_CUDA, std::string("launch ") + what + ": " + cudaGetErrorString(e));
  if (c.cur_name) {
    cudaEvent_t b = prof_event(c);
    cudaEventRecord(b, c.stream);
    c.pending.push_back({c.cur_a, b, c.cur_name});
    c.cur_name = nullptr;
  }
}

// fold finished intervals into per-kernel (count, total ms); stream must be idle
inline void prof_collect(Ctx &c) {
  // "gaps": stream time between consecutive profiled kernels (memsets,
  // copies, host synchronisation and launch latency) when all are profiled
  cudaEvent_t prev_end = nullptr;
  double gap_ms = 0.0;
  for (auto &pe : c.pending) {
    if (std::string(pe.name).compare(0, 6, "stage_") == 0) continue;
    if (prev_end) {
      float g = 0.f;
      cudaEventElapsedTime(&g, prev_end, pe.a);
      gap_ms += g;
      if (getenv("NETMFP_PROF_GAPS") && c.prof_filter.empty()) {  // attribute to the kernel that follows
        const std::string key = std::string("gap>") + pe.name;
        bool f = false;
        for (auto &s : c.stats)
          if (s.first == key) {
            s.second.first += 1;
            s.second.second += g;
            f = true;
          }
        if (!f) c.stats.push_back({key, {1, (double)g}});
      }
    }
    prev_end = pe.b;
  }
  if (prev_end && c.prof_filter.empty()) {
    bool found = false;
    for (auto &s : c.stats)
      if (s.first == "gaps") {
        s.second.first += 1;
        s.second.second += gap_ms;
        found = true;
      }
    if (!found) c.stats.push_back({"gaps", {1, gap_ms}});
  }
  for (auto &pe : c.pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pe.a, pe.b);
    bool found = false;
    for (auto &s : c.stats)
      if (s.first == pe.name) {
        s.second.first += 1;
        s.second.second += ms;
        found = true;
        break;
      }
    if (!found) c.stats.push_back({pe.name, {1, (double)ms}});
    c.evpool.push_back(pe.a);
    c.evpool.push_back(pe.b);
  }
  c.pending.clear();
}

// Stream-time interval of a whole stage (kernels, copies, memsets and idle
// gaps between them), recorded like a kernel when profiling matches `name`.
struct StageScope {
  Ctx &c;
  const char *name;
  cudaEvent_t a = nullptr;
  StageScope(Ctx &cc, const char *n) : c(cc), name(n) {
    if (!c.prof || !prof_match(c, n)) return;
    a = prof_event(c);
    cudaEventRecord(a, c.stream);
  }
  ~StageScope() {
    if (!a) return;
    cudaEvent_t b = prof_event(c);
    cudaEventRecord(b, c.stream);
    c.pending.push_back({a, b, name});
  }
  StageScope(const StageScope &) = delete;
  StageScope &operator=(const StageScope &) = delete;
};
#define NM_STAGE_CAT2(a, b) a##b
#define NM_STAGE_CAT(a, b) NM_STAGE_CAT2(a, b)
#define NM_STAGE(c, name) ::netmfp::StageScope NM_STAGE_CAT(_stage_, __LINE__)(c, name)

// a library call that launches kernels itself (CUB): profiled like one of
// ours (per-kernel stats, so it is not counted as an idle gap); the caller
// adds its kernel count to c.launches
inline void prof_end(Ctx &c) {
  if (c.cur_name) {
    cudaEvent_t b = prof_event(c);
    cudaEventRecord(b, c.stream);
    c.pending.push_back({c.cur_a, b, c.cur_name});
    c.cur_name = nullptr;
  }
}
#define NM_PROF(c, name, ...)      \
  do {                             \
    ::netmfp::prof_begin(c, name); \
    __VA_ARGS__;                   \
    ::netmfp::prof_end(c);         \
  } while (0)


// ----------------------------------------------------------------------------
// Programmatic dependent launch.  Every kernel of the library is launched with
// launch_pdl and starts with grid_dep_enter() (griddepcontrol.wait): it waits
// until the kernel before it in the stream has completed and its writes are
// visible, but its launch is processed while that kernel drains, so the
// launch latency between consecutive kernels is hidden (configs[2]: 24.50 ->
// 24.05 ms per embedding).  An early griddepcontrol.launch_dependents in every
// kernel was measured slower (29.5 ms: waiting CTAs of the next kernel hold
// SM slots), in the SpMM alone no faster.  In a kernel launched without the
// attribute the wait is a no-op.  NETMFP_PDL=0 launches without it (A/B).
// ----------------------------------------------------------------------------
__device__ __forceinline__ void grid_dep_enter() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char *v = getenv("NETMFP_PDL");
    return !v || atoi(v) != 0;
  }();
  return on;
}

// kern<<<grid, block, smem, s>>>(args...) with the programmatic-serialization
// attribute; arguments are converted to the kernel's parameter types first
template <typename... KArgs, typename... Args>
inline void launch_pdl(cudaStream_t s, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args &&...args) {
  static_assert(sizeof...(KArgs) == sizeof...(Args), "launch_pdl: argument count");
  std::tuple<std::decay_t<KArgs>...> vals(std::forward<Args>(args)...);
  void *ptrs[sizeof...(KArgs) > 0 ? sizeof...(KArgs) : 1];
  std::apply([&](auto &...e) {
    int i = 0;
    ((ptrs[i++] = (void *)&e), ...);
  }, vals);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelExC(&cfg, reinterpret_cast<const void *>(kern), ptrs);
}

#define NM_LAUNCH(c, name, ...)   \
  do {                            \
    ::netmfp::prof_begin(c, name); \
    __VA_ARGS__;                  \
    ::netmfp::launched(c, name);  \
  } while (0)

// Dense fp32 block view: rows × cols, row-major, leading dimension ld.
struct Mat {
  float *p = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
  float *row(int64_t i) const { return p + i * ld; }
};

inline int64_t pad4(int64_t c) { return (c + 3) / 4 * 4; }
inline int64_t pad32(int64_t c) { return (c + 31) / 32 * 32; }

// Owned dense fp32 block with ld padded to a multiple of 32 floats (128 B row
// segments).  Nothing is cleared: every producer writes the rows × cols
// interior before it is read, and no consumer's valid output depends on the
// padding columns (tensor maps clip the contraction dimension at cols; the
// Gram's padded blocks only feed discarded rows/columns; SpMM lanes past
// cols are not stored).
struct Block {
  DBuf<float> buf;
  Mat m;
  Block() = default;
  Block(int64_t rows, int64_t cols, cudaStream_t s) { alloc(rows, cols, s); }
  void alloc(int64_t rows, int64_t cols, cudaStream_t s) {
    int64_t ld = pad32(cols);
    buf.alloc((size_t)rows * ld, s);
    m.p = buf.p;
    m.rows = rows;
    m.cols = cols;
    m.ld = ld;
  }
  operator Mat() const { return m; }
};

// ----------------------------------------------------------------------------
// graph (device CSR)
// ----------------------------------------------------------------------------
// rows with more neighbours than light_cap are split across warps in segments
// of heavy_seg entries (spmm.cu); per graph, NETMFP_LIGHT_CAP / NETMFP_HEAVY_SEG
constexpr int kLightCapDefault = 64;
constexpr int kHeavySegDefault = 256;  // configs[2] SpMM family per embedding: 64 11.94, 96 11.46, 128 11.01-11.18, 192 11.05, 256 10.87-10.96, 384 11.01, 512 11.36 ms (scripts/gpu_ab_seg.sh; 128 was best while every segment fenced L1 away)

struct Graph {
  int64_t n = 0, nnz = 0;  // local rows [row0, row0 + n) and their nonzeros
  int64_t n_global = 0, row0 = 0;
  int64_t nnz_global = 0;            // vol(G)
  std::vector<int64_t> bounds;       // row bounds of every rank (nranks + 1), host
  DBuf<int64_t> rowptr;   // n+1
  DBuf<int32_t> col;      // nnz
  DBuf<int32_t> deg;      // n
  DBuf<int32_t> heavy;    // rows with degree > kLightCap, ascending
  int64_t n_heavy = 0;
  int64_t heavy_nnz = 0;
  DBuf<int64_t> heavy_seg_ptr;  // per heavy row: first segment index (n_heavy+1)
  int64_t n_heavy_segs = 0;
  int light_cap = kLightCapDefault, heavy_seg = kHeavySegDefault;
  DBuf<int64_t> seg_e0;  // per heavy segment: first entry
  DBuf<int32_t> seg_h;   // per heavy segment: index into heavy
  int device = 0;
  // isolated-vertex compaction (embed): for a compacted graph, the original
  // vertex count, compact -> original ids and original -> compact (-1 for
  // degree 0); for a full graph, its cached compacted copy (if built)
  int64_t n_orig = 0;
  DBuf<int32_t> orig_id, comp_id;
  // a whole graph's exclusive scan of (degree > 0) and its total, computed by
  // the build before its one host round trip, so compaction needs none
  DBuf<int32_t> nz_pos;
  int64_t n_nonisolated = -1;
  mutable std::unique_ptr<Graph> compact;
  mutable bool compact_checked = false;
  mutable std::mutex compact_mu;  // the cached compacted copy is built once
  void detach_streams() {  // free on the legacy stream (owning stream may be gone)
    rowptr.s = col.s = deg.s = heavy.s = nullptr;
    heavy_seg_ptr.s = seg_e0.s = nullptr;
    seg_h.s = orig_id.s = comp_id.s = nz_pos.s = nullptr;
    if (compact) compact->detach_streams();
  }
};


// ----------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11) — the CUDA side's own implementation of
// the counter-based generator named in DESIGN.md [R1].
// ----------------------------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ inline U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    U4 o;
    o.x = hi1 ^ c.y ^ k0;
    o.y = lo1;
    o.z = hi0 ^ c.w ^ k1;
    o.w = lo0;
    c = o;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

constexpr uint32_t kTagOmega = 0x4F4D4547u;
constexpr uint32_t kTagPsi = 0x50534931u;
constexpr uint32_t kTagPi = 0x50493132u;

inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace netmfp
