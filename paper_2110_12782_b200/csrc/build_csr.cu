// build_csr.cu — row a1: CSR of the undirected simple graph.
//
// Edge pairs -> 64-bit keys (u << cb | v, cb = bits of a column id) for both
// directions (self loops become the sentinel key (n-1, n-1): a self loop
// itself, so no real edge has it, and it sorts last) -> CUB radix sort over the
// 2 cb + 1 significant bits -> unique -> rowptr by per-row binary search.
// Deterministic and bit-exact (integer work only).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace netmfp {

__global__ void k_make_keys(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                            int64_t m, uint64_t n, uint64_t row0, uint64_t row1, int cb, uint64_t *__restrict__ keys,
                            int *bad) {
  grid_dep_enter();
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  int32_t s = src[e], t = dst[e];
  const uint64_t sentinel = ((n - 1) << cb) | (n - 1);  // the key of the self loop (n-1, n-1)
  if (s < 0 || t < 0 || (uint64_t)s >= n || (uint64_t)t >= n) {
    atomicExch(bad, 1);
    keys[2 * e] = keys[2 * e + 1] = sentinel;
    return;
  }
  if (s == t) {  // self loop: dropped (the sentinel sorts last)
    keys[2 * e] = keys[2 * e + 1] = sentinel;
  } else {
    // rows outside this rank's range [row0, row1) become the sentinel
    keys[2 * e] = ((uint64_t)s >= row0 && (uint64_t)s < row1) ? (((uint64_t)s << cb) | (uint32_t)t) : sentinel;
    keys[2 * e + 1] = ((uint64_t)t >= row0 && (uint64_t)t < row1) ? (((uint64_t)t << cb) | (uint32_t)s) : sentinel;
  }
}

// Row-range builds (one rank's rows [row0, row1)): only the keys of this
// rank's rows are made and sorted — O(m / nranks) device memory for the sort
// instead of 2m keys.  Pass 1 counts them (and flags bad ids), pass 2 appends
// them with warp-aggregated atomics (order irrelevant: they are sorted next).
__device__ __forceinline__ int local_dirs(int32_t s, int32_t t, uint64_t row0, uint64_t row1) {
  if (s == t) return 0;  // self loop: dropped
  return ((uint64_t)s >= row0 && (uint64_t)s < row1 ? 1 : 0) | ((uint64_t)t >= row0 && (uint64_t)t < row1 ? 2 : 0);
}
__global__ void k_count_local(const int32_t *__restrict__ src, const int32_t *__restrict__ dst, int64_t m, uint64_t n,
                              uint64_t row0, uint64_t row1, unsigned long long *__restrict__ cnt, int *bad) {
  grid_dep_enter();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int c = 0;
  if (e < m) {
    const int32_t s = src[e], t = dst[e];
    if (s < 0 || t < 0 || (uint64_t)s >= n || (uint64_t)t >= n) {
      atomicExch(bad, 1);
    } else {
      const int d = local_dirs(s, t, row0, row1);
      c = (d & 1) + (d >> 1);
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}
__global__ void k_make_keys_local(const int32_t *__restrict__ src, const int32_t *__restrict__ dst, int64_t m,
                                  uint64_t n, uint64_t row0, uint64_t row1, int cb, uint64_t *__restrict__ keys,
                                  unsigned long long *__restrict__ pos) {
  grid_dep_enter();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int d = 0;
  int32_t s = 0, t = 0;
  if (e < m) {
    s = src[e];
    t = dst[e];
    if (s >= 0 && t >= 0 && (uint64_t)s < n && (uint64_t)t < n) d = local_dirs(s, t, row0, row1);
  }
  const int c = (d & 1) + (d >> 1);
  int incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  unsigned long long base = 0;
  if (lane == 31 && incl) base = atomicAdd(pos, (unsigned long long)incl);
  base = __shfl_sync(0xffffffffu, base, 31);
  uint64_t at = base + (uint64_t)(incl - c);
  if (d & 1) keys[at++] = ((uint64_t)s << cb) | (uint32_t)t;
  if (d & 2) keys[at] = ((uint64_t)t << cb) | (uint32_t)s;
}

// rowptr[u] = first key index with row >= row0 + u (lower bound), u in [0, n]
// nnz = unique keys minus the sentinel (the last unique key if present)
__global__ void k_nnz(const uint64_t *__restrict__ keys, const int64_t *__restrict__ nuniq, uint64_t n_all, int cb,
                      int64_t *__restrict__ nnz) {
  grid_dep_enter();
  const int64_t u = *nuniq;
  const uint64_t sentinel = ((n_all - 1) << cb) | (n_all - 1);
  *nnz = (u > 0 && keys[u - 1] == sentinel) ? u - 1 : u;
}

__global__ void k_rowptr(const uint64_t *__restrict__ keys, const int64_t *__restrict__ dnnz, int64_t n, int64_t row0,
                         int cb, int64_t *__restrict__ rowptr) {
  grid_dep_enter();
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u > n) return;
  const int64_t nnz = *dnnz;
  uint64_t target = (uint64_t)(u + row0) << cb;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < target) lo = mid + 1; else hi = mid;
  }
  rowptr[u] = lo;
}

__global__ void k_col_deg(const uint64_t *__restrict__ keys, const int64_t *__restrict__ dnnz,
                          const int64_t *__restrict__ rowptr, int64_t n, int cb, int32_t *__restrict__ col,
                          int32_t *__restrict__ deg, uint8_t *__restrict__ heavy_flag, int light_cap) {
  grid_dep_enter();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nnz = *dnnz;
  if (i < nnz) col[i] = (int32_t)(keys[i] & ((1ull << cb) - 1));
  if (i < n) {
    int64_t dg = rowptr[i + 1] - rowptr[i];
    deg[i] = (int32_t)dg;
    heavy_flag[i] = dg > light_cap ? 1 : 0;
  }
}

__global__ void k_heavy_seg_map(const int32_t *__restrict__ heavy, const int64_t *__restrict__ dnh,
                                const int64_t *__restrict__ seg_ptr, const int64_t *__restrict__ rowptr,
                                int64_t *__restrict__ seg_e0, int32_t *__restrict__ seg_h, int heavy_seg) {
  grid_dep_enter();
  const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (h >= *dnh) return;
  const int64_t b = rowptr[heavy[h]];
  for (int64_t sg = seg_ptr[h]; sg < seg_ptr[h + 1]; ++sg) {
    seg_e0[sg] = b + (sg - seg_ptr[h]) * heavy_seg;
    seg_h[sg] = (int32_t)h;
  }
}

// segments per heavy row, zero-padded to n + 1 entries (the heavy count nh is
// a device value): the exclusive scan of all n + 1 gives seg_ptr[0..nh] and
// the total at every index >= nh
__global__ void k_heavy_segs(const int32_t *__restrict__ heavy, const int64_t *__restrict__ dnh, int64_t n,
                             const int32_t *__restrict__ deg, int64_t *__restrict__ nseg, int heavy_seg) {
  grid_dep_enter();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  nseg[i] = i < *dnh ? (deg[heavy[i]] + heavy_seg - 1) / heavy_seg : 0;
}

__global__ void k_flag_nz(const int32_t *__restrict__ deg, int64_t n, int32_t *__restrict__ flag);

static int bits_for(uint64_t v) {
  int b = 0;
  while ((1ull << b) <= v && b < 63) ++b;
  return b;
}

Graph *build_csr_device(Ctx &c, int64_t n_all, const int32_t *src, const int32_t *dst, int64_t m, int64_t row0,
                        int64_t row1) {
  NM_REQUIRE(n_all > 0 && n_all < (1ll << 31), "build_csr: need 0 < n < 2^31");
  NM_REQUIRE(m >= 0, "build_csr: m_in < 0");
  if (row1 < 0) row1 = n_all;
  NM_REQUIRE(row0 >= 0 && row0 <= row1 && row1 <= n_all, "build_csr: bad row range");
  cudaStream_t s = c.stream;
  auto g = new Graph();
  const int64_t n = row1 - row0;  // local rows
  g->n = n;
  g->n_global = n_all;
  g->row0 = row0;
  g->bounds = {0, n_all};
  g->device = c.device;
  if (const char *v = getenv("NETMFP_LIGHT_CAP")) g->light_cap = std::max(1, atoi(v));
  if (const char *v = getenv("NETMFP_HEAVY_SEG")) g->heavy_seg = std::max(1, atoi(v));
  try {
    const bool part = row0 > 0 || row1 < n_all;  // one rank's rows: sort only their keys
    int64_t nk = 2 * m;
    const int cb = std::max(1, bits_for((uint64_t)(n_all - 1)));  // bits of a column id
    DBuf<int> bad(1, s);
    bad.zero();
    DBuf<unsigned long long> kcnt;
    if (part) {
      kcnt.alloc(2, s);
      kcnt.zero();
      unsigned long long hk = 0;
      int hb = 0;
      if (m > 0)
        NM_LAUNCH(c, "count_local", launch_pdl(s, k_count_local, ceil_div(m, 256), 256, 0, src, dst, m, (uint64_t)n_all,
                                                                                  (uint64_t)row0, (uint64_t)row1,
                                                                                  kcnt.p, bad));
      NM_CUDA(cudaMemcpyAsync(&hk, kcnt.p, 8, cudaMemcpyDeviceToHost, s));
      NM_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
      NM_CUDA(cudaStreamSynchronize(s));
      NM_REQUIRE(!hb, "build_csr: vertex id out of [0, n)");
      nk = (int64_t)hk;
    }
    DBuf<uint64_t> keys(nk > 0 ? nk : 1, s), keys2(nk > 0 ? nk : 1, s);
    if (part && nk > 0) {
      NM_LAUNCH(c, "make_keys_local", launch_pdl(s, k_make_keys_local, ceil_div(m, 256), 256, 0, src, dst, m, (uint64_t)n_all, (uint64_t)row0, (uint64_t)row1, cb, keys,
                                          kcnt.p + 1));
    } else if (!part && m > 0) {
      NM_LAUNCH(c, "make_keys", launch_pdl(s, k_make_keys, ceil_div(m, 256), 256, 0, src, dst, m, (uint64_t)n_all, (uint64_t)row0,
                                                                             (uint64_t)row1, cb, keys, bad));
    }
    // key = row << cb | col with rows < n: 2 cb significant bits (one radix
    // pass fewer than with a sentinel row n at 2^20 vertices)
    const int end_bit = cb + bits_for((uint64_t)(n_all - 1));
    size_t tmp_bytes = 0, tmp2 = 0;
    DBuf<int64_t> nsel(1, s);
    if (nk > 0) {
      NM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.p, keys2.p, nk, 0, end_bit, s));
      NM_CUDA(cub::DeviceSelect::Unique(nullptr, tmp2, keys2.p, keys.p, nsel.p, nk, s));
      DBuf<char> tmp(std::max(tmp_bytes, tmp2), s);
      NM_PROF(c, "cub_radix_sort", NM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.p, keys2.p, nk, 0, end_bit, s)));
      c.launches += 4;
      NM_PROF(c, "cub_unique", NM_CUDA(cub::DeviceSelect::Unique(tmp.p, tmp2, keys2.p, keys.p, nsel.p, nk, s)));
      c.launches += 2;
    } else {
      nsel.zero();
    }
    // Everything below sizes its buffers from upper bounds known on the host
    // (nnz <= nk, heavy rows <= n, segments <= nk / heavy_seg + n) and reads
    // the actual counts from device memory, so the build synchronises with
    // the host once, at the end, to fill the graph's host-side counts.
    // drop the sentinel if present: it is the last unique key
    DBuf<int64_t> dnnz(1, s), dnh(1, s);
    NM_LAUNCH(c, "nnz", launch_pdl(s, k_nnz, 1, 1, 0, keys, nsel, (uint64_t)n_all, cb, dnnz));
    const int64_t nnz_cap = nk;
    g->rowptr.alloc(n + 1, s);
    g->col.alloc(nnz_cap > 0 ? nnz_cap : 1, s);
    g->deg.alloc(n > 0 ? n : 1, s);
    DBuf<uint8_t> hflag(n > 0 ? n : 1, s);
    NM_LAUNCH(c, "rowptr", launch_pdl(s, k_rowptr, ceil_div(n + 1, 256), 256, 0, keys, dnnz, n, row0, cb, g->rowptr));
    const int64_t mx = std::max(nnz_cap, n);
    if (mx > 0)  // an empty row range (a rank with no rows) has nothing to fill
      NM_LAUNCH(c, "col_deg", launch_pdl(s, k_col_deg, ceil_div(mx, 256), 256, 0, keys, dnnz, g->rowptr, n, cb, g->col, g->deg,
                                                                               hflag, g->light_cap));
    // heavy rows (degree > light_cap) for the split SpMM path
    g->heavy.alloc(n > 0 ? n : 1, s);
    if (n > 0) {
      size_t tb = 0;
      cub::CountingInputIterator<int32_t> it(0);
      NM_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, hflag.p, g->heavy.p, dnh.p, n, s));
      DBuf<char> tmp(tb, s);
      NM_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, it, hflag.p, g->heavy.p, dnh.p, n, s));
      c.launches += 2;
    } else {
      dnh.zero();
    }
    g->heavy_seg_ptr.alloc(n + 1, s);
    {
      DBuf<int64_t> nseg(n + 1, s);
      NM_LAUNCH(c, "heavy_segs", launch_pdl(s, k_heavy_segs, ceil_div(n + 1, 256), 256, 0, g->heavy, dnh, n, g->deg, nseg,
                                                                                  g->heavy_seg));
      size_t tb2 = 0;
      NM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, nseg.p, g->heavy_seg_ptr.p, n + 1, s));
      DBuf<char> tmp2b(tb2, s);
      NM_CUDA(cub::DeviceScan::ExclusiveSum(tmp2b.p, tb2, nseg.p, g->heavy_seg_ptr.p, n + 1, s));
      c.launches += 1;
    }
    // per segment: first entry and heavy-row index (no search in the SpMM)
    const int64_t seg_cap = nnz_cap / g->heavy_seg + n + 1;
    g->seg_e0.alloc(seg_cap, s);
    g->seg_h.alloc(seg_cap, s);
    if (n > 0)
      NM_LAUNCH(c, "heavy_seg_map", launch_pdl(s, k_heavy_seg_map, ceil_div(n, 128), 128, 0, g->heavy, dnh, g->heavy_seg_ptr, g->rowptr, g->seg_e0, g->seg_h, g->heavy_seg));
    // a whole graph: the scan of (degree > 0) for isolated-vertex compaction
    int32_t hne = -1;
    if (!part && n > 0) {
      DBuf<int32_t> flag(n + 1, s);
      g->nz_pos.alloc(n + 1, s);
      NM_LAUNCH(c, "flag_nz", launch_pdl(s, k_flag_nz, ceil_div(n + 1, 256), 256, 0, g->deg, n, flag));
      size_t tb3 = 0;
      NM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb3, flag.p, g->nz_pos.p, n + 1, s));
      DBuf<char> tmp3(tb3, s);
      NM_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.p, tb3, flag.p, g->nz_pos.p, n + 1, s));
      c.launches += 1;
      NM_CUDA(cudaMemcpyAsync(&hne, g->nz_pos.p + n, 4, cudaMemcpyDeviceToHost, s));
    }
    // the one host round trip: nnz, the bad-id flag, heavy rows, segments
    int64_t hc[3] = {0, 0, 0};
    int hbad = 0;
    NM_CUDA(cudaMemcpyAsync(&hc[0], dnnz.p, 8, cudaMemcpyDeviceToHost, s));
    NM_CUDA(cudaMemcpyAsync(&hc[1], dnh.p, 8, cudaMemcpyDeviceToHost, s));
    NM_CUDA(cudaMemcpyAsync(&hc[2], g->heavy_seg_ptr.p + n, 8, cudaMemcpyDeviceToHost, s));
    NM_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    NM_CUDA(cudaStreamSynchronize(s));
    NM_REQUIRE(!hbad, "build_csr: vertex id out of [0, n)");
    g->nnz = hc[0];
    g->nnz_global = hc[0];
    g->n_heavy = hc[1];
    g->n_heavy_segs = hc[2];
    g->n_nonisolated = hne;
  } catch (...) {
    delete g;
    throw;
  }
  return g;
}

// ---------------------------------------------------------------------------
// Isolated-vertex compaction.  A vertex of degree 0 has a zero
// row and column in every operator of the method ([R2]: d^e := 0), so every
// dense block of embed is zero on it; the compacted graph keeps the other
// vertices in their original order.  Edge offsets are unchanged (isolated
// rows own no entries), so the heavy-row segment tables carry over as is.
// Works on one rank's rows [b0, b1) of a row-partitioned graph too: `degall`
// holds every vertex's degree (all-gathered), compact ids are global, and the
// rank keeps the image [pos[b0], pos[b1]) of its rows.
// ---------------------------------------------------------------------------
__global__ void k_flag_nz(const int32_t *__restrict__ deg, int64_t n, int32_t *__restrict__ flag) {
  grid_dep_enter();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = deg[i] > 0;
  if (i == n) flag[i] = 0;
}
__global__ void k_compact_ids(const int32_t *__restrict__ deg, const int32_t *__restrict__ pos, int64_t n,
                              int64_t b0, int64_t b1, int64_t row0c, int32_t *__restrict__ orig,
                              int32_t *__restrict__ comp) {
  grid_dep_enter();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (deg[i] > 0) {
    comp[i] = pos[i];
    if (i >= b0 && i < b1) orig[pos[i] - row0c] = (int32_t)i;
  } else {
    comp[i] = -1;
  }
}
__global__ void k_compact_rows(const int32_t *__restrict__ orig, int64_t ne, int64_t b0,
                               const int64_t *__restrict__ rowptr, const int32_t *__restrict__ deg, int64_t nnz,
                               int64_t *__restrict__ rp_c, int32_t *__restrict__ deg_c) {
  grid_dep_enter();
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < ne) {
    rp_c[j] = rowptr[orig[j] - b0];
    deg_c[j] = deg[orig[j] - b0];
  }
  if (j == ne) rp_c[ne] = nnz;
}
__global__ void k_remap_ids(const int32_t *__restrict__ in, int64_t m, const int32_t *__restrict__ comp,
                            int32_t *__restrict__ out) {
  grid_dep_enter();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) out[i] = comp[in[i]];
}
// local row index -> local compact row index
__global__ void k_remap_local(const int32_t *__restrict__ in, int64_t m, const int32_t *__restrict__ comp, int64_t b0,
                              int64_t row0c, int32_t *__restrict__ out) {
  grid_dep_enter();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) out[i] = (int32_t)(comp[b0 + in[i]] - row0c);
}

Graph *compact_graph(Ctx &c, const Graph &g, const int32_t *degall) {
  const int64_t n_all = g.n_global;
  if (n_all == 0) return nullptr;
  cudaStream_t s = c.stream;
  const int64_t b0 = g.row0, b1 = g.row0 + g.n;
  std::vector<int64_t> bounds = g.bounds.size() >= 2 ? g.bounds : std::vector<int64_t>{0, n_all};
  std::vector<int32_t> pb(bounds.size());
  int32_t p0 = 0, p1 = 0;
  DBuf<int32_t> pos_own;
  const int32_t *pos = nullptr;
  const bool whole = b0 == 0 && b1 == n_all;
  if (whole && g.n_nonisolated >= 0 && degall == g.deg.p) {
    // the build's scan: no host round trip here
    pos = g.nz_pos.p;
    p0 = 0;
    p1 = (int32_t)g.n_nonisolated;
    pb = {0, (int32_t)g.n_nonisolated};
  } else {
    DBuf<int32_t> flag(n_all + 1, s);
    pos_own.alloc(n_all + 1, s);
    NM_LAUNCH(c, "flag_nz", launch_pdl(s, k_flag_nz, ceil_div(n_all + 1, 256), 256, 0, degall, n_all, flag));
    size_t tb = 0;
    NM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, pos_own.p, n_all + 1, s));
    DBuf<char> tmp(tb, s);
    NM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.p, pos_own.p, n_all + 1, s));
    c.launches += 1;
    pos = pos_own.p;
    // compact images of every rank's bounds (bounds.back() = n_all: the total)
    for (size_t r = 0; r < bounds.size(); ++r)
      NM_CUDA(cudaMemcpyAsync(&pb[r], pos + bounds[r], 4, cudaMemcpyDeviceToHost, s));
    NM_CUDA(cudaMemcpyAsync(&p0, pos + b0, 4, cudaMemcpyDeviceToHost, s));
    NM_CUDA(cudaMemcpyAsync(&p1, pos + b1, 4, cudaMemcpyDeviceToHost, s));
    NM_CUDA(cudaStreamSynchronize(s));
  }
  const int64_t ne_all = pb.back(), row0c = p0, ne = (int64_t)p1 - p0;
  if (ne_all == n_all || ne_all == 0) return nullptr;
  auto gc = new Graph();
  try {
    gc->n = ne;
    gc->n_global = ne_all;
    gc->row0 = row0c;
    gc->bounds.assign(pb.begin(), pb.end());
    gc->nnz = g.nnz;
    gc->nnz_global = g.nnz_global;
    gc->device = g.device;
    gc->light_cap = g.light_cap;
    gc->heavy_seg = g.heavy_seg;
    gc->n_orig = n_all;
    gc->orig_id.alloc(ne > 0 ? ne : 1, s);
    gc->comp_id.alloc(n_all, s);
    NM_LAUNCH(c, "compact_ids", launch_pdl(s, k_compact_ids, ceil_div(n_all, 256), 256, 0, degall, pos, n_all, b0, b1, row0c,
                                                                                    gc->orig_id, gc->comp_id));
    gc->rowptr.alloc(ne + 1, s);
    gc->deg.alloc(ne > 0 ? ne : 1, s);
    NM_LAUNCH(c, "compact_rows", launch_pdl(s, k_compact_rows, ceil_div(ne + 1, 256), 256, 0, gc->orig_id, ne, b0, g.rowptr,
                                                                                        g.deg, g.nnz, gc->rowptr,
                                                                                        gc->deg));
    gc->col.alloc(g.nnz > 0 ? g.nnz : 1, s);
    if (g.nnz > 0)
      NM_LAUNCH(c, "remap_col", launch_pdl(s, k_remap_ids, ceil_div(g.nnz, 256), 256, 0, g.col, g.nnz, gc->comp_id, gc->col));
    gc->n_heavy = g.n_heavy;
    gc->heavy_nnz = g.heavy_nnz;
    gc->n_heavy_segs = g.n_heavy_segs;
    gc->heavy.alloc(g.n_heavy > 0 ? g.n_heavy : 1, s);
    if (g.n_heavy > 0)
      NM_LAUNCH(c, "remap_heavy", launch_pdl(s, k_remap_local, ceil_div(g.n_heavy, 256), 256, 0, g.heavy, g.n_heavy,
                                                                                         gc->comp_id, b0, row0c,
                                                                                         gc->heavy));
    gc->heavy_seg_ptr.alloc(g.n_heavy + 1, s);
    NM_CUDA(cudaMemcpyAsync(gc->heavy_seg_ptr.p, g.heavy_seg_ptr.p, (g.n_heavy + 1) * 8, cudaMemcpyDeviceToDevice, s));
    const int64_t ns = g.n_heavy_segs > 0 ? g.n_heavy_segs : 1;
    gc->seg_e0.alloc(ns, s);
    gc->seg_h.alloc(ns, s);
    NM_CUDA(cudaMemcpyAsync(gc->seg_e0.p, g.seg_e0.p, ns * 8, cudaMemcpyDeviceToDevice, s));
    NM_CUDA(cudaMemcpyAsync(gc->seg_h.p, g.seg_h.p, ns * 4, cudaMemcpyDeviceToDevice, s));
  } catch (...) {
    delete gc;
    throw;
  }
  return gc;
}

// rows[i] <- comp[rows[i]] (-1 for an isolated vertex: its terms are zero and
// every row gather skips indices outside this rank's rows)
void remap_rows(Ctx &c, int32_t *rows, int64_t m, const int32_t *comp) {
  if (m > 0) NM_LAUNCH(c, "remap_rows", launch_pdl(c.stream, k_remap_ids, ceil_div(m, 256), 256, 0, rows, m, comp, rows));
}

}  // namespace netmfp
