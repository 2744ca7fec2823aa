// spmm.cu — row a2: Y = coef · D^-a A D^-b X (+ β·Yprev), Acc = σ·Acc + γ·Y.
//
// The normalized-adjacency SpMM of PAPER.md:217 (D^-α A D^-α, freigs) and
// PAPER.md:171 (L~ = -D^-1 A, Chebyshev propagation), applied to an n×c
// row-major fp32 block.  B200 design:
//  * column passes of 4·LPR columns are the grid's y-dimension: 128-column
//    passes (LPR = 32 lanes, one float4 each, per row) and the leftover
//    columns as one narrower pass (LPR = 8/16: 4/2 rows per warp at a time);
//  * light rows (deg <= light_cap): a warp owns 32 consecutive rows (a tile);
//    one coalesced load brings their rowptr, each lane computes its row's
//    scale and prefetches the row's first four column indices, and the warp
//    walks the rows taking that metadata by shuffles, so a row costs one
//    round of X gathers (every lane reads the same column index — an L1
//    broadcast — and its own 16 B of the neighbour's row);
//  * heavy rows (deg > light_cap, power-law hubs): split into heavy_seg-nnz
//    segments, one warp each; every segment stores its partial sum in its own
//    scratch slot and the segment that completes the row (arrival counter)
//    adds the row's partials in segment order and runs the epilogue — the
//    result does not depend on the order segments finish (deterministic);
//  * both kinds of work are blocks of ONE launch (interleaved), so the
//    L2-bound hub gathers overlap the latency-bound light rows;
//  * fused epilogue: row scaling d_u^-a, optional β·prev and σ·acc_in terms
//    (one Clenshaw step of the Chebyshev filter per SpMM).
// The general path with a column scale (D^-b, b != 0) keeps the simpler
// warp-per-row kernels k_spmm_rows / k_spmm_heavy.
#include "common.cuh"
#include "kernels.cuh"

#include <cstdlib>

namespace netmfp {

__device__ __forceinline__ float row_scale(int dg, float a) {
  if (dg <= 0) return 0.f;
  if (a == 0.f) return 1.f;
  if (a == 1.f) return __fdividef(1.f, (float)dg);
  if (a == 0.5f) return rsqrtf((float)dg);
  return exp2f(-a * __log2f((float)dg));
}

__device__ __forceinline__ float4 f4_fma(float s, float4 x, float4 a) {
  a.x = fmaf(s, x.x, a.x);
  a.y = fmaf(s, x.y, a.y);
  a.z = fmaf(s, x.z, a.z);
  a.w = fmaf(s, x.w, a.w);
  return a;
}
__device__ __forceinline__ float4 f4_add(float4 x, float4 a) {
  a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
  return a;
}

// Partial sum over neighbours e in [e0, e1) of one row for this lane's float4
// (Xc = X + this lane's column offset).  Every lane of the row's group reads
// the same column index (an L1 broadcast) and its own 16 B of the neighbour's
// row, so a group moves one full 128-B segment per neighbour; 4 neighbours are
// in flight per iteration.  No shuffles: lanes never wait on each other.
template <bool SCOL>
__device__ __forceinline__ float4 gather_sum(const int32_t *__restrict__ col, int64_t e0, int64_t e1,
                                             const float *__restrict__ Xc, uint32_t ldx,
                                             const float *__restrict__ s_col) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int32_t *cp = col + e0;
  int cnt = (int)(e1 - e0);
  for (; cnt >= 4; cnt -= 4, cp += 4) {
    const uint32_t v0 = __ldg(cp), v1 = __ldg(cp + 1), v2 = __ldg(cp + 2), v3 = __ldg(cp + 3);
    const float4 x0 = __ldg(reinterpret_cast<const float4 *>(Xc + (uint64_t)v0 * ldx));
    const float4 x1 = __ldg(reinterpret_cast<const float4 *>(Xc + (uint64_t)v1 * ldx));
    const float4 x2 = __ldg(reinterpret_cast<const float4 *>(Xc + (uint64_t)v2 * ldx));
    const float4 x3 = __ldg(reinterpret_cast<const float4 *>(Xc + (uint64_t)v3 * ldx));
    if (SCOL) {
      acc = f4_fma(__ldg(s_col + v0), x0, acc);
      acc = f4_fma(__ldg(s_col + v1), x1, acc);
      acc = f4_fma(__ldg(s_col + v2), x2, acc);
      acc = f4_fma(__ldg(s_col + v3), x3, acc);
    } else {
      acc = f4_add(f4_add(x0, x1), acc);
      acc = f4_add(f4_add(x2, x3), acc);
    }
  }
  for (; cnt > 0; --cnt, ++cp) {
    const uint32_t v = __ldg(cp);
    const float4 x = __ldg(reinterpret_cast<const float4 *>(Xc + (uint64_t)v * ldx));
    acc = SCOL ? f4_fma(__ldg(s_col + v), x, acc) : f4_add(x, acc);
  }
  return acc;
}

// per heavy segment: its partial sum into its own slot part[sidx, :] (the
// row kernel adds a row's slots in segment order: deterministic)
template <int LPR, bool SCOL>
__global__ void __launch_bounds__(256, 8) k_spmm_heavy(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                    const int32_t *__restrict__ col,
                                                    const int32_t *__restrict__ heavy,
                                                    const int64_t *__restrict__ seg_e0,
                                                    const int32_t *__restrict__ seg_h, int64_t nsegs,
                                                    float *__restrict__ part, int64_t ldh) {
  grid_dep_enter();
  constexpr int GPB = 256 / LPR;
  const int li = threadIdx.x % LPR;
  const int gi = threadIdx.x / LPR;
  const int c = blockIdx.y * (LPR * 4) + li * 4;
  const bool active = c < p.cols;
  const int64_t sidx = (int64_t)blockIdx.x * GPB + gi;
  if (sidx >= nsegs) return;
  const int64_t h = __ldg(seg_h + sidx);
  const int64_t e0 = __ldg(seg_e0 + sidx);
  const int64_t re = __ldg(rowptr + __ldg(heavy + h) + 1);
  const int64_t e1 = min(e0 + (int64_t)p.heavy_seg, re);
  if (active) {
    float4 acc = gather_sum<SCOL>(col, e0, e1, p.X + c, (uint32_t)p.ldx, p.s_col);
    *reinterpret_cast<float4 *>(part + sidx * ldh + c) = acc;
  }
}

template <int LPR, bool SCOL, int MINB>
__global__ void __launch_bounds__(256, MINB) k_spmm_rows(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                   const int32_t *__restrict__ col, int64_t n,
                                                   const int32_t *__restrict__ heavy, int64_t nh,
                                                   const int64_t *__restrict__ seg_ptr,
                                                   const float *__restrict__ part, int64_t ldh) {
  grid_dep_enter();
  constexpr int GPB = 256 / LPR;
  const int li = threadIdx.x % LPR;
  const int gi = threadIdx.x / LPR;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu
                                     : (((1u << LPR) - 1u) << ((threadIdx.x % 32) / LPR * LPR));
  const int c = blockIdx.y * (LPR * 4) + li * 4;
  const bool active = c < p.cols;
  const int64_t stride = (int64_t)gridDim.x * GPB;
  for (int64_t u = (int64_t)blockIdx.x * GPB + gi; u < n; u += stride) {
    int64_t e0 = __ldg(rowptr + u), e1 = __ldg(rowptr + u + 1);
    int64_t dg = e1 - e0;
    // epilogue operands do not depend on the gather: issue their loads first
    float4 pv = make_float4(0.f, 0.f, 0.f, 0.f), a0 = pv;
    if (active && p.prev) pv = *reinterpret_cast<const float4 *>(p.prev + u * p.ldp + c);
    if (active && p.acc_out && p.acc_in && p.acc_scale != 0.f)
      a0 = *reinterpret_cast<const float4 *>(p.acc_in + u * p.ldai + c);
    float4 acc;
    if (dg > p.light_cap) {
      // heavy row: its segments' partial sums (k_spmm_heavy), added in order
      int64_t lo = 0, hi = nh - 1;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (heavy[mid] < u) lo = mid + 1; else hi = mid;
      }
      acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (active)
        for (int64_t sg = seg_ptr[lo]; sg < seg_ptr[lo + 1]; ++sg)
          acc = f4_add(*reinterpret_cast<const float4 *>(part + sg * ldh + c), acc);
    } else if (active) {
      acc = gather_sum<SCOL>(col, e0, e1, p.X + c, (uint32_t)p.ldx, p.s_col);
    }
    if (!active) continue;
    const float s = p.coef * row_scale(dg, p.a);
    float4 y = make_float4(s * acc.x, s * acc.y, s * acc.z, s * acc.w);
    if (p.prev) y = f4_fma(p.beta, pv, y);
    const int nv = p.cols - c;  // valid floats in this float4 (>= 1)
    if (p.Y) {
      float *dst = p.Y + u * p.ldy + c;
      if (nv >= 4) {
        *reinterpret_cast<float4 *>(dst) = y;
      } else {
        dst[0] = y.x;
        if (nv > 1) dst[1] = y.y;
        if (nv > 2) dst[2] = y.z;
      }
    }
    if (p.acc_out) {
      float4 r;
      r.x = p.acc_scale * a0.x + p.gamma * y.x;
      r.y = p.acc_scale * a0.y + p.gamma * y.y;
      r.z = p.acc_scale * a0.z + p.gamma * y.z;
      r.w = p.acc_scale * a0.w + p.gamma * y.w;
      float *dst = p.acc_out + u * p.ldacc + c;
      if (nv >= 4) {
        *reinterpret_cast<float4 *>(dst) = r;
      } else {
        dst[0] = r.x;
        if (nv > 1) dst[1] = r.y;
        if (nv > 2) dst[2] = r.z;
      }
    }
  }
}

// epilogue traffic is single-use: streamed (.cs: evict-first) so that it does
// not displace the gathered neighbour rows from L1 / L2
__device__ __forceinline__ void store_f4(float *dst, float4 v, int nv) {
  if (nv >= 4) {
    __stcs(reinterpret_cast<float4 *>(dst), v);
  } else {
    dst[0] = v.x;
    if (nv > 1) dst[1] = v.y;
    if (nv > 2) dst[2] = v.z;
  }
}

// Epilogue for row u of one float4 column slice c (nv valid floats):
// y = sr·acc (+ β·prev); Y = y; Acc = σ·Acc + γ·y.
template <bool GEN>
__device__ __forceinline__ void slice_epilogue(const SpmmArgs &p, int64_t u, int c, float sr, float4 acc) {
  const int nv = (int)p.cols - c;
  float4 pv = make_float4(0.f, 0.f, 0.f, 0.f), a0 = pv;
  if (GEN && p.prev) pv = __ldcs(reinterpret_cast<const float4 *>(p.prev + u * p.ldp + c));
  if (GEN && p.acc_out && p.acc_in && p.acc_scale != 0.f)
    a0 = __ldcs(reinterpret_cast<const float4 *>(p.acc_in + u * p.ldai + c));
  float4 y = make_float4(sr * acc.x, sr * acc.y, sr * acc.z, sr * acc.w);
  if (GEN && p.prev) y = f4_fma(p.beta, pv, y);
  if (!GEN || p.Y) store_f4(p.Y + u * p.ldy + c, y, nv);
  if (GEN && p.acc_out) {
    float4 o;
    o.x = p.acc_scale * a0.x + p.gamma * y.x;
    o.y = p.acc_scale * a0.y + p.gamma * y.y;
    o.z = p.acc_scale * a0.z + p.gamma * y.z;
    o.w = p.acc_scale * a0.w + p.gamma * y.w;
    store_f4(p.acc_out + u * p.ldacc + c, o, nv);
  }
}

__device__ __forceinline__ float4 ldx4(const float *__restrict__ Xc, uint32_t v, uint32_t ldx) {
  return __ldg(reinterpret_cast<const float4 *>(Xc + (uint64_t)v * ldx));
}

// One 32-row tile t of light rows (heavy rows are left to their segments).
// Lane groups of LPR lanes (one float4 column slice each) take rows
// gq, gq + GPW, ... of the tile.
template <int LPR, bool GEN>
__device__ __forceinline__ void spmm_tile_rows(const SpmmArgs &p, const int64_t *__restrict__ rowptr,
                                               const int32_t *__restrict__ col, int64_t n, int64_t t, int py) {
  constexpr int GPW = 32 / LPR;  // row groups per warp
  const int lane = threadIdx.x & 31;
  const int gq = lane / LPR, li = lane % LPR;
  const int c = py * (LPR * 4) + li * 4;
  const bool active = c < p.cols;
  const uint32_t ldx = (uint32_t)p.ldx;
  const float *__restrict__ Xc = p.X + c;
  const int64_t u0 = t << 5;
  const int nrows = (int)min((int64_t)32, n - u0);
  const int64_t rp = __ldg(rowptr + u0 + min(lane, nrows));
  const int64_t rpn = __ldg(rowptr + u0 + min(lane + 1, nrows));
  const int dl = (int)(rpn - rp);
  const bool hv = dl > p.light_cap;  // heavy: written by its last segment
  const unsigned hmask = __ballot_sync(0xffffffffu, hv);
  uint32_t k0 = 0, k1 = 0, k2 = 0, k3 = 0;
  if (!hv) {
    if (dl > 0) k0 = __ldg(col + rp);
    if (dl > 1) k1 = __ldg(col + rp + 1);
    if (dl > 2) k2 = __ldg(col + rp + 2);
    if (dl > 3) k3 = __ldg(col + rp + 3);
  }
  const float sl = p.coef * row_scale(dl, p.a);
  const int64_t eb = __shfl_sync(0xffffffffu, rp, 0);
  const int rel = (int)(rp - eb);
#pragma unroll 1
  for (int j = 0; j < LPR; ++j) {
    const int r = gq + j * GPW;
    const int d = __shfl_sync(0xffffffffu, dl, r);
    const int ro = __shfl_sync(0xffffffffu, rel, r);
    const float sr = __shfl_sync(0xffffffffu, sl, r);
    const uint32_t q0 = __shfl_sync(0xffffffffu, k0, r), q1 = __shfl_sync(0xffffffffu, k1, r);
    const uint32_t q2 = __shfl_sync(0xffffffffu, k2, r), q3 = __shfl_sync(0xffffffffu, k3, r);
    if (r >= nrows || !active || ((hmask >> r) & 1u)) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (d > 0) {
      acc = ldx4(Xc, q0, ldx);
      if (d > 1) {
        const float4 x1 = ldx4(Xc, q1, ldx);
        float4 x2 = make_float4(0.f, 0.f, 0.f, 0.f), x3 = x2;
        if (d > 2) x2 = ldx4(Xc, q2, ldx);
        if (d > 3) x3 = ldx4(Xc, q3, ldx);
        acc = f4_add(f4_add(x1, acc), f4_add(x2, x3));
        if (d > 4) acc = f4_add(gather_sum<false>(col, eb + ro + 4, eb + ro + d, Xc, ldx, nullptr), acc);
      }
    }
    slice_epilogue<GEN>(p, u0 + r, c, sr, acc);
  }
}

// Fused SpMM: one launch whose blocks alternate between heavy-row segments
// (L2-bandwidth-bound gathers of hub rows) and 32-row tiles (latency-bound
// light rows), so the two kinds of work overlap instead of running back to
// back.  A heavy segment stores its partial sum in its own slot; the group
// that brings a (row, column pass) counter to the row's segment count adds
// the row's slots in segment order, applies the epilogue and returns the
// counter to zero, so the counters need no clearing between launches.  `py` is the column pass of
// this geometry (4·LPR columns), `cnt_stride` the counters per heavy row.
template <int LPR, bool GEN>
__device__ __forceinline__ void fused_body(const SpmmArgs &p, int py, int bx, const int64_t *__restrict__ rowptr,
                                           const int32_t *__restrict__ col, int64_t n,
                                           const int32_t *__restrict__ heavy, const int64_t *__restrict__ seg_ptr,
                                           const int64_t *__restrict__ seg_e0, const int32_t *__restrict__ seg_h,
                                           int64_t nsegs, float *__restrict__ part,
                                           int32_t *__restrict__ hcnt, int cnt_stride, int nblk_heavy,
                                           int nblk_tile) {
  constexpr int GPB = 256 / LPR;
  const int m = min(nblk_heavy, nblk_tile);
  bool is_heavy;
  int idx;
  if (bx < 2 * m) {
    is_heavy = (bx & 1) == 0;
    idx = bx >> 1;
  } else {
    is_heavy = nblk_heavy > nblk_tile;
    idx = m + (bx - 2 * m);
  }
  if (!is_heavy) {
    if (idx >= nblk_tile) return;
    const int64_t ntiles = (n + 31) >> 5;
    const int64_t wstride = (int64_t)nblk_tile * 8;
    for (int64_t t = (int64_t)idx * 8 + (threadIdx.x >> 5); t < ntiles; t += wstride)
      spmm_tile_rows<LPR, GEN>(p, rowptr, col, n, t, py);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int li = threadIdx.x % LPR;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (lane / LPR * LPR));
  const int c = py * (LPR * 4) + li * 4;
  const bool active = c < p.cols;
  const int64_t sidx = (int64_t)idx * GPB + threadIdx.x / LPR;
  if (sidx >= nsegs) return;
  const int64_t h = __ldg(seg_h + sidx);
  const int64_t e0 = __ldg(seg_e0 + sidx);
  const int64_t u = __ldg(heavy + h);
  const int64_t rb = __ldg(rowptr + u), re = __ldg(rowptr + u + 1);
  const int64_t e1 = min(e0 + (int64_t)p.heavy_seg, re);
  // this segment's slot of the pass: part[(py * nsegs + sidx) * 4·LPR + 4·li]
  constexpr int PW = LPR * 4;
  float *slot = part + ((int64_t)py * nsegs + sidx) * PW + li * 4;
  const float4 acc = active ? gather_sum<false>(col, e0, e1, p.X + c, (uint32_t)p.ldx, nullptr)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
  if (e0 == rb && e1 == re) {  // the whole row in one segment: no partial, no counter
    if (active) slice_epilogue<GEN>(p, u, c, p.coef * row_scale((int)(re - rb), p.a), acc);
    return;
  }
  __stcg(reinterpret_cast<float4 *>(slot), acc);
  // the group's stores are ordered before the arrival by the group barrier
  // and the leader's release RMW at gpu scope (cumulativity).  The partials
  // are written and read at L2 (st/ld .cg), so the last arriver reads them
  // after its RMW without an acquire fence.  No __threadfence here: at gpu
  // scope it compiles to MEMBAR + CCTL.IVALL, and invalidating the SM's L1
  // on every heavy segment threw away the cached hub rows (configs[2], two
  // 128-column passes: 0.477 -> 0.461 ms, bitwise identical)
  __syncwarp(gmask);
  const int64_t s0 = __ldg(seg_ptr + h), s1 = __ldg(seg_ptr + h + 1);
  int32_t *cnt = hcnt + h * cnt_stride + py;
  int last = 0;
  if (li == 0) {
    int old;
    asm volatile("atom.add.release.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    last = old == (int)(s1 - s0) - 1;
  }
  last = __shfl_sync(gmask, last, lane / LPR * LPR);
  if (!last) return;
  if (active) {
    // the row's partials in segment order (independent of arrival order)
    const float *sp = part + ((int64_t)py * nsegs + s0) * PW + li * 4;
    const int64_t ns = s1 - s0;
    float4 tot = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t j = 0;
    for (; j + 4 <= ns; j += 4) {
      const float4 a0 = __ldcg(reinterpret_cast<const float4 *>(sp + (j + 0) * PW));
      const float4 a1 = __ldcg(reinterpret_cast<const float4 *>(sp + (j + 1) * PW));
      const float4 a2 = __ldcg(reinterpret_cast<const float4 *>(sp + (j + 2) * PW));
      const float4 a3 = __ldcg(reinterpret_cast<const float4 *>(sp + (j + 3) * PW));
      tot = f4_add(a3, f4_add(a2, f4_add(a1, f4_add(a0, tot))));
    }
    for (; j < ns; ++j) tot = f4_add(__ldcg(reinterpret_cast<const float4 *>(sp + j * PW)), tot);
    slice_epilogue<GEN>(p, u, c, p.coef * row_scale((int)(re - rb), p.a), tot);
  }
  if (li == 0) *cnt = 0;
}

// Graph operands of the fused launch.
struct FusedGraph {
  const int64_t *rowptr;
  const int32_t *col;
  int64_t n;
  const int32_t *heavy;
  const int64_t *seg_ptr, *seg_e0;
  const int32_t *seg_h;
  int64_t nsegs;
  float *part;  // (column pass, segment) partial sums: passes x nsegs x 4·LPR
  int32_t *hcnt;
  int nblk_tile;
};

template <int LPR, int MINB, bool GEN>
__global__ void __launch_bounds__(256, MINB) k_spmm_fused(SpmmArgs p, FusedGraph fg, int nblk_heavy) {
  grid_dep_enter();
  fused_body<LPR, GEN>(p, blockIdx.y, blockIdx.x, fg.rowptr, fg.col, fg.n, fg.heavy, fg.seg_ptr, fg.seg_e0, fg.seg_h,
                       fg.nsegs, fg.part, fg.hcnt, gridDim.y, nblk_heavy, fg.nblk_tile);
}

// 286 = 2·128 + 30 columns in ONE launch: blockIdx.y < mpasses runs the
// 128-column passes (warp per row), blockIdx.y == mpasses the narrow tail pass
// (8-lane groups), so the tail's blocks start while the last 128-column
// blocks drain instead of after them.  The two share the counter array
// (stride mpasses + 1: the tail's counters are slot mpasses) and use disjoint
// partial-slot regions.
template <bool GEN>
__global__ void __launch_bounds__(256, 8) k_spmm_fused_tail(SpmmArgs pm, SpmmArgs pt, FusedGraph fg, float *part_t,
                                                            int nblk_heavy_m, int nblk_heavy_t) {
  grid_dep_enter();
  const int mpasses = (int)gridDim.y - 1;
  if ((int)blockIdx.y < mpasses) {
    fused_body<32, GEN>(pm, blockIdx.y, blockIdx.x, fg.rowptr, fg.col, fg.n, fg.heavy, fg.seg_ptr, fg.seg_e0,
                        fg.seg_h, fg.nsegs, fg.part, fg.hcnt, gridDim.y, nblk_heavy_m, fg.nblk_tile);
  } else {
    if ((int)blockIdx.x >= fg.nblk_tile + nblk_heavy_t) return;
    fused_body<8, GEN>(pt, 0, blockIdx.x, fg.rowptr, fg.col, fg.n, fg.heavy, fg.seg_ptr, fg.seg_e0, fg.seg_h,
                       fg.nsegs, part_t, fg.hcnt + mpasses, gridDim.y, nblk_heavy_t, fg.nblk_tile);
  }
}

// Warp-per-row path for a column scale s_col (general D^-a A D^-b): heavy
// rows' partial sums from k_spmm_heavy, then k_spmm_rows with the epilogue.
template <int LPR, bool SCOL, int MINB>
static void spmm_rows_impl(Ctx &c, const Graph &g, const SpmmArgs &p) {
  constexpr int GPB = 256 / LPR;
  constexpr int CW = LPR * 4;
  const unsigned chunks = ceil_div(p.cols, CW);
  DBuf<float> part;
  int64_t ldh = pad4(p.cols);
  if (g.n_heavy > 0) {
    part.alloc((size_t)g.n_heavy_segs * ldh, c.stream);
    dim3 gh(ceil_div(g.n_heavy_segs, GPB), chunks);
    NM_LAUNCH(c, "spmm_heavy", launch_pdl(c.stream, k_spmm_heavy<LPR, SCOL>, gh, 256, 0, p, g.rowptr, g.col, g.heavy, g.seg_e0, g.seg_h,
                                                      g.n_heavy_segs, part, ldh));
  }
  int64_t row_blocks = ceil_div(g.n, GPB);
  int64_t cap = (int64_t)c.num_sms * 64;
  dim3 grid((unsigned)std::min<int64_t>(row_blocks, cap), chunks);
  NM_LAUNCH(c, "spmm_rows", launch_pdl(c.stream, k_spmm_rows<LPR, SCOL, MINB>, grid, 256, 0, p, g.rowptr, g.col, g.n, g.heavy, g.n_heavy,
                                                     g.heavy_seg_ptr.p, part.p, ldh));
}

template <int LPR>
static void spmm_fused_impl(Ctx &c, const Graph &g, const SpmmArgs &p) {
  const unsigned passes = ceil_div(p.cols, LPR * 4);
  if (g.n_heavy > 0) {
    // context-owned scratch (one stream per context: launches are ordered);
    // counters are allocated zeroed and every launch leaves them zero
    const size_t need = (size_t)g.n_heavy_segs * passes * LPR * 4, needc = (size_t)g.n_heavy * passes;
    if (c.spmm_part.n < need) c.spmm_part.alloc(need, c.stream);
    if (c.spmm_cnt.n < needc) {
      c.spmm_cnt.alloc(needc, c.stream);
      c.spmm_cnt.zero();
    }
  }
  FusedGraph fg{g.rowptr, g.col, g.n, g.heavy, g.heavy_seg_ptr, g.seg_e0, g.seg_h, g.n_heavy_segs,
                c.spmm_part.p, c.spmm_cnt.p, 0};
  const int64_t ntiles = ceil_div(g.n, 32);
  fg.nblk_tile = (int)std::min<int64_t>(ceil_div(ntiles, 8), (int64_t)c.num_sms * 32);
  const int nbh = g.n_heavy > 0 ? (int)ceil_div(g.n_heavy_segs, 256 / LPR) : 0;
  dim3 grid((unsigned)(fg.nblk_tile + nbh), passes);
  if (p.prev || p.acc_out || !p.Y)
    NM_LAUNCH(c, "spmm_fused", launch_pdl(c.stream, k_spmm_fused<LPR, 8, true>, grid, 256, 0, p, fg, nbh));
  else
    NM_LAUNCH(c, "spmm_fused", launch_pdl(c.stream, k_spmm_fused<LPR, 8, false>, grid, 256, 0, p, fg, nbh));
}

// main (multiple of 128 columns) + tail (<= 32 columns) in one launch
static void spmm_fused_tail_impl(Ctx &c, const Graph &g, const SpmmArgs &pm, const SpmmArgs &pt) {
  const unsigned mpasses = ceil_div(pm.cols, 128);
  if (g.n_heavy > 0) {
    const size_t need = (size_t)g.n_heavy_segs * (mpasses * 128 + 32), needc = (size_t)g.n_heavy * (mpasses + 1);
    if (c.spmm_part.n < need) c.spmm_part.alloc(need, c.stream);
    if (c.spmm_cnt.n < needc) {
      c.spmm_cnt.alloc(needc, c.stream);
      c.spmm_cnt.zero();
    }
  }
  FusedGraph fg{g.rowptr, g.col, g.n, g.heavy, g.heavy_seg_ptr, g.seg_e0, g.seg_h, g.n_heavy_segs,
                c.spmm_part.p, c.spmm_cnt.p, 0};
  const int64_t ntiles = ceil_div(g.n, 32);
  fg.nblk_tile = (int)std::min<int64_t>(ceil_div(ntiles, 8), (int64_t)c.num_sms * 32);
  const int nbh_m = g.n_heavy > 0 ? (int)ceil_div(g.n_heavy_segs, 256 / 32) : 0;
  const int nbh_t = g.n_heavy > 0 ? (int)ceil_div(g.n_heavy_segs, 256 / 8) : 0;
  float *part_t = c.spmm_part.p ? c.spmm_part.p + (size_t)g.n_heavy_segs * mpasses * 128 : nullptr;
  dim3 grid((unsigned)(fg.nblk_tile + nbh_m), mpasses + 1);
  if (pm.prev || pm.acc_out || !pm.Y)
    NM_LAUNCH(c, "spmm_fused", launch_pdl(c.stream, k_spmm_fused_tail<true>, grid, 256, 0, pm, pt, fg, part_t, nbh_m, nbh_t));
  else
    NM_LAUNCH(c, "spmm_fused", launch_pdl(c.stream, k_spmm_fused_tail<false>, grid, 256, 0, pm, pt, fg, part_t, nbh_m, nbh_t));
}

void spmm(Ctx &c, const Graph &g, const SpmmArgs &p_in) {
  SpmmArgs p = p_in;
  p.light_cap = g.light_cap;
  p.heavy_seg = g.heavy_seg;
  NM_REQUIRE(p.cols > 0 && p.ldx % 4 == 0 && p.ldy % 4 == 0, "spmm: ld must be a multiple of 4");
  NM_REQUIRE(p.ldx < (int64_t)1 << 32, "spmm: ldx must fit 32 bits");
  NM_REQUIRE(((uintptr_t)p.X & 15) == 0 && (!p.Y || ((uintptr_t)p.Y & 15) == 0),
             "spmm: buffers must be 16-byte aligned");
  if (g.n == 0) return;
  NM_STAGE(c, "stage_spmm");
  if (p.s_col) {
    spmm_rows_impl<32, true, 4>(c, g, p);
    return;
  }
  // 128-column passes with a warp per row; the leftover columns (286 = 2·128
  // + 30) as one more launch with narrower lane groups (4 or 2 rows per warp
  // at a time) instead of a mostly idle 128-column pass
  static const int pass_w = [] {
    const char *v = getenv("NETMFP_SPMM_W");
    return v ? atoi(v) : 128;
  }();
  const int64_t main = p.cols / pass_w * pass_w, tail = p.cols - main;
  static const bool merge_tail = [] {
    const char *v = getenv("NETMFP_SPMM_MERGE_TAIL");
    return !v || atoi(v) != 0;
  }();
  if (merge_tail && pass_w == 128 && main > 0 && tail > 0 && tail <= 32) {
    SpmmArgs pm = p, pt = p;
    pm.cols = main;
    pt.cols = tail;
    pt.X = p.X + main;
    if (pt.Y) pt.Y = p.Y + main;
    if (pt.prev) pt.prev = p.prev + main;
    if (pt.acc_in) pt.acc_in = p.acc_in + main;
    if (pt.acc_out) pt.acc_out = p.acc_out + main;
    spmm_fused_tail_impl(c, g, pm, pt);
    return;
  }
  if (main > 0) {
    SpmmArgs pm = p;
    pm.cols = main;
    if (pass_w == 64)
      spmm_fused_impl<16>(c, g, pm);
    else if (pass_w == 32)
      spmm_fused_impl<8>(c, g, pm);
    else
      spmm_fused_impl<32>(c, g, pm);
  }
  if (tail > 0) {
    SpmmArgs pt = p;
    pt.cols = tail;
    pt.X = p.X + main;
    if (pt.Y) pt.Y = p.Y + main;
    if (pt.prev) pt.prev = p.prev + main;
    if (pt.acc_in) pt.acc_in = p.acc_in + main;
    if (pt.acc_out) pt.acc_out = p.acc_out + main;
    if (tail <= 32)
      spmm_fused_impl<8>(c, g, pt);
    else if (tail <= 64)
      spmm_fused_impl<16>(c, g, pt);
    else
      spmm_fused_impl<32>(c, g, pt);
  }
}

// d^-e (0 for d = 0) as fp32 — column scaling vector for general (a, b)
__global__ void k_deg_pow(const int32_t *__restrict__ deg, int64_t n, float e, float *__restrict__ out) {
  grid_dep_enter();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = row_scale(deg[i], e);
}

void deg_pow(Ctx &c, const Graph &g, float e, float *out) {
  NM_LAUNCH(c, "deg_pow", launch_pdl(c.stream, k_deg_pow, ceil_div(g.n, 256), 256, 0, g.deg, g.n, e, out));
}

}  // namespace netmfp
