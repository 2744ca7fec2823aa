// spmm.cu — row a2: Y = coef · D^-a A D^-b X (+ β·Yprev), Acc = σ·Acc + γ·Y.
//
// The normalized-adjacency SpMM of PAPER.md:217 (D^-α A D^-α, freigs) and
// PAPER.md:171 (L~ = -D^-1 A, Chebyshev propagation), applied to an n×c
// row-major fp32 block.  B200 design:
//  * column chunks of CW = 4·LPR floats (128 B at LPR = 8) are the grid's
//    y-dimension, so all row-blocks of chunk 0 run before chunk 1: the
//    gathered working set per chunk is n·128 B and stays L2-resident;
//  * light rows (deg <= light_cap): one LPR-lane group per row, each lane a
//    float4 column slice; the group loads LPR column indices in one coalesced
//    read, shuffles them, and keeps LPR independent 16-B gathers in flight;
//  * heavy rows (deg > light_cap, power-law hubs): split into heavy_seg-nnz
//    segments, one group each, partial sums reduced with float4 atomics into
//    a small buffer that the light kernel's epilogue reads;
//  * fused epilogue: row scaling d_u^-a (degree from rowptr, no extra load),
//    optional β·prev (Chebyshev three-term recurrence) and acc update.
#include "common.cuh"
#include "kernels.cuh"

#include <cstdlib>

namespace netmfp {

__device__ __forceinline__ float row_scale(int64_t dg, float a) {
  if (dg <= 0) return 0.f;
  if (a == 0.f) return 1.f;
  if (a == 1.f) return 1.f / (float)dg;
  if (a == 0.5f) return rsqrtf((float)dg);
  return powf((float)dg, -a);
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

template <int LPR, bool SCOL>
__global__ void __launch_bounds__(256, 8) k_spmm_heavy(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                    const int32_t *__restrict__ col,
                                                    const int32_t *__restrict__ heavy,
                                                    const int64_t *__restrict__ seg_e0,
                                                    const int32_t *__restrict__ seg_h, int64_t nsegs,
                                                    float *__restrict__ hsum, int64_t ldh) {
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
    float *dst = hsum + h * ldh + c;
    atomicAdd(reinterpret_cast<float4 *>(dst), acc);
  }
}

template <int LPR, bool SCOL, int MINB>
__global__ void __launch_bounds__(256, MINB) k_spmm_rows(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                   const int32_t *__restrict__ col, int64_t n,
                                                   const int32_t *__restrict__ heavy, int64_t nh,
                                                   const float *__restrict__ hsum, int64_t ldh) {
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
      // heavy row: partial sums were reduced by k_spmm_heavy
      int64_t lo = 0, hi = nh - 1;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (heavy[mid] < u) lo = mid + 1; else hi = mid;
      }
      acc = active ? *reinterpret_cast<const float4 *>(hsum + lo * ldh + c)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
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

// Fused epilogue for row u: y = coef·d_u^-a·acc (+ β·prev); Y = y; Acc = σ·Acc + γ·y.
__device__ __forceinline__ void row_epilogue(const SpmmArgs &p, int64_t u, int64_t dg, float4 acc, int c) {
  const float s = p.coef * row_scale(dg, p.a);
  float4 y = make_float4(s * acc.x, s * acc.y, s * acc.z, s * acc.w);
  if (p.prev) y = f4_fma(p.beta, *reinterpret_cast<const float4 *>(p.prev + u * p.ldp + c), y);
  const int nv = (int)p.cols - c;
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
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p.acc_in && p.acc_scale != 0.f) a0 = *reinterpret_cast<const float4 *>(p.acc_in + u * p.ldai + c);
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

// Flattened row-block SpMM: each warp owns blocks of 32 consecutive rows whose
// rowptr it stages in shared memory once; each LPR-lane group streams the
// neighbours of its 32/GPW rows in batches of 4 that cross row boundaries
// (segmented accumulation), so short rows never serialise memory latency.
// Heavy rows (a ballot mask per block) are skipped and finalised from hsum.
template <int LPR, bool SCOL>
__global__ void __launch_bounds__(256) k_spmm_flat(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                   const int32_t *__restrict__ col, int64_t n,
                                                   const int32_t *__restrict__ heavy, int64_t nh,
                                                   const float *__restrict__ hsum, int64_t ldh) {
  constexpr int GPW = 32 / LPR;  // groups per warp
  constexpr int RPG = 32 / GPW;  // rows per group in a 32-row block
  __shared__ int64_t srp_all[8][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int64_t *srp = srp_all[wib];
  const int gi = lane / LPR, li = lane % LPR;
  const int c = blockIdx.y * (LPR * 4) + li * 4;
  const bool active = c < p.cols;
  const float *Xc = p.X + c;
  const uint32_t ldx = (uint32_t)p.ldx;
  const int64_t wstride = (int64_t)gridDim.x * 8 * 32;
  for (int64_t r0 = ((int64_t)blockIdx.x * 8 + wib) * 32; r0 < n; r0 += wstride) {
    srp[lane] = __ldg(rowptr + min(r0 + lane, n));
    if (lane == 31) srp[32] = __ldg(rowptr + min(r0 + 32, n));
    __syncwarp();
    const unsigned hmask = __ballot_sync(0xffffffffu, srp[lane + 1] - srp[lane] > p.light_cap);
    const int rb = gi * RPG, re = rb + RPG;
    const unsigned range = (re == 32 ? 0xffffffffu : ((1u << re) - 1u));
    const int64_t gend = srp[re];
    int row = rb;
    int64_t e = srp[rb];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    auto finalize = [&](int ri) {
      const int64_t u = r0 + ri;
      if (u >= n || !active) return;
      const int64_t dg = srp[ri + 1] - srp[ri];
      if (dg > p.light_cap) {
        int64_t lo = 0, hi = nh - 1;
        while (lo < hi) {
          int64_t mid = (lo + hi) >> 1;
          if (heavy[mid] < u) lo = mid + 1; else hi = mid;
        }
        acc = *reinterpret_cast<const float4 *>(hsum + lo * ldh + c);
      }
      row_epilogue(p, u, dg, acc, c);
    };
    while (true) {
      while (row < re && srp[row + 1] <= e) {
        finalize(row);
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        ++row;
      }
      if (row >= re) break;
      if ((hmask >> row) & 1u) {
        finalize(row);
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        e = srp[row + 1];
        ++row;
        continue;
      }
      const unsigned hm = hmask & range & (row == 31 ? 0u : ~((2u << row) - 1u));
      const int64_t run_end = hm ? srp[__ffs(hm) - 1] : gend;
      const int nb = (int)min((int64_t)4, run_end - e);
      uint32_t v[4];
      float4 x[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) v[t] = t < nb ? (uint32_t)__ldg(col + e + t) : 0u;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        x[t] = (t < nb && active) ? __ldg(reinterpret_cast<const float4 *>(Xc + (uint64_t)v[t] * ldx))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        if (SCOL && t < nb && active) {
          const float sc = __ldg(p.s_col + v[t]);
          x[t].x *= sc; x[t].y *= sc; x[t].z *= sc; x[t].w *= sc;
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t < nb) {
          while (srp[row + 1] <= e + t) {
            finalize(row);
            acc = make_float4(0.f, 0.f, 0.f, 0.f);
            ++row;
          }
          acc = f4_add(x[t], acc);
        }
      }
      e += nb;
    }
    __syncwarp();
  }
}

// Segmented warp-per-32-rows SpMM.  A warp owns 32 consecutive rows and a
// column pass of 128·NV columns (lane = NV float4 slices).  Their neighbour
// lists are walked as one flat run: each 32-entry chunk loads its column
// indices coalesced (one per lane), lanes find their row by a shuffle binary
// search, and the X gathers of 8 entries are issued back to back (8·NV
// independent 16-B loads per lane in flight) before the accumulation, which
// flushes a row through the fused epilogue whenever the (warp-uniform) row
// index advances.  Entries of heavy rows are skipped (their partial sums come
// from k_spmm_heavy) and whole heavy ranges are jumped over.
template <int NV, bool SCOL>
__global__ void __launch_bounds__(256) k_spmm_seg(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                  const int32_t *__restrict__ col, int64_t n,
                                                  const int32_t *__restrict__ heavy, int64_t nh,
                                                  const float *__restrict__ hsum, int64_t ldh) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  int cq[NV];
  bool aq[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    cq[q] = blockIdx.y * (128 * NV) + (q * 32 + lane) * 4;
    aq[q] = cq[q] < p.cols;
  }
  const uint32_t ldx = (uint32_t)p.ldx;
  for (int64_t r0 = wid * 32; r0 < n; r0 += nwarps * 32) {
    const int rows = (int)min((int64_t)32, n - r0);
    const int64_t rs = __ldg(rowptr + r0 + min(lane, rows));
    const int64_t re = __ldg(rowptr + r0 + min(lane + 1, rows));
    const unsigned hmask = __ballot_sync(FULL, lane < rows && re - rs > p.light_cap);
    const int64_t E0 = __shfl_sync(FULL, rs, 0), E1 = __shfl_sync(FULL, re, rows - 1);
    float4 acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    int cur = 0;
    // flush rows [cur, upto): row cur gets acc, later ones are empty (or heavy)
    auto flush_to = [&](int upto) {
      for (; cur < upto; ++cur) {
        const int64_t u = r0 + cur;
        const int64_t dg = __shfl_sync(FULL, re, cur) - __shfl_sync(FULL, rs, cur);
        if ((hmask >> cur) & 1u) {
          int64_t lo = 0, hi = nh - 1;
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(heavy + mid) < u) lo = mid + 1; else hi = mid;
          }
#pragma unroll
          for (int q = 0; q < NV; ++q)
            if (aq[q]) acc[q] = *reinterpret_cast<const float4 *>(hsum + lo * ldh + cq[q]);
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          if (aq[q]) row_epilogue(p, u, dg, acc[q], cq[q]);
          acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    };
    int64_t e = E0;
    while (e < E1) {
      const int64_t idx = e + lane;
      // row of this lane's entry: largest r with rs_r <= idx (shuffle binary search)
      int lo = 0, hi = rows - 1;
#pragma unroll
      for (int it = 0; it < 5; ++it) {
        const int mid = (lo + hi + 1) >> 1;
        const int64_t v = __shfl_sync(FULL, rs, mid);
        if (v <= idx) lo = mid; else hi = mid - 1;
      }
      const int myrow = idx < E1 ? lo : 32;
      const int row0 = __shfl_sync(FULL, myrow, 0);
      if ((hmask >> row0) & 1u) {  // chunk starts inside a heavy row: jump over it
        e = __shfl_sync(FULL, re, row0);
        continue;
      }
      const bool valid = idx < E1 && !((hmask >> myrow) & 1u);
      const int32_t cv = valid ? __ldg(col + idx) : -1;
#pragma unroll 1
      for (int j = 0; j < 32; j += 8) {
        float4 x[8][NV];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int32_t v = __shfl_sync(FULL, cv, j + t);
          float sc = 1.f;
          if (SCOL && v >= 0) sc = __ldg(p.s_col + v);
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            x[t][q] = (v >= 0 && aq[q]) ? __ldg(reinterpret_cast<const float4 *>(p.X + (uint64_t)(uint32_t)v * ldx + cq[q]))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
            if (SCOL) { x[t][q].x *= sc; x[t][q].y *= sc; x[t][q].z *= sc; x[t][q].w *= sc; }
          }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int r = __shfl_sync(FULL, myrow, j + t);
          if (r >= 32) break;
          if (r != cur) flush_to(r);
#pragma unroll
          for (int q = 0; q < NV; ++q) acc[q] = f4_add(x[t][q], acc[q]);
        }
      }
      e += 32;
    }
    flush_to(rows);
  }
}

// Warp-per-row SpMM with a column pass of 128·NV columns (lane = NV float4
// slices).  Per row: the row's column indices are loaded coalesced (one per
// lane, 32 at a time) and broadcast by shuffles, and the X gathers of 8
// neighbours are issued back to back (8·NV independent 16-B loads per lane)
// before they are summed; the next row's rowptr pair is prefetched while the
// current row is gathered.  Heavy rows take their sums from k_spmm_heavy.
template <int NV, bool SCOL>
__global__ void __launch_bounds__(256) k_spmm_wr(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                 const int32_t *__restrict__ col, int64_t n,
                                                 const int32_t *__restrict__ heavy, int64_t nh,
                                                 const float *__restrict__ hsum, int64_t ldh) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  int cq[NV];
  bool aq[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    cq[q] = blockIdx.y * (128 * NV) + (q * 32 + lane) * 4;
    aq[q] = cq[q] < p.cols;
  }
  const uint32_t ldx = (uint32_t)p.ldx;
  int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  int64_t e0 = 0, e1 = 0;
  if (u < n) {
    e0 = __ldg(rowptr + u);
    e1 = __ldg(rowptr + u + 1);
  }
  for (; u < n; u += nwarps) {
    // prefetch the next row's range
    const int64_t un = u + nwarps;
    int64_t f0 = 0, f1 = 0;
    if (un < n) {
      f0 = __ldg(rowptr + un);
      f1 = __ldg(rowptr + un + 1);
    }
    const int64_t dg = e1 - e0;
    float4 acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (dg > p.light_cap) {
      int64_t lo = 0, hi = nh - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(heavy + mid) < u) lo = mid + 1; else hi = mid;
      }
#pragma unroll
      for (int q = 0; q < NV; ++q)
        if (aq[q]) acc[q] = *reinterpret_cast<const float4 *>(hsum + lo * ldh + cq[q]);
    } else {
      for (int64_t b = e0; b < e1; b += 32) {
        const int cnt = (int)min((int64_t)32, e1 - b);
        const int32_t cv = lane < cnt ? __ldg(col + b + lane) : 0;
        for (int j = 0; j < cnt; j += 8) {
          float4 x[8][NV];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int32_t v = __shfl_sync(FULL, cv, j + t);
            const bool ok = j + t < cnt;
            float sc = 1.f;
            if (SCOL && ok) sc = __ldg(p.s_col + v);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
              x[t][q] = (ok && aq[q]) ? __ldg(reinterpret_cast<const float4 *>(p.X + (uint64_t)(uint32_t)v * ldx + cq[q]))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
              if (SCOL) { x[t][q].x *= sc; x[t][q].y *= sc; x[t][q].z *= sc; x[t][q].w *= sc; }
            }
          }
#pragma unroll
          for (int t = 0; t < 8; ++t)
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] = f4_add(x[t][q], acc[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q)
      if (aq[q]) row_epilogue(p, u, dg, acc[q], cq[q]);
    e0 = f0;
    e1 = f1;
  }
}

template <int NV, bool SCOL>
static void spmm_wr_impl(Ctx &c, const Graph &g, const SpmmArgs &p) {
  constexpr int CW = 128 * NV;
  const unsigned chunks = ceil_div(p.cols, CW);
  DBuf<float> hsum;
  int64_t ldh = pad4(p.cols);
  if (g.n_heavy > 0) {
    hsum.alloc((size_t)g.n_heavy * ldh, c.stream);
    hsum.zero();
    dim3 gh(ceil_div(g.n_heavy_segs, 8), ceil_div(p.cols, 128));
    NM_LAUNCH(c, "spmm_heavy", k_spmm_heavy<32, SCOL><<<gh, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.heavy, g.seg_e0,
                                                                                 g.seg_h, g.n_heavy_segs, hsum, ldh));
  }
  const int64_t blocks = ceil_div(g.n, 8);  // 8 warps, one row each per iteration
  dim3 grid((unsigned)std::min<int64_t>(blocks, (int64_t)c.num_sms * 64), chunks);
  NM_LAUNCH(c, "spmm_wr", k_spmm_wr<NV, SCOL><<<grid, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.n, g.heavy,
                                                                            g.n_heavy, hsum.p, ldh));
}

template <int NV, bool SCOL>
static void spmm_seg_impl(Ctx &c, const Graph &g, const SpmmArgs &p) {
  constexpr int CW = 128 * NV;
  const unsigned chunks = ceil_div(p.cols, CW);
  DBuf<float> hsum;
  int64_t ldh = pad4(p.cols);
  if (g.n_heavy > 0) {
    hsum.alloc((size_t)g.n_heavy * ldh, c.stream);
    hsum.zero();
    dim3 gh(ceil_div(g.n_heavy_segs, 8), chunks * NV);
    NM_LAUNCH(c, "spmm_heavy", k_spmm_heavy<32, SCOL><<<gh, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.heavy, g.seg_e0,
                                                                                 g.seg_h, g.n_heavy_segs, hsum, ldh));
  }
  const int64_t blocks = ceil_div(g.n, 256);  // 8 warps × 32 rows
  dim3 grid((unsigned)std::min<int64_t>(blocks, (int64_t)c.num_sms * 16), chunks);
  NM_LAUNCH(c, "spmm_seg", k_spmm_seg<NV, SCOL><<<grid, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.n, g.heavy,
                                                                              g.n_heavy, hsum.p, ldh));
}

template <int LPR, bool SCOL>
static void spmm_flat_impl(Ctx &c, const Graph &g, const SpmmArgs &p) {
  constexpr int GPB = 256 / LPR;
  constexpr int CW = LPR * 4;
  const unsigned chunks = ceil_div(p.cols, CW);
  DBuf<float> hsum;
  int64_t ldh = pad4(p.cols);
  if (g.n_heavy > 0) {
    hsum.alloc((size_t)g.n_heavy * ldh, c.stream);
    hsum.zero();
    dim3 gh(ceil_div(g.n_heavy_segs, GPB), chunks);
    NM_LAUNCH(c, "spmm_heavy", k_spmm_heavy<LPR, SCOL><<<gh, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.heavy, g.seg_e0, g.seg_h,
                                                      g.n_heavy_segs, hsum, ldh));
  }
  const int64_t blocks = ceil_div(g.n, 256);  // 8 warps × 32 rows
  dim3 grid((unsigned)std::min<int64_t>(blocks, (int64_t)c.num_sms * 32), chunks);
  NM_LAUNCH(c, "spmm_flat", k_spmm_flat<LPR, SCOL><<<grid, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.n, g.heavy,
                                                                             g.n_heavy, hsum.p, ldh));
}

// Two-slice variants: a column pass of cw <= 256 columns (cw = 4·(32 + extra)),
// lane li owns columns c0 = base + 4 li and, for li < extra, c1 = base + 128 + 4 li.
// 286 columns thus take two passes of 144 instead of 128 + 128 + 30.
template <bool SCOL>
__device__ __forceinline__ void gather_sum2(const int32_t *__restrict__ col, int64_t e0, int64_t e1,
                                            const float *__restrict__ X0, const float *__restrict__ X1, bool two,
                                            uint32_t ldx, const float *__restrict__ s_col, float4 &a0,
                                            float4 &a1) {
  a0 = make_float4(0.f, 0.f, 0.f, 0.f);
  a1 = a0;
  const int32_t *cp = col + e0;
  int cnt = (int)(e1 - e0);
  for (; cnt >= 4; cnt -= 4, cp += 4) {
    const uint32_t v0 = __ldg(cp), v1 = __ldg(cp + 1), v2 = __ldg(cp + 2), v3 = __ldg(cp + 3);
    float4 x0 = __ldg(reinterpret_cast<const float4 *>(X0 + (uint64_t)v0 * ldx));
    float4 x1 = __ldg(reinterpret_cast<const float4 *>(X0 + (uint64_t)v1 * ldx));
    float4 x2 = __ldg(reinterpret_cast<const float4 *>(X0 + (uint64_t)v2 * ldx));
    float4 x3 = __ldg(reinterpret_cast<const float4 *>(X0 + (uint64_t)v3 * ldx));
    float4 y0 = make_float4(0.f, 0.f, 0.f, 0.f), y1 = y0, y2 = y0, y3 = y0;
    if (two) {
      y0 = __ldg(reinterpret_cast<const float4 *>(X1 + (uint64_t)v0 * ldx));
      y1 = __ldg(reinterpret_cast<const float4 *>(X1 + (uint64_t)v1 * ldx));
      y2 = __ldg(reinterpret_cast<const float4 *>(X1 + (uint64_t)v2 * ldx));
      y3 = __ldg(reinterpret_cast<const float4 *>(X1 + (uint64_t)v3 * ldx));
    }
    if (SCOL) {
      const float s0 = __ldg(s_col + v0), s1 = __ldg(s_col + v1), s2 = __ldg(s_col + v2), s3 = __ldg(s_col + v3);
      a0 = f4_fma(s0, x0, a0); a0 = f4_fma(s1, x1, a0); a0 = f4_fma(s2, x2, a0); a0 = f4_fma(s3, x3, a0);
      a1 = f4_fma(s0, y0, a1); a1 = f4_fma(s1, y1, a1); a1 = f4_fma(s2, y2, a1); a1 = f4_fma(s3, y3, a1);
    } else {
      a0 = f4_add(f4_add(x0, x1), a0);
      a0 = f4_add(f4_add(x2, x3), a0);
      a1 = f4_add(f4_add(y0, y1), a1);
      a1 = f4_add(f4_add(y2, y3), a1);
    }
  }
  for (; cnt > 0; --cnt, ++cp) {
    const uint32_t v = __ldg(cp);
    const float4 x = __ldg(reinterpret_cast<const float4 *>(X0 + (uint64_t)v * ldx));
    const float4 y = two ? __ldg(reinterpret_cast<const float4 *>(X1 + (uint64_t)v * ldx)) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float sc = SCOL ? __ldg(s_col + v) : 1.f;
    a0 = f4_fma(sc, x, a0);
    a1 = f4_fma(sc, y, a1);
  }
}

template <bool SCOL>
__global__ void __launch_bounds__(256) k_spmm_heavy2(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                     const int32_t *__restrict__ col, const int32_t *__restrict__ heavy,
                                                     const int64_t *__restrict__ seg_e0,
                                                     const int32_t *__restrict__ seg_h, int64_t nsegs, int cw,
                                                     float *__restrict__ hsum, int64_t ldh) {
  const int li = threadIdx.x & 31;
  const int64_t sidx = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (sidx >= nsegs) return;
  const int base = blockIdx.y * cw;
  const int c0 = base + li * 4, c1 = base + 128 + li * 4;
  const bool act0 = c0 < p.cols && c0 < base + cw;
  const bool act1 = c1 < p.cols && c1 < base + cw;
  const int64_t h = __ldg(seg_h + sidx);
  const int64_t e0 = __ldg(seg_e0 + sidx);
  const int64_t re = __ldg(rowptr + __ldg(heavy + h) + 1);
  const int64_t e1 = min(e0 + (int64_t)p.heavy_seg, re);
  if (!act0) return;
  float4 a0, a1;
  gather_sum2<SCOL>(col, e0, e1, p.X + c0, p.X + (act1 ? c1 : c0), act1, (uint32_t)p.ldx, p.s_col, a0, a1);
  atomicAdd(reinterpret_cast<float4 *>(hsum + h * ldh + c0), a0);
  if (act1) atomicAdd(reinterpret_cast<float4 *>(hsum + h * ldh + c1), a1);
}

template <bool SCOL>
__global__ void __launch_bounds__(256, 4) k_spmm_rows2(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                       const int32_t *__restrict__ col, int64_t n, int cw,
                                                       const int32_t *__restrict__ heavy, int64_t nh,
                                                       const float *__restrict__ hsum, int64_t ldh) {
  const int li = threadIdx.x & 31;
  const int base = blockIdx.y * cw;
  const int c0 = base + li * 4, c1 = base + 128 + li * 4;
  const bool act0 = c0 < p.cols && c0 < base + cw;
  const bool act1 = c1 < p.cols && c1 < base + cw;
  const int64_t stride = (int64_t)gridDim.x * 8;
  for (int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); u < n; u += stride) {
    const int64_t e0 = __ldg(rowptr + u), e1 = __ldg(rowptr + u + 1);
    const int64_t dg = e1 - e0;
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
    if (dg > p.light_cap) {
      int64_t lo = 0, hi = nh - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(heavy + mid) < u) lo = mid + 1; else hi = mid;
      }
      if (act0) a0 = *reinterpret_cast<const float4 *>(hsum + lo * ldh + c0);
      if (act1) a1 = *reinterpret_cast<const float4 *>(hsum + lo * ldh + c1);
    } else if (act0) {
      gather_sum2<SCOL>(col, e0, e1, p.X + c0, p.X + (act1 ? c1 : c0), act1, (uint32_t)p.ldx, p.s_col, a0, a1);
    }
    if (act0) row_epilogue(p, u, dg, a0, c0);
    if (act1) row_epilogue(p, u, dg, a1, c1);
  }
}

template <bool SCOL>
static void spmm2_impl(Ctx &c, const Graph &g, const SpmmArgs &p) {
  const int nch = (int)ceil_div(p.cols, 256);
  const int cw = (int)((ceil_div(p.cols, nch) + 3) / 4 * 4);
  DBuf<float> hsum;
  int64_t ldh = pad4(p.cols);
  if (g.n_heavy > 0) {
    hsum.alloc((size_t)g.n_heavy * ldh, c.stream);
    hsum.zero();
    dim3 gh(ceil_div(g.n_heavy_segs, 8), nch);
    NM_LAUNCH(c, "spmm_heavy", k_spmm_heavy2<SCOL><<<gh, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.heavy, g.seg_e0,
                                                                            g.seg_h, g.n_heavy_segs, cw, hsum, ldh));
  }
  const int64_t row_blocks = ceil_div(g.n, 8);
  dim3 grid((unsigned)std::min<int64_t>(row_blocks, (int64_t)c.num_sms * 64), nch);
  NM_LAUNCH(c, "spmm_rows", k_spmm_rows2<SCOL><<<grid, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.n, cw, g.heavy,
                                                                          g.n_heavy, hsum.p, ldh));
}

template <int LPR, bool SCOL, int MINB>
static void spmm_impl(Ctx &c, const Graph &g, const SpmmArgs &p) {
  constexpr int GPB = 256 / LPR;
  constexpr int CW = LPR * 4;
  const unsigned chunks = ceil_div(p.cols, CW);
  DBuf<float> hsum;
  int64_t ldh = pad4(p.cols);
  if (g.n_heavy > 0) {
    hsum.alloc((size_t)g.n_heavy * ldh, c.stream);
    hsum.zero();
    dim3 gh(ceil_div(g.n_heavy_segs, GPB), chunks);
    NM_LAUNCH(c, "spmm_heavy", k_spmm_heavy<LPR, SCOL><<<gh, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.heavy, g.seg_e0, g.seg_h,
                                                      g.n_heavy_segs, hsum, ldh));
  }
  // rows per group: enough blocks for ~16 resident 256-thread blocks per SM
  int64_t row_blocks = ceil_div(g.n, GPB);
  int64_t cap = (int64_t)c.num_sms * 64;
  dim3 grid((unsigned)std::min<int64_t>(row_blocks, cap), chunks);
  NM_LAUNCH(c, "spmm_rows", k_spmm_rows<LPR, SCOL, MINB><<<grid, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.n, g.heavy, g.n_heavy,
                                                     hsum.p, ldh));
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
  // tuning variants (NETMFP_SPMM env var, default 0): lanes per row x min blocks/SM
  static int variant = [] {
    const char *v = getenv("NETMFP_SPMM");
    return v ? atoi(v) : 32;
  }();
  if (p.s_col) {
    spmm_impl<32, true, 4>(c, g, p);
    return;
  }
  if (variant == 32 && p.cols > 128 && (p.cols % 128) != 0) {
    // 128-column passes with a warp per row, then the leftover columns with
    // narrower lane groups (4 or 2 rows per warp) instead of a mostly idle pass
    const int64_t main = p.cols / 128 * 128, tail = p.cols - main;
    SpmmArgs pm = p, pt = p;
    pm.cols = main;
    pt.cols = tail;
    pt.X = p.X + main;
    if (pt.Y) pt.Y = p.Y + main;
    if (pt.prev) pt.prev = p.prev + main;
    if (pt.acc_in) pt.acc_in = p.acc_in + main;
    if (pt.acc_out) pt.acc_out = p.acc_out + main;
    spmm_impl<32, false, 8>(c, g, pm);
    if (tail <= 32)
      spmm_impl<8, false, 8>(c, g, pt);
    else if (tail <= 64)
      spmm_impl<16, false, 8>(c, g, pt);
    else
      spmm_impl<32, false, 8>(c, g, pt);
    return;
  }
  switch (variant) {
    case 30: spmm2_impl<false>(c, g, p); break;
    case 31: spmm_impl<32, false, 6>(c, g, p); break;
    case 32: spmm_impl<32, false, 8>(c, g, p); break;
    case 21: spmm_wr_impl<1, false>(c, g, p); break;
    case 22: spmm_wr_impl<2, false>(c, g, p); break;
    case 23: spmm_wr_impl<3, false>(c, g, p); break;
    case 11: spmm_seg_impl<1, false>(c, g, p); break;
    case 12: spmm_seg_impl<2, false>(c, g, p); break;
    case 13: spmm_seg_impl<3, false>(c, g, p); break;
    case 0: spmm_impl<8, false, 4>(c, g, p); break;
    case 1: spmm_impl<8, false, 5>(c, g, p); break;
    case 8: spmm_impl<16, false, 5>(c, g, p); break;
    case 9: spmm_impl<32, false, 4>(c, g, p); break;
    case 10: spmm_impl<16, false, 3>(c, g, p); break;
    case 2: spmm_impl<4, false, 4>(c, g, p); break;
    case 3: spmm_impl<16, false, 4>(c, g, p); break;
    case 4: spmm_impl<4, false, 6>(c, g, p); break;
    case 5: spmm_flat_impl<8, false>(c, g, p); break;
    case 6: spmm_flat_impl<16, false>(c, g, p); break;
    case 7: spmm_flat_impl<32, false>(c, g, p); break;
    default: spmm_impl<16, false, 4>(c, g, p); break;  // variant 3: 64-column chunks
  }
}

// d^-e (0 for d = 0) as fp32 — column scaling vector for general (a, b)
__global__ void k_deg_pow(const int32_t *__restrict__ deg, int64_t n, float e, float *__restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = row_scale(deg[i], e);
}

void deg_pow(Ctx &c, const Graph &g, float e, float *out) {
  NM_LAUNCH(c, "deg_pow", k_deg_pow<<<ceil_div(g.n, 256), 256, 0, c.stream>>>(g.deg, g.n, e, out));
}

}  // namespace netmfp
