// spmm.cu — row a2: Y = coef · D^-a A D^-b X (+ β·Yprev), Acc = σ·Acc + γ·Y.
//
// The normalized-adjacency SpMM of PAPER.md:217 (D^-α A D^-α, freigs) and
// PAPER.md:171 (L~ = -D^-1 A, Chebyshev propagation), applied to an n×c
// row-major fp32 block.  B200 design:
//  * column chunks of CW = 4·LPR floats (128 B at LPR = 8) are the grid's
//    y-dimension, so all row-blocks of chunk 0 run before chunk 1: the
//    gathered working set per chunk is n·128 B and stays L2-resident;
//  * light rows (deg <= kLightCap): one LPR-lane group per row, each lane a
//    float4 column slice; the group loads LPR column indices in one coalesced
//    read, shuffles them, and keeps LPR independent 16-B gathers in flight;
//  * heavy rows (deg > kLightCap, power-law hubs): split into kHeavySeg-nnz
//    segments, one group each, partial sums reduced with float4 atomics into
//    a small buffer that the light kernel's epilogue reads;
//  * fused epilogue: row scaling d_u^-a (degree from rowptr, no extra load),
//    optional β·prev (Chebyshev three-term recurrence) and acc update.
#include "common.cuh"
#include "kernels.cuh"

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

// Partial sum over neighbours e in [e0, e1) of one row for this lane's float4.
template <int LPR, bool SCOL>
__device__ __forceinline__ float4 gather_sum(const int32_t *__restrict__ col, int64_t e0, int64_t e1,
                                             const float *__restrict__ X, int64_t ldx, int c,
                                             bool active, const float *__restrict__ s_col,
                                             int li, unsigned gmask) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t e = e0; e < e1; e += LPR) {
    int64_t my = e + li;
    int vidx = my < e1 ? __ldg(col + my) : -1;
    float sc = 1.f;
    if (SCOL && vidx >= 0) sc = __ldg(s_col + vidx);
    float4 xs[LPR];
    float ss[LPR];
#pragma unroll
    for (int t = 0; t < LPR; ++t) {
      int v = __shfl_sync(gmask, vidx, t, LPR);
      ss[t] = SCOL ? __shfl_sync(gmask, sc, t, LPR) : 1.f;
      xs[t] = (v >= 0 && active) ? __ldg(reinterpret_cast<const float4 *>(X + (int64_t)v * ldx + c))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int t = 0; t < LPR; ++t) acc = SCOL ? f4_fma(ss[t], xs[t], acc) : f4_add(xs[t], acc);
  }
  return acc;
}

template <int LPR, bool SCOL>
__global__ void __launch_bounds__(256) k_spmm_heavy(SpmmArgs p, const int64_t *__restrict__ rowptr,
                                                    const int32_t *__restrict__ col,
                                                    const int32_t *__restrict__ heavy,
                                                    const int64_t *__restrict__ seg_ptr, int64_t nh,
                                                    int64_t nsegs, float *__restrict__ hsum,
                                                    int64_t ldh) {
  constexpr int GPB = 256 / LPR;
  const int li = threadIdx.x % LPR;
  const int gi = threadIdx.x / LPR;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu
                                     : (((1u << LPR) - 1u) << ((threadIdx.x % 32) / LPR * LPR));
  const int c = blockIdx.y * (LPR * 4) + li * 4;
  const bool active = c < p.cols;
  int64_t sidx = (int64_t)blockIdx.x * GPB + gi;
  if (sidx >= nsegs) return;
  // heavy row owning this segment: largest h with seg_ptr[h] <= sidx
  int64_t lo = 0, hi = nh - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (seg_ptr[mid] <= sidx) lo = mid; else hi = mid - 1;
  }
  int64_t h = lo;
  int u = heavy[h];
  int64_t rb = rowptr[u], re = rowptr[u + 1];
  int64_t e0 = rb + (sidx - seg_ptr[h]) * kHeavySeg;
  int64_t e1 = min(e0 + (int64_t)kHeavySeg, re);
  float4 acc = gather_sum<LPR, SCOL>(col, e0, e1, p.X, p.ldx, c, active, p.s_col, li, gmask);
  if (active) {
    float *dst = hsum + h * ldh + c;
    atomicAdd(reinterpret_cast<float4 *>(dst), acc);
  }
}

template <int LPR, bool SCOL>
__global__ void __launch_bounds__(256) k_spmm_rows(SpmmArgs p, const int64_t *__restrict__ rowptr,
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
    float4 acc;
    if (dg > kLightCap) {
      // heavy row: partial sums were reduced by k_spmm_heavy
      int64_t lo = 0, hi = nh - 1;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (heavy[mid] < u) lo = mid + 1; else hi = mid;
      }
      acc = active ? *reinterpret_cast<const float4 *>(hsum + lo * ldh + c)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      acc = gather_sum<LPR, SCOL>(col, e0, e1, p.X, p.ldx, c, active, p.s_col, li, gmask);
    }
    if (!active) continue;
    const float s = p.coef * row_scale(dg, p.a);
    float4 y = make_float4(s * acc.x, s * acc.y, s * acc.z, s * acc.w);
    if (p.prev) {
      float4 pv = *reinterpret_cast<const float4 *>(p.prev + u * p.ldp + c);
      y = f4_fma(p.beta, pv, y);
    }
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
      float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p.acc_in && p.acc_scale != 0.f)
        a0 = *reinterpret_cast<const float4 *>(p.acc_in + u * p.ldai + c);
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

template <int LPR, bool SCOL>
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
    NM_LAUNCH(c, "spmm_heavy", k_spmm_heavy<LPR, SCOL><<<gh, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.heavy, g.heavy_seg_ptr,
                                                      g.n_heavy, g.n_heavy_segs, hsum, ldh));
  }
  // rows per group: enough blocks for ~16 resident 256-thread blocks per SM
  int64_t row_blocks = ceil_div(g.n, GPB);
  int64_t cap = (int64_t)c.num_sms * 64;
  dim3 grid((unsigned)std::min<int64_t>(row_blocks, cap), chunks);
  NM_LAUNCH(c, "spmm_rows", k_spmm_rows<LPR, SCOL><<<grid, 256, 0, c.stream>>>(p, g.rowptr, g.col, g.n, g.heavy, g.n_heavy,
                                                     hsum.p, ldh));
}

void spmm(Ctx &c, const Graph &g, const SpmmArgs &p) {
  NM_REQUIRE(p.cols > 0 && p.ldx % 4 == 0 && p.ldy % 4 == 0, "spmm: ld must be a multiple of 4");
  NM_REQUIRE(((uintptr_t)p.X & 15) == 0 && (!p.Y || ((uintptr_t)p.Y & 15) == 0),
             "spmm: buffers must be 16-byte aligned");
  if (g.n == 0) return;
  if (p.s_col) spmm_impl<8, true>(c, g, p);
  else spmm_impl<8, false>(c, g, p);
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
