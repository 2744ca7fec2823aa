// tc_gemm.cu — tall-skinny dense contractions on the 5th-gen tensor cores
// (Gram matrices of CholeskyQR / Rayleigh–Ritz / Eq. 3, and the n×c · c×c
// products Q = Y R⁻¹, U = Q Û, F·C, E = Q Û √Σ of Alg. 2 / 4 / 5).
//
// Precision: 3xTF32.  An fp32 operand x is used as hi = x (the tensor core
// reads the top 19 bits, i.e. trunc_tf32(x)) and lo = x − trunc_tf32(x)
// (exact in fp32), and C = A_hi·B_hi + A_hi·B_lo + A_lo·B_hi is accumulated
// in fp32 TMEM by tcgen05.mma.kind::tf32 (dropped lo·lo term ~2^-21 relative).
//
// Both kernels are warp-specialised and TMA-fed (one CTA per SM, 192 threads):
//   warp 0      TMA producer: cp.async.bulk.tensor 2-D boxes, SWIZZLE_128B,
//               into an S-stage ring guarded by mbarriers (expect_tx);
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; commits
//               release ring slots (tcgen05.commit → mbarrier);
//   warps 2-5   "workers": compute the lo parts of each staged chunk in shared
//               memory (generic proxy → fence.proxy.async → mbarrier) and run
//               the epilogue (tcgen05.ld; warp w owns TMEM lanes 32·(w%4)..+31).
//
// Gram  G = Aᵀ diag(w) B over the n rows: the row-major n×c block is the
//   contraction (K) dimension, so chunks of BK rows × 32 columns are loaded
//   as-is and fed to the MMA as MN-major operands (no transposition): a
//   column block of 32 fp32 = one 128-B swizzle row, 8 rows = one 1-KB atom.
//   One CTA reduces a K-slab ("chain") of rows into all output tiles it owns
//   (Σ widths ≤ 512 TMEM columns), then writes an fp32 partial (units stored
//   column-major: coalesced stores); partials are summed in fp64 by a
//   deterministic reduction.  Exact chains are kept short (≈2k rows) because
//   the tensor core's fp32 accumulation truncates.  A tf32-only Gram without
//   row weights has nothing to prepare per chunk: the MMA issuer consumes the
//   TMA stage directly.  The issue loop reads host-computed per-unit
//   constants from the parameter space (uniform datapath, ~15 instructions
//   per MMA); with them in registers the issuer, not the tensor core, was the
//   bottleneck.
// GEMM  C = diag(rs)·A·B (B small, fp64 on input): persistent over 128-row
//   tiles of A (K-major operand straight from the row-major block); Bᵀ hi/lo
//   are prepared once in fp32 and streamed per K-chunk from L2.  With
//   tri_upper (B = R⁻¹ upper triangular) K-chunk kb only touches output
//   columns ≥ 32·kb, halving MMA work.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"

#ifdef TC_PROF
__device__ unsigned long long g_tcprof[1024 * 8];
#define TCP_T0() const unsigned long long _t0 = clock64()
#define TCP_ADD(slot) atomicAdd(&g_tcprof[(blockIdx.x % 1024) * 8 + (slot)], clock64() - _t0)
#else
#define TCP_T0()
#define TCP_ADD(slot)
#endif
namespace netmfp {
namespace tc {

// ===========================================================================
// Gram
// ===========================================================================
constexpr int kMaxUnits = 12;
struct GUnit {
  int mblk;   // first 32-col block of A forming the 128-row M tile (4 blocks)
  int nblk;   // first 32-col block of B for this unit's N range
  int nw;     // N width (multiple of 16, <= 256)
  int tcol;   // TMEM column of the accumulator
  int64_t off;  // float offset of the unit inside one chain's partial
};
struct GramP {
  int64_t n;        // rows (K extent)
  int64_t kslab;    // rows per chain (multiple of BK)
  int na_blk, nb_blk;  // 32-col blocks staged of A and (if !sym) B
  int nunits;
  GUnit u[kMaxUnits];
  int a3d, b3d;     // operand loaded as one 3-D box {32, BK, nblk} (ld covers all blocks)
  uint32_t tcols;   // TMEM allocation
  int stages;
  const float *wrow;    // optional per-row weights (d^-wexp, or its square root applied to both sides if sym)
  int64_t part_stride;  // floats per chain partial
  float *part;
  // issue constants per unit (host-computed so the MMA issuer reads them from
  // the parameter space with a uniform index: no per-MMA register moves)
  uint32_t uao[kMaxUnits], ubo[kMaxUnits], utc[kMaxUnits], uid[kMaxUnits];
  int exact;            // 1: 3xTF32 (A_hi B_hi + A_hi B_lo + A_lo B_hi); 0: A_hi B_hi only (no lo parts)
};

// position in an S-slot ring: slot and how many times it was used before
// (advanced incrementally: a 64-bit g % S / g / S per chunk cost each role
// a software division on its issue path)
struct RingPos {
  int s = 0;
  int use = 0;
  __device__ __forceinline__ void next(int S) {
    if (++s == S) {
      s = 0;
      ++use;
    }
  }
};
template <int BK, bool SYM, bool EXACT>
__global__ void __launch_bounds__(NT, 1) k_gram_tc(const __grid_constant__ CUtensorMap tmA,
                                                   const __grid_constant__ CUtensorMap tmB, const GramP p) {
  grid_dep_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = align1024(smem_raw);
  constexpr int BLK = BK * 128;  // bytes of one 32-col block of BK rows
  const int nblk = p.na_blk + (SYM ? 0 : p.nb_blk);
  const int stage_bytes = (EXACT ? 2 : 1) * nblk * BLK;  // raw (+ lo)
  const int S = p.stages;
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + S * stage_bytes + 3 * BLK);
  uint64_t *full = bars, *split = bars + S, *empty = bars + 2 * S, *done = bars + 3 * S;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 3 * S + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chain = blockIdx.x;
  const int64_t r0 = chain * p.kslab;
  const int64_t r1 = min(r0 + p.kslab, p.n);
  const int nk = (int)((r1 - r0 + BK - 1) / BK);
  // nothing to prepare per chunk (no lo parts, no row weights): the MMA
  // issuer consumes the TMA-filled stage directly
  const bool direct = !EXACT && !p.wrow;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], kWorkers);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      if (!SYM) tma_prefetch_desc(&tmB);
      RingPos rg;
      for (int kc = 0; kc < nk; ++kc, rg.next(S)) {
        const int s = rg.s, use = rg.use;
        {
          TCP_T0();
          if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
          TCP_ADD(0);
        }
        uint8_t *st = base + s * stage_bytes;
        mbar_expect_tx(&full[s], (uint32_t)(nblk * BLK));
        const int row = (int)(r0 + (int64_t)kc * BK);
        if (p.a3d)
          tma_load_3d(st, &tmA, 0, row, 0, &full[s]);
        else
          for (int b = 0; b < p.na_blk; ++b) tma_load_2d(st + b * BLK, &tmA, b * 32, row, &full[s]);
        if (!SYM) {
          if (p.b3d)
            tma_load_3d(st + p.na_blk * BLK, &tmB, 0, row, 0, &full[s]);
          else
            for (int b = 0; b < p.nb_blk; ++b) tma_load_2d(st + (p.na_blk + b) * BLK, &tmB, b * 32, row, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp (uniform addresses), one elected lane issues
      RingPos rg;
      for (int kc = 0; kc < nk; ++kc, rg.next(S)) {
        const int s = rg.s, use = rg.use;
        {
          TCP_T0();
          mbar_wait(direct ? &full[s] : &split[s], (uint32_t)(use & 1));
          if (lane == 0) TCP_ADD(2);
        }
        TCP_T0();
        tc_fence_after();
        if (elect_one()) {
          const uint32_t raw = smem_u32(base + s * stage_bytes);
          const uint32_t lo = raw + nblk * BLK;
          const uint32_t braw = SYM ? raw : raw + p.na_blk * BLK;
          const uint32_t blo = SYM ? lo : lo + p.na_blk * BLK;
          // descriptors once per chunk; per unit / K step only the address field moves
          const uint64_t dA = make_desc_mn32(raw, BLK), dAl = make_desc_mn32(lo, BLK);
          const uint64_t dB = make_desc_mn32(braw, BLK), dBl = make_desc_mn32(blo, BLK);
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t ko = ks * (1024 >> 4);
            const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
#pragma unroll 1
            for (int ui = 0; ui < p.nunits; ++ui) {
              const uint32_t d = tmem + p.utc[ui], id = p.uid[ui];
              const uint32_t ao = p.uao[ui] + ko, bo = p.ubo[ui] + ko;
              mma_tf32(d, dA + ao, dB + bo, id, acc0);
              if (EXACT) {
                mma_tf32(d, dA + ao, dBl + bo, id, 1u);
                mma_tf32(d, dAl + ao, dB + bo, id, 1u);
              }
            }
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
        if (lane == 0) TCP_ADD(5);
      }
      if (elect_one()) mma_commit(done);
      __syncwarp();
    }
  } else {
    // workers: lo split (+ row weights) for every chunk, then the epilogue
    const int wt = threadIdx.x - 64;  // 0..127
    const int q = warp & 3;
    RingPos rg;
    for (int kc = 0; kc < (direct ? 0 : nk); ++kc, rg.next(S)) {
      const int s = rg.s, use = rg.use;
      const int64_t row0 = r0 + (int64_t)kc * BK;
      // a worker's float4s i = wt, wt + kWorkers, … fall on at most two rows
      // of the chunk (ra, rb): their weights are loaded before the wait, not
      // one dependent global load per float4 (ncu: ~30% of the weighted
      // Gram's stall samples)
      static_assert((BLK / 16) % kWorkers == 0 || (2 * kWorkers) % (BLK / 16) == 0, "row pattern");
      const int ra = (wt % (BLK / 16)) / 8, rb = ((wt + kWorkers) % (BLK / 16)) / 8;
      float wa = 0.f, wb = 0.f;
      if (p.wrow) {
        if (row0 + ra < p.n) wa = __ldg(p.wrow + row0 + ra);
        if (row0 + rb < p.n) wb = __ldg(p.wrow + row0 + rb);
      }
      {
        TCP_T0();
        mbar_wait(&full[s], (uint32_t)(use & 1));
        if (wt == 0) TCP_ADD(3);
      }
      TCP_T0();
      uint8_t *raw = base + s * stage_bytes;
      uint8_t *lo = raw + nblk * BLK;
      const int n16 = nblk * BLK / 16;
      for (int i = wt; i < n16; i += kWorkers) {
        float4 v = reinterpret_cast<float4 *>(raw)[i];
        if (p.wrow) {
          const int blk = i / (BLK / 16);
          const int r = (i % (BLK / 16)) / 8;  // row inside the chunk (128-B rows): ra or rb
          if (SYM || blk < p.na_blk) {
            const float w = r == ra ? wa : wb;
            v.x *= w; v.y *= w; v.z *= w; v.w *= w;
            reinterpret_cast<float4 *>(raw)[i] = v;
          }
        }
        if (EXACT) {
          float4 l;
          l.x = v.x - tf32_trunc(v.x);
          l.y = v.y - tf32_trunc(v.y);
          l.z = v.z - tf32_trunc(v.z);
          l.w = v.w - tf32_trunc(v.w);
          reinterpret_cast<float4 *>(lo)[i] = l;
        }
      }
      fence_async_smem();
      mbar_arrive(&split[s]);
      if (wt == 0) TCP_ADD(6);
    }
    // epilogue: TMEM lanes 32q..32q+31 = rows of every unit's 128-row M tile
    {
      TCP_T0();
      mbar_wait(done, 0);
      if (wt == 0) TCP_ADD(4);
    }
    tc_fence_after();
    const int r = 32 * q + lane;
    float *dst0 = p.part + chain * p.part_stride;
    for (int ui = 0; ui < p.nunits; ++ui) {
      const GUnit &u = p.u[ui];
      float *dst = dst0 + u.off + r;  // column-major unit: lanes write consecutive rows
      for (int c = 0; c < u.nw; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(u.tcol + c), v);
#pragma unroll
        for (int i = 0; i < 16; ++i) __stcs(dst + (int64_t)(c + i) * 128, nk == 0 ? 0.f : v[i]);
      }
    }
    (void)wt;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, p.tcols);
}

// partial sums over chain groups: tmp[g][i*b+j] = Σ_{chains in g} part(i, j)
struct GramRed {
  int nunits;
  GUnit u[kMaxUnits];
  int64_t a, b;
  bool sym;
  int64_t nchain, part_stride;
};

// G = Σ_chains partials, one block per 128 consecutive partial positions (a
// partial unit is stored column-major, position = off + 128·col + row, so the
// epilogue's stores and these loads are coalesced); warp w sums chains
// w, w+8, … in a fixed order and the 8 warp sums are added in warp order
// (deterministic).  Symmetric: only i <= j is reduced and mirrored.
constexpr int kRedWarps = 8;
__global__ void __launch_bounds__(32 * kRedWarps) k_gram_reduce(const float *__restrict__ part, GramRed R,
                                                               double *__restrict__ G, int64_t ldg) {
  grid_dep_enter();
  // 128 positions per block, 4 per lane (16-B loads); warp w sums chains
  // w, w+8, … in order, the 8 warp sums are added in warp order
  __shared__ double red[kRedWarps][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p4 = blockIdx.x * 128LL + 4 * lane;  // part_stride is a multiple of 4
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  if (p4 < R.part_stride) {
    const float *src = part + p4;
    int64_t c = warp;
    for (; c + kRedWarps < R.nchain; c += 2 * kRedWarps) {
      const float4 a = __ldg(reinterpret_cast<const float4 *>(src + c * R.part_stride));
      const float4 b = __ldg(reinterpret_cast<const float4 *>(src + (c + kRedWarps) * R.part_stride));
      s[0] += (double)a.x; s[1] += (double)a.y; s[2] += (double)a.z; s[3] += (double)a.w;
      s[0] += (double)b.x; s[1] += (double)b.y; s[2] += (double)b.z; s[3] += (double)b.w;
    }
    if (c < R.nchain) {
      const float4 a = __ldg(reinterpret_cast<const float4 *>(src + c * R.part_stride));
      s[0] += (double)a.x; s[1] += (double)a.y; s[2] += (double)a.z; s[3] += (double)a.w;
    }
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) red[warp][4 * lane + t] = s[t];
  __syncthreads();
  if (threadIdx.x >= 128) return;
  const int64_t pos = blockIdx.x * 128LL + threadIdx.x;
  if (pos >= R.part_stride) return;
  double sum = 0.0;
#pragma unroll
  for (int w = 0; w < kRedWarps; ++w) sum += red[w][threadIdx.x];
  for (int ui = 0; ui < R.nunits; ++ui) {
    const GUnit &u = R.u[ui];
    const int64_t loc = pos - u.off;
    if (loc < 0 || loc >= 128LL * u.nw) continue;
    const int64_t i = (int64_t)u.mblk * 32 + loc % 128, j = (int64_t)u.nblk * 32 + loc / 128;
    if (i >= R.a || j >= R.b) return;
    if (!R.sym) {
      G[i * ldg + j] = sum;
    } else if (i <= j) {
      G[i * ldg + j] = sum;
      G[j * ldg + i] = sum;
    }
    return;
  }
}

// ===========================================================================
// tall GEMM  C = diag(rs) · A · B
// ===========================================================================
struct GemmP {
  int64_t n;      // rows of A / C
  int K;          // contraction length
  int nk;         // K chunks of 32
  int ntot;       // MMA N total (multiple of 16)
  int nh, hr;     // output columns split into nh parts of hr (multiple of 32, <= 192) columns
  int c16;        // output columns rounded up to 16 (the last part is c16 - (nh-1) hr wide)
  int order;      // item order (item_of)
  int skip;       // triangular B: skip the K chunks a part does not need
  int bexact;     // 1: A_hi B_hi + A_hi B_lo + A_lo B_hi; 0: B rounded to tf32, A_hi B + A_lo B
  int tri;        // B upper triangular: chunk kb touches columns >= 32 kb
  int64_t nitems; // (M tile, part) work items
  int stages;     // shared-memory ring (A raw + Bᵀ part)
  int astages;    // TMEM A stages (hi + lo, 64 columns each)
  float *C;
  int64_t ldc;
  int64_t ccols;  // valid output columns
  const int32_t *deg;
  float rexp;
};

// items = (M tile t, column part h), h fastest so that both parts of a tile
// read the same A rows back to back (the second time from L2).  The A tile
// goes to TMEM (hi and lo parts written by 4 "split" warps with tcgen05.st),
// so the MMAs (kind::tf32, A from TMEM) only read Bᵀ from shared memory; every
// item accumulates into one of two TMEM buffers and 4 separate epilogue warps
// drain the previous one while the next item's MMAs run.
// TMEM columns: acc[0] [0, hr), acc[1] [hr, 2hr), A stage s [2hr + 64s, +64).
constexpr int NTG = 320;  // 10 warps: TMA, MMA, 4 split, 4 epilogue
// K chunks part h reads: all, or (upper-triangular B) the chunks whose rows k
// can be <= the part's last column, 32 kc < pc1
// k-th item of this CTA (it = t * nh + h), or -1 when done.  order 0: items
// round-robin with the part fastest (the parts of a tile run at the same time
// on neighbouring CTAs: A is fetched once); order 1: part-major, every CTA
// works on the same part (the same Bᵀ chunks) at the same time.
__device__ __forceinline__ int64_t item_of(const GemmP &p, int64_t k) {
  const int64_t q = blockIdx.x + k * gridDim.x;
  if (q >= p.nitems) return -1;
  if (p.order == 0) return q;
  const int nt = (int)(p.nitems / p.nh);
  return (int64_t)((int)q % nt) * p.nh + (int)q / nt;
}
__device__ __forceinline__ int part_chunks(const GemmP &p, int h) {
  return (p.tri && p.skip) ? min(p.nk, (min(h * p.hr + p.hr, p.c16) + 31) / 32) : p.nk;
}
__global__ void __launch_bounds__(NTG, 1) k_gemm_tc(const __grid_constant__ CUtensorMap tmA,
                                                    const __grid_constant__ CUtensorMap tmBh,
                                                    const __grid_constant__ CUtensorMap tmC, const GemmP p) {
  grid_dep_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = align1024(smem_raw);
  constexpr int ABYTES = 128 * 128;  // 128 rows × 32 fp32 (raw, SWIZZLE_128B)
  const int bbytes = p.hr * 128;     // one part of Bᵀ (hi or lo)
  const int stage_bytes = ABYTES + (p.bexact ? 2 : 1) * bbytes;  // Bᵀ lo only for the exact product
  const int S = p.stages;
  // epilogue staging: 4 warps × 2 buffers × (32 rows × 128 B, SWIZZLE_128B)
  uint8_t *stg = base + S * stage_bytes;  // stage_bytes is a multiple of 1024
  uint64_t *bars = reinterpret_cast<uint64_t *>(stg + 4 * 2 * 4096);
  uint64_t *full = bars, *split = bars + S, *empty = bars + 2 * S;
  uint64_t *done = bars + 3 * S, *tfree = bars + 3 * S + 2;
  const int ST = p.astages;
  uint64_t *aempty = bars + 3 * S + 4;  // TMEM A stage free (MMA done reading it)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 3 * S + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], kWorkers);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&done[b], 1);
      mbar_init(&tfree[b], kWorkers);
    }
    for (int b = 0; b < ST; ++b) mbar_init(&aempty[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tA = tmem + (uint32_t)(2 * p.hr);

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmBh);
      RingPos rg;
      for (int64_t kq = 0, it = item_of(p, 0); it >= 0; ++kq, it = item_of(p, kq)) {
        const int64_t t = (int)it / p.nh;  // items < 2^31
        const int h = (int)it % p.nh;
        const int nkp = part_chunks(p, h);
        for (int kc = 0; kc < nkp; ++kc, rg.next(S)) {
          const int s = rg.s;
          const int use = rg.use;
          if (use > 0) {
            TCP_T0();
            mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
            TCP_ADD(0);
          }
          uint8_t *st = base + s * stage_bytes;
          mbar_expect_tx(&full[s], (uint32_t)(ABYTES + (p.bexact ? 2 : 1) * bbytes));
          tma_load_2d(st, &tmA, kc * 32, (int)(t * 128), &full[s]);
          tma_load_4d(st + ABYTES, &tmBh, 0, 0, h, 2 * kc, &full[s]);  // hi (and lo) parts
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp runs the loop (uniform addresses); one elected lane issues
      RingPos rg, ra;
      int64_t ic = 0;
      for (int64_t kq = 0, it = item_of(p, 0); it >= 0; ++kq, it = item_of(p, kq), ++ic) {
        const int h = (int)it % p.nh;
        const int buf = (int)(ic & 1);
        const int64_t use_b = ic >> 1;
        if (use_b > 0) {
          TCP_T0();
          mbar_wait(&tfree[buf], (uint32_t)((use_b - 1) & 1));
          TCP_ADD(1);
        }
        tc_fence_after();
        const int pc0 = h * p.hr, pc1 = min(pc0 + p.hr, p.c16);  // this part's output columns
        const int nkp = part_chunks(p, h);
        for (int kc = 0; kc < nkp; ++kc, rg.next(S), ra.next(ST)) {
          const int s = rg.s;
          const int use = rg.use;
          {
            TCP_T0();
            mbar_wait(&split[s], (uint32_t)(use & 1));
            if (lane == 0) TCP_ADD(2);
          }
          tc_fence_after();
          TCP_T0();
          const uint32_t bhi = smem_u32(base + s * stage_bytes) + ABYTES, blo = bhi + bbytes;
          const int sa = ra.s;
          const uint32_t ahi = tA + (uint32_t)(64 * sa), alo = ahi + 32;
          int c0 = pc0;
          if (p.tri) c0 = max(c0, (kc * 32) & ~15);
          if (c0 < pc1 && elect_one()) {
            const int N = pc1 - c0;
            const uint32_t idesc = make_idesc(N, 0, 0);
            const uint32_t d = tmem + (uint32_t)(buf * p.hr + (c0 - pc0));
            const uint32_t bo = (uint32_t)(c0 - pc0) * 128;
            // descriptors built once per chunk; a K step of 8 tf32 is +32 B = +2 in
            // the descriptor's address field (lean issue loop: the MMA issue rate,
            // not the tensor core, bounds kernels that rebuild them per MMA)
            const uint64_t dbh = make_desc(bhi + bo, 16, 1024), dbl = make_desc(blo + bo, 16, 1024);
            const uint32_t acc0 = (kc == 0) ? 0u : 1u;
            // every column is first touched by K-chunk 0 (tri: chunk kb only adds to
            // columns >= 32 kb), so chunk 0 / kstep 0 starts the sums
            if (p.bexact) {
              mma_tf32_ts(d, ahi, dbh, idesc, acc0);
              mma_tf32_ts(d, ahi, dbl, idesc, 1u);
              mma_tf32_ts(d, alo, dbh, idesc, 1u);
#pragma unroll
              for (int ks = 1; ks < 4; ++ks) {
                mma_tf32_ts(d, ahi + ks * 8, dbh + 2 * ks, idesc, 1u);
                mma_tf32_ts(d, ahi + ks * 8, dbl + 2 * ks, idesc, 1u);
                mma_tf32_ts(d, alo + ks * 8, dbh + 2 * ks, idesc, 1u);
              }
            } else {  // B = tf32(B): A's full fp32 against it (2 products)
              mma_tf32_ts(d, ahi, dbh, idesc, acc0);
              mma_tf32_ts(d, alo, dbh, idesc, 1u);
#pragma unroll
              for (int ks = 1; ks < 4; ++ks) {
                mma_tf32_ts(d, ahi + ks * 8, dbh + 2 * ks, idesc, 1u);
                mma_tf32_ts(d, alo + ks * 8, dbh + 2 * ks, idesc, 1u);
              }
            }
          }
          __syncwarp();
          if (elect_one()) {
            mma_commit(&empty[s]);
            mma_commit(&aempty[sa]);
          }
          __syncwarp();
          if (lane == 0) TCP_ADD(6);
        }
        if (elect_one()) mma_commit(&done[buf]);
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // split warps: this thread's A row (raw, from the swizzled smem tile) → TMEM hi / lo
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const int wt = threadIdx.x - 64;
    RingPos rg, ra;
    for (int64_t kq = 0, it = item_of(p, 0); it >= 0; ++kq, it = item_of(p, kq)) {
      const int h = (int)it % p.nh;
      const int nkp = part_chunks(p, h);
      for (int kc = 0; kc < nkp; ++kc, rg.next(S), ra.next(ST)) {
        const int s = rg.s;
        const int use = rg.use;
        {
          TCP_T0();
          mbar_wait(&full[s], (uint32_t)(use & 1));
          if (wt == 0) TCP_ADD(3);
        }
        const uint8_t *rowp = base + s * stage_bytes + r * 128;
        float hi[32], lo[32];
#pragma unroll
        for (int cch = 0; cch < 8; ++cch) {
          const float4 v = *reinterpret_cast<const float4 *>(rowp + ((cch ^ (r & 7)) << 4));
          hi[4 * cch] = v.x; hi[4 * cch + 1] = v.y; hi[4 * cch + 2] = v.z; hi[4 * cch + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) lo[i] = hi[i] - tf32_trunc(hi[i]);
        const int sa = ra.s;
        const int ua = ra.use;
        if (ua > 0) mbar_wait(&aempty[sa], (uint32_t)((ua - 1) & 1));  // MMAs done with this TMEM stage
        tc_fence_after();
        const uint32_t ta = tA + ((uint32_t)(32 * q) << 16) + (uint32_t)(64 * sa);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&split[s]);
      }
    }
  } else {
    // epilogue warps: acc[buf] rows (lane = row) → swizzled 32×32 staging tile
    // → one TMA store per tile (rows >= n and columns >= ccols are clipped
    // by the tensor map); the TMEM buffer is released as soon as it is read
    const int q = warp & 3;
    const int et = threadIdx.x - 192;
    uint8_t *myst = stg + q * 2 * 4096;
    int nst = 0;  // stores issued by this warp (staging buffer = nst & 1)
    int64_t ic = 0;
    for (int64_t kq = 0, it = item_of(p, 0); it >= 0; ++kq, it = item_of(p, kq), ++ic) {
      const int64_t t = (int)it / p.nh;  // items < 2^31
      const int h = (int)it % p.nh;
      const int buf = (int)(ic & 1);
      // the row's degree scale is loaded before waiting for the accumulator
      // (its global load latency sat on the epilogue's path, ncu)
      const int64_t r0 = t * 128 + 32 * q;
      const int64_t row = r0 + lane;
      float sc = 1.f;
      if (p.deg && row < p.n) sc = deg_pow_dev(p.deg, row, p.rexp);
      {
        TCP_T0();
        mbar_wait(&done[buf], (uint32_t)((ic >> 1) & 1));
        if (et == 0) TCP_ADD(4);
      }
      TCP_T0();
      tc_fence_after();
      const int pc0 = h * p.hr;
      const int nblk = (min(p.hr, p.c16 - pc0) + 31) / 32;  // hr is a multiple of 32
      for (int cb = 0; cb < nblk; ++cb) {
        uint32_t v[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * p.hr + 32 * cb);
        tmem_ld32_nowait(ta, v);
        tmem_wait_ld();
        if (cb + 1 == nblk) {  // accumulator fully read: hand it back to the MMA warp
          tc_fence_before();
          mbar_arrive(&tfree[buf]);
        }
        uint8_t *sb = myst + (nst & 1) * 4096;
        if (nst >= 2) {  // the store that last used this buffer has finished reading it
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
        }
        uint8_t *rowp = sb + lane * 128;
#pragma unroll
        for (int cch = 0; cch < 8; ++cch) {
          float4 o;
          o.x = sc * __uint_as_float(v[4 * cch]);
          o.y = sc * __uint_as_float(v[4 * cch + 1]);
          o.z = sc * __uint_as_float(v[4 * cch + 2]);
          o.w = sc * __uint_as_float(v[4 * cch + 3]);
          *reinterpret_cast<float4 *>(rowp + ((cch ^ (lane & 7)) << 4)) = o;
        }
        fence_proxy_async_smem();
        __syncwarp();
        // (parts are multiples of 32 columns except the last, whose columns
        // past c16 are >= ccols and clipped by the tensor map)
        if (lane == 0) {
          tma_store_2d(&tmC, sb, pc0 + 32 * cb, (int)r0);
          bulk_commit();
        }
        ++nst;
      }
      if (et == 0) TCP_ADD(5);
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace tc

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    NM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) throw Error(NETMFP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 2-D fp32 row-major [rows][cols] (row stride ld floats), box {box_cols, box_rows}:
// SWIZZLE_128B (K-major, 32 fp32 per row), SWIZZLE_128B_ATOM_32B (MN-major
// tf32) or SWIZZLE_64B (K-major, 16 fp32 per row)
CUtensorMap make_map(const float *p, int64_t rows, int64_t cols, int64_t ld, int box_rows, MapSwizzle sw,
                     int box_cols) {
  NM_REQUIRE(((uintptr_t)p & 15) == 0 && ld % 4 == 0, "tensor map: 16-byte aligned base and ld % 4 == 0 required");
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(p), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           sw == SW128_32B ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                           : sw == SW64    ? CU_TENSOR_MAP_SWIZZLE_64B
                                           : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(NETMFP_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// 2-D fp16 row-major [rows][cols] (row stride ld elements), box {box_cols, box_rows}, SWIZZLE_128B
CUtensorMap make_map_f16(const void *p, int64_t rows, int64_t cols, int64_t ld, int box_rows, int box_cols) {
  NM_REQUIRE(((uintptr_t)p & 15) == 0 && ld % 8 == 0, "tensor map (fp16): 16-byte aligned base and ld % 8 == 0 required");
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(p), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(NETMFP_ERR_CUDA, "cuTensorMapEncodeTiled (fp16) failed: " + std::to_string((int)r));
  return m;
}

CUtensorMap make_map_nd(const float *p, int rank, const int64_t *dims, const int64_t *strides_bytes, const int *box,
                        MapSwizzle sw) {
  NM_REQUIRE(((uintptr_t)p & 15) == 0 && rank >= 1 && rank <= 5, "tensor map: alignment / rank");
  CUtensorMap m;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = (cuuint64_t)dims[i];
    b[i] = (cuuint32_t)box[i];
    es[i] = 1u;
  }
  for (int i = 0; i + 1 < rank; ++i) {
    NM_REQUIRE(strides_bytes[i] % 16 == 0, "tensor map: strides must be multiples of 16 B");
    st[i] = (cuuint64_t)strides_bytes[i];
  }
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float *>(p), d, st, b, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           sw == SW128_32B ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                           : sw == SW64    ? CU_TENSOR_MAP_SWIZZLE_64B
                                           : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(NETMFP_ERR_CUDA, "cuTensorMapEncodeTiled (nd) failed: " + std::to_string((int)r));
  return m;
}

static uint32_t tmem_cols_for(int cols) {
  uint32_t t = 32;
  while (t < (uint32_t)cols) t <<= 1;
  return t;
}

static constexpr size_t kSmemMax = 227 * 1024;
// An M tile reads 4 column blocks of A; when A has fewer blocks the last tile
// reads past its region (into B / lo / the next stage: finite data that only
// feeds output rows >= a, which are never reduced).  The ring is followed by
// this many spare blocks so the last stage's over-read stays in bounds.
static constexpr int kPadBlocks = 3;

template <int BK, bool SYM>
static void launch_gram(Ctx &c, const CUtensorMap &ma, const CUtensorMap &mb, tc::GramP &p, int64_t nchain,
                        int ngroup_units_offset) {
  (void)ngroup_units_offset;
  const int nblk = p.na_blk + (SYM ? 0 : p.nb_blk);
  const size_t stage = (size_t)(p.exact ? 2 : 1) * nblk * BK * 128;
  for (int ui = 0; ui < p.nunits; ++ui) {
    p.uao[ui] = (uint32_t)(p.u[ui].mblk * BK * 128) >> 4;
    p.ubo[ui] = (uint32_t)(p.u[ui].nblk * BK * 128) >> 4;
    p.utc[ui] = (uint32_t)p.u[ui].tcol;
    p.uid[ui] = tc::make_idesc(p.u[ui].nw, 1, 1);
  }
  auto kern = p.exact ? tc::k_gram_tc<BK, SYM, true> : tc::k_gram_tc<BK, SYM, false>;
  int S = (int)std::min<size_t>(6, (kSmemMax - 1024 - 256 - kPadBlocks * BK * 128) / stage);
  NM_REQUIRE(S >= 2, "tc_gram: too many columns for the staged chunk");
  p.stages = S;
  const size_t smem = 1024 + S * stage + kPadBlocks * BK * 128 + (3 * S + 2) * 8 + 16;
  smem_attr(tc::k_gram_tc<BK, SYM, true>, kSmemMax);
  smem_attr(tc::k_gram_tc<BK, SYM, false>, kSmemMax);
  NM_LAUNCH(c, "tc_gram", launch_pdl(c.stream, kern, (unsigned)nchain, tc::NT, smem, ma, mb, p));
}

__global__ void k_gram_wrow(const int32_t *__restrict__ deg, int64_t n, float e, float *__restrict__ w) {
  grid_dep_enter();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) w[i] = tc::deg_pow_dev(deg, i, e);
}

// G[a×b] (fp64, ldg) = Aᵀ diag(d^-wexp) B over the n rows
void tc_gram(Ctx &c, const Mat &A, const Mat &B, const int32_t *deg, float wexp, double *G, int64_t ldg, bool exact,
             bool sym_result) {
  using namespace tc;
  NM_REQUIRE(A.rows == B.rows, "tc_gram: row mismatch");
  const int64_t n = A.rows, a = A.cols, b = B.cols;
  if (n == 0) {
    NM_CUDA(cudaMemset2DAsync(G, ldg * 8, 0, b * 8, a, c.stream));
    return;
  }
  const bool sym = (A.p == B.p && A.cols == B.cols && A.ld == B.ld);
  // a symmetric result (same operand, or the caller says so) needs only the
  // upper block-triangle of output units; the reduction mirrors it
  const bool upper = sym || (sym_result && a == b);
  const int na_blk = (int)ceil_div(a, 32), nb_blk = (int)ceil_div(b, 32);
  // output units: M tiles of 128 rows (4 blocks of A), N ranges of <= 256 cols
  std::vector<GUnit> all;
  const int mt = (int)ceil_div(a, 128);
  for (int m = 0; m < mt; ++m) {
    const int n_lo = upper ? 4 * m : 0;  // upper block-triangle only
    const int n_hi = nb_blk;
    int ncols = (n_hi - n_lo) * 32;
    if (ncols <= 0) continue;
    const int parts = (ncols + 255) / 256;
    const int blks = n_hi - n_lo;
    int start = n_lo;
    for (int pi = 0; pi < parts; ++pi) {
      const int nb = (blks - (start - n_lo) + (parts - pi) - 1) / (parts - pi);
      all.push_back(GUnit{4 * m, start, nb * 32, 0, 0});
      start += nb;
    }
  }
  // global partial offsets, then pack units into groups of <= 512 TMEM columns
  int64_t total = 0;
  for (auto &u : all) {
    u.off = total;
    total += (int64_t)128 * u.nw;
  }
  NM_REQUIRE((int)all.size() <= kMaxUnits, "tc_gram: too many output units");
  std::vector<std::vector<GUnit>> groups;
  {
    std::vector<GUnit> cur;
    int w = 0;
    for (auto u : all) {
      if (w + u.nw > 512) {
        groups.push_back(cur);
        cur.clear();
        w = 0;
      }
      u.tcol = w;
      w += u.nw;
      cur.push_back(u);
    }
    if (!cur.empty()) groups.push_back(cur);
  }
  // chains: a multiple of the SM count, ~2k rows each (short TMEM chains)
  constexpr int BKs = 32, BKn = 16;
  const int BK = sym ? BKs : BKn;
  // (a tf32-only Gram is ~1e-3 accurate anyway: one chain per SM, fewer partials)
  const int64_t waves =
      exact ? std::max<int64_t>(1, (n + (int64_t)c.num_sms * 2048 - 1) / ((int64_t)c.num_sms * 2048)) : 1;
  int64_t nchain = std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * waves, ceil_div(n, BK)));
  const int64_t kslab = (ceil_div(n, nchain) + BK - 1) / BK * BK;
  nchain = ceil_div(n, kslab);
  // one 3-D box per operand when the row pitch covers every 32-column block
  // (the view then reads the ld padding of the last block: those columns only
  // feed output rows/cols >= a, b, which are never reduced)
  const bool a3d = A.ld >= 32 * na_blk, b3d = B.ld >= 32 * nb_blk;
  auto map3 = [&](const Mat &M, int nblk) {
    const int64_t dims[3] = {32, n, nblk};
    const int64_t str[2] = {M.ld * 4, 128};
    const int box[3] = {32, BK, nblk};
    return make_map_nd(M.p, 3, dims, str, box, SW128_32B);
  };
  CUtensorMap ma = a3d ? map3(A, na_blk) : make_map(A.p, n, a, A.ld, BK, SW128_32B);
  CUtensorMap mb = sym ? ma : (b3d ? map3(B, nb_blk) : make_map(B.p, n, b, B.ld, BK, SW128_32B));
  DBuf<float> part((size_t)nchain * total, c.stream);
  // per-row weights once (d^-wexp on A; sym: d^(-wexp/2) on both sides)
  DBuf<float> wrow;
  if (deg) {
    wrow.alloc(n, c.stream);
    NM_LAUNCH(c, "gram_wrow", launch_pdl(c.stream, k_gram_wrow, ceil_div(n, 256), 256, 0, deg, n, sym ? 0.5f * wexp : wexp, wrow.p));
  }
  for (auto &grp : groups) {
    GramP p{};
    p.n = n;
    p.kslab = kslab;
    p.na_blk = na_blk;
    p.nb_blk = sym ? 0 : nb_blk;
    p.nunits = (int)grp.size();
    int w = 0;
    for (int i = 0; i < p.nunits; ++i) {
      p.u[i] = grp[i];
      w += grp[i].nw;
    }
    p.tcols = tmem_cols_for(w);
    p.a3d = a3d ? 1 : 0;
    p.b3d = b3d ? 1 : 0;
    p.wrow = wrow.p;
    p.part_stride = total;
    p.part = part.p;
    p.exact = exact ? 1 : 0;
    if (sym)
      launch_gram<BKs, true>(c, ma, mb, p, nchain, 0);
    else
      launch_gram<BKn, false>(c, ma, mb, p, nchain, 0);
  }
  GramRed R{};
  R.nunits = (int)all.size();
  for (int i = 0; i < R.nunits; ++i) R.u[i] = all[i];
  R.a = a;
  R.b = b;
  R.sym = upper;
  R.nchain = nchain;
  R.part_stride = total;
  NM_LAUNCH(c, "tc_gram_reduce",
            launch_pdl(c.stream, k_gram_reduce, ceil_div(total, 128), 32 * kRedWarps, 0, part.p, R, G, ldg));
}

// Bᵀ for the tensor-core GEMM, zero padded to nrows × 32 nk:
// Bt[kc][part][j][kk] with part 0 = hi = tf32(B[32 kc + kk][j]) (round to
// nearest) and part 1 = lo = B - hi
__global__ void k_bt_split(const double *__restrict__ Bs, int64_t ldb, int64_t K, int64_t N, int64_t nrows, int64_t nk,
                           float *__restrict__ Bt) {
  grid_dep_enter();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= nk * nrows * 32) return;
  const int64_t kk = idx & 31, j = (idx >> 5) % nrows, kc = idx / (32 * nrows);
  const int64_t k = kc * 32 + kk;
  const double x = (j < N && k < K) ? Bs[k * ldb + j] : 0.0;
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"((float)x));
  const float h = __uint_as_float(r);
  float *base = Bt + kc * 2 * nrows * 32;
  base[j * 32 + kk] = h;
  base[nrows * 32 + j * 32 + kk] = (float)(x - (double)h);
}

// C[n×b] = rs ⊙ (A[n×a] · Bs[a×b])
static void tc_gemm_tall_impl(Ctx &c, const Mat &A, const double *Bs, int64_t ldb, int64_t bcols, const int32_t *deg,
                              float rexp, const Mat &C, bool tri, bool exact) {
  using namespace tc;
  const int64_t n = A.rows, K = A.cols;
  // output columns in nh parts of hr (multiple of 32, <= 192) so that two
  // accumulators and the TMEM A stages fit the 512 TMEM columns
  const int c16 = (int)((bcols + 15) / 16) * 16;
  const int nh = (c16 + 191) / 192;
  const int hr = ((c16 + nh - 1) / nh + 31) / 32 * 32;
  const int ntot = nh * hr;
  const int64_t nk = ceil_div(K, 32);
  DBuf<float> bt((size_t)nk * 2 * ntot * 32, c.stream);
  NM_LAUNCH(c, "bt_split", launch_pdl(c.stream, k_bt_split, ceil_div(nk * ntot * 32, 256), 256, 0, Bs, ldb, K, bcols, ntot, nk,
                                                                                             bt.p));
  CUtensorMap ma = make_map(A.p, n, K, A.ld, 128);
  const int64_t bdims[4] = {32, hr, nh, 2 * nk};
  const int64_t bstr[3] = {128, (int64_t)hr * 128, (int64_t)ntot * 128};
  const int bbox[4] = {32, hr, 1, exact ? 2 : 1};  // one part (hi + lo, or hi only) per box
  CUtensorMap mb = make_map_nd(bt.p, 4, bdims, bstr, bbox, SW128);
  GemmP p{};
  p.n = n;
  p.K = (int)K;
  p.nk = (int)nk;
  p.ntot = ntot;
  p.nh = nh;
  p.hr = hr;
  p.c16 = c16;
  p.tri = tri ? 1 : 0;
  p.nitems = ceil_div(n, 128) * nh;
  p.C = C.p;
  p.ldc = C.ld;
  p.ccols = bcols;
  p.deg = deg;
  p.rexp = rexp;
  const size_t staging = (size_t)4 * 2 * 4096;
  const size_t stage = (size_t)128 * 128 + (size_t)(exact ? 2 : 1) * hr * 128;  // a multiple of 1024
  const int S = (int)std::min<size_t>(6, (kSmemMax - 1024 - 256 - staging) / stage);
  const int ST = std::min(4, (512 - 2 * hr) / 64);
  NM_REQUIRE(S >= 2 && ST >= 2, "tc_gemm_tall: stage does not fit");
  p.stages = S;
  p.astages = ST;
  const size_t smem = 1024 + S * stage + staging + (3 * S + 10) * 8;
  smem_attr(k_gemm_tc, kSmemMax);
  // Parts of a tile side by side (order 0: the two CTAs working on a tile's
  // parts read its A rows once from HBM, the second time from L2), the
  // unneeded K chunks of triangular B skipped.  Triangular B with an odd grid:
  // every CTA alternates between the short and the long part, so neighbouring
  // CTAs stay within a few K chunks of each other; configs[2], tall GEMM per
  // embedding 2.91-3.06 -> 2.74-2.80 ms against part-major order (every CTA on
  // the same part: A read twice, 755 MB per n'×286 call instead of ~470).
  // NETMFP_GEMM_TRI_ORDER=1 restores part-major order for A/B measurements.
  p.bexact = exact ? 1 : 0;
  static const int tri_order = [] {
    const char *v = getenv("NETMFP_GEMM_TRI_ORDER");
    return v ? atoi(v) : 0;
  }();
  p.order = tri ? tri_order : 0;
  p.skip = tri ? 1 : 0;
  int64_t grid = std::min<int64_t>(p.nitems, c.num_sms);
  // triangular B, parts side by side: an odd grid alternates every CTA
  // between the short and the long part (an even one pins each CTA to one)
  if (tri && p.order == 0 && nh == 2 && grid % 2 == 0 && grid > 1) --grid;
  CUtensorMap mc = make_map(C.p, n, bcols, C.ld, 32, SW128, 32);
  NM_LAUNCH(c, "tc_gemm_tall", launch_pdl(c.stream, k_gemm_tc, (unsigned)grid, NTG, smem, ma, mb, mc, p));
}

void tc_gemm_tall(Ctx &c, const Mat &A, const double *Bs, int64_t ldb, int64_t bcols, const int32_t *deg, float rexp,
                  const Mat &C) {
  // column groups of <= 288 outputs
  for (int64_t c0 = 0; c0 < bcols; c0 += 288) {
    const int64_t w = std::min<int64_t>(288, bcols - c0);
    Mat Cg = C;
    Cg.p = C.p + c0;
    Cg.cols = w;
    tc_gemm_tall_impl(c, A, Bs + c0, ldb, w, deg, rexp, Cg, false, true);
  }
}

void tc_gemm_tall_tri(Ctx &c, const Mat &A, const double *Rinv, int64_t ldb, int64_t bcols, const int32_t *deg,
                      float rexp, const Mat &C, bool exact) {
  NM_REQUIRE(A.cols == bcols, "tc_gemm_tall_tri: square upper-triangular B");
  if (bcols <= 288) {
    tc_gemm_tall_impl(c, A, Rinv, ldb, bcols, deg, rexp, C, true, exact);
    return;
  }
  // wider: column groups of <= 288; group [c0, c0 + w) needs only the first
  // c0 + w rows of the upper-triangular B (the rest are zero)
  for (int64_t c0 = 0; c0 < bcols; c0 += 288) {
    const int64_t w = std::min<int64_t>(288, bcols - c0);
    Mat Ak = A, Cg = C;
    Ak.cols = c0 + w;
    Cg.p = C.p + c0;
    Cg.cols = w;
    tc_gemm_tall_impl(c, Ak, Rinv + c0, ldb, w, deg, rexp, Cg, false, exact);
  }
}

}  // namespace netmfp
