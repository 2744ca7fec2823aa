// sketch_tc.cu — rows a6/a7: the sketches of Alg. 4 without materialising the
// NetMF matrix (Eq. 5), on the tensor cores.
//
// A sparse-sign matrix Ψ (Alg. 3) has, in column c, z entries (row r_{c,t},
// sign s_{c,t}).  Eq. 5's sketch Y = f(M̂')Ψ with M̂' = scale·F C Fᵀ is then
//
//   Y[i, c] = Σ_{t<z} s_{c,t} · f(scale · (FC)_i · F_{r_{c,t}}ᵀ)              (Y mode)
//
// i.e. a GEMM of A = FC (n × k) against B = the h·z rows F_{r_{c,t}} laid out
// column group by column group, followed by a fixed segmented sum of z
// consecutive output columns.  The core sketch of Alg. 4 step 6 is the same
// with the row side gathered too:
//
//   Z[c', c] = Σ_{t'} s_{c',t'} Σ_t s_{c,t} f(scale · (FC)_{r_{c',t'}} · F_{r_{c,t}}ᵀ)   (Z mode)
//
// Group sizes are padded to zp = next power of two ≥ z with sign-0 dummy rows,
// so every group is an aligned run of zp columns (and, in Z mode, zp lanes).
// This needs neither the unique coordinate set p of Alg. 3 nor a scatter: the
// epilogue is f(·), one FFMA per element and a register / shuffle reduction.
//
// One CTA per SM, persistent over (128-row M tile, N-tile range) items:
//   warp 0      TMA: A chunk (128 rows × 32 fp32, SWIZZLE_128B) and the
//               B hi / lo chunks (256 rows × 32) of the current N tile, one
//               box each, issued by three lanes in parallel;
//   warp 1      tcgen05.mma 3xTF32 (A_hi·B_hi + A_hi·B_lo + A_lo·B_hi) into one
//               of two 256-column TMEM accumulators (double-buffered);
//   warps 2-3, 8-9  split the staged A chunk into lo parts (x − trunc_tf32(x));
//   warps 4-7   epilogue: tcgen05.ld, f(scale·x)·sign, segmented sums; Y mode
//               stages a row's 256/zp outputs per N tile in shared memory and
//               writes them as one contiguous run; Z mode reduces zp lanes
//               with shuffles and stores one value per (row group, col group).
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"

#include <algorithm>

#ifdef SK_PROF
__device__ unsigned long long g_skprof[148 * 8];
#define SKP_T0() const unsigned long long _t0 = clock64()
#define SKP_ADD(slot) atomicAdd(&g_skprof[blockIdx.x * 8 + (slot)], clock64() - _t0)
#else
#define SKP_T0()
#define SKP_ADD(slot)
#endif
namespace netmfp {
namespace tcs {

using namespace tc;

constexpr int THREADS = 320;
constexpr int NW = 256;           // N tile per accumulator
constexpr int BK = 32;             // K per stage (128-B swizzled rows)
constexpr int ABYTES = 128 * 128;  // A chunk: 128 rows × 32 fp32
constexpr int BBYTES = NW * 128;   // B chunk: NW rows × 32 fp32
constexpr int STAGE = 2 * ABYTES + 2 * BBYTES;
constexpr int S = 2;
constexpr int kSplit = 128;  // split threads (warps 2-3 and 8-9)
constexpr int kEpi = 128;   // epilogue threads (warps 4-7)

struct SkP {
  int64_t m;        // rows of A
  int k, nk;        // contraction length, K chunks
  int64_t ncols;    // N = h·zp
  int ntn;          // N tiles
  int64_t nmt;      // M tiles
  int nsplit;       // N-tile ranges per M tile (items = nmt × nsplit)
  int zp, lzp;      // group size (power of two) and log2
  int64_t h;        // output column groups
  float scale;
  int logmode;
  const uint32_t *neg_bits;  // per 32 columns: 1 = sign −1
  const uint32_t *val_bits;  // per 32 columns: 0 = padding (sign 0)
  int epi;                   // epilogue variant: zp·4 + zmode·2 + log1p
  const float *row_sign;  // m (Z mode) or null (Y mode)
  float *out;
  int64_t ldo;
};

// f(x) = trunc_log(x) = log(max(x, 1)) or log1p(max(x, 0))   [R4]
__device__ __forceinline__ float apply_f(float x, int logmode) {
  return logmode == 0 ? __logf(fmaxf(x, 1.f)) : log1pf(fmaxf(x, 0.f));
}

// One 128 × NW accumulator tile → f, signs, segmented sums (see file header).
// f is evaluated as ln2 · log2(max(scale x, 1)) (trunc_log) or log1p(max(scale x, 0)).
// Column signs come as bit masks (neg, valid) of the N tile, 32 columns a word.
// CW columns starting at column cbeg of the N tile (tb addresses column cbeg;
// cbeg is a multiple of 32 and of the group size)
template <int ZP, bool ZM, bool L1P, int CW = NW, bool VMASK = true>
__device__ __forceinline__ void epi_tile(const SkP &p, uint32_t tb, int nt, int64_t row, float rsign, int lane,
                                         float xs = 1.f, int cbeg = 0) {
  const int64_t j0 = (int64_t)nt * NW + cbeg;
  const int ncol = (int)min((int64_t)CW, p.ncols - j0);
  uint32_t neg[CW / 32], val[CW / 32];
#pragma unroll
  for (int w = 0; w < CW / 32; ++w) {
    neg[w] = __ldg(p.neg_bits + (j0 >> 5) + w);
    val[w] = __ldg(p.val_bits + (j0 >> 5) + w);
  }
  const float sc = p.scale * xs;
  constexpr float kLn2 = 0.69314718055994531f;
  float run = 0.f;
  float outs[16 / ZP > 0 ? 16 / ZP : 1];
#pragma unroll
  for (int cc = 0; cc < CW; cc += 16) {
    if (cc < ncol) {
      float x[16];
      tmem_ld16(tb + (uint32_t)cc, x);
      const uint32_t nb = (neg[cc >> 5] >> (cc & 16)) & 0xFFFFu;
      const uint32_t vb = (val[cc >> 5] >> (cc & 16)) & 0xFFFFu;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float v = L1P ? log1pf(fmaxf(sc * x[i], 0.f)) : __log2f(fmaxf(sc * x[i], 1.f));
        // VMASK = false: padding columns have all-zero B rows, so f(0) = 0 already
        if (VMASK) v = ((vb >> i) & 1u) ? v : 0.f;
        run += __uint_as_float(__float_as_uint(v) ^ ((nb << (31 - i)) & 0x80000000u));  // sign s_{c,t}
        if (((i + 1) % ZP) == 0 || (ZP > 16 && i == 15 && ((cc + 16) % ZP) == 0)) {
          const float res = L1P ? run : run * kLn2;
          run = 0.f;
          if (ZP <= 16) {
            outs[i / ZP] = res;
          } else {
            outs[0] = res;
          }
          if (ZM) {
            float w = outs[ZP <= 16 ? i / ZP : 0] * rsign;
#pragma unroll
            for (int o = 1; o < (ZP < 32 ? ZP : 32); o <<= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            const int64_t cg = (j0 + cc + i) / ZP;
            const int64_t rg = row / ZP;
            if ((lane & ((ZP < 32 ? ZP : 32) - 1)) == 0 && row < p.m && cg < p.h) {
              if (ZP <= 32)
                p.out[rg * p.ldo + cg] = w;
              else
                atomicAdd(p.out + rg * p.ldo + cg, w);  // 2 warps per group: a + b, order-free
            }
          }
        }
      }
      if (!ZM && row < p.m) {
        // this chunk's outputs: contiguous in the row
        if (ZP <= 16 || ((cc + 16) % ZP) == 0) {
          const int64_t cg0 = (j0 + cc + 16) / ZP - (ZP <= 16 ? 16 / ZP : 1);
          float *dst = p.out + row * p.ldo + cg0;
          const int nval = (int)min((int64_t)(ZP <= 16 ? 16 / ZP : 1), p.h - cg0);
          if (ZP <= 4 && nval == 16 / ZP) {
#pragma unroll
            for (int o = 0; o < 16 / ZP; o += 4)
              *reinterpret_cast<float4 *>(dst + o) = make_float4(outs[o], outs[o + 1], outs[o + 2], outs[o + 3]);
          } else if (ZP == 8 && nval == 2) {
            *reinterpret_cast<float2 *>(dst) = make_float2(outs[0], outs[1]);
          } else {
#pragma unroll
            for (int o = 0; o < (ZP <= 16 ? 16 / ZP : 1); ++o)
              if (o < nval) dst[o] = outs[o];
          }
        }
      }
    }
  }
}

template <int ZP, bool ZM, bool L1P>
__global__ void __launch_bounds__(THREADS, 1) k_sketch_tc(const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmBh,
                                                          const __grid_constant__ CUtensorMap tmBl, const SkP p) {
  grid_dep_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = align1024(smem_raw);
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + S * STAGE);
  uint64_t *full = bars, *split = bars + S, *empty = bars + 2 * S;
  uint64_t *done = bars + 3 * S, *tfree = bars + 3 * S + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 3 * S + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nitems = p.nmt * p.nsplit;
  const int per = (p.ntn + p.nsplit - 1) / p.nsplit;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], kSplit);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&done[b], 1);
      mbar_init(&tfree[b], kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // lanes 0-2 issue the stage's three boxes in parallel (a TMA issue blocks
    // the issuing thread for ~150-300 cycles regardless of the box size)
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmBh);
      tma_prefetch_desc(&tmBl);
    }
    int64_t g = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int64_t mt = it / p.nsplit;
      const int nt0 = (int)(it % p.nsplit) * per, nt1 = min(p.ntn, nt0 + per);
      for (int nt = nt0; nt < nt1; ++nt) {
        for (int kc = 0; kc < p.nk; ++kc, ++g) {
          const int s = (int)(g % S);
          const int64_t use = g / S;
          if (use > 0) {
            SKP_T0();
            mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
            if (lane == 0) SKP_ADD(0);
          }
          uint8_t *st = base + s * STAGE;
          if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(ABYTES + 2 * BBYTES));
          __syncwarp();
          if (lane == 0) tma_load_2d(st, &tmA, kc * BK, (int)(mt * 128), &full[s]);
          if (lane == 1) tma_load_2d(st + 2 * ABYTES, &tmBh, kc * BK, nt * NW, &full[s]);
          if (lane == 2) tma_load_2d(st + 2 * ABYTES + BBYTES, &tmBl, kc * BK, nt * NW, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp (uniform addresses), one elected lane issues
      int64_t g = 0, tcount = 0;
      for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int nt0 = (int)(it % p.nsplit) * per, nt1 = min(p.ntn, nt0 + per);
        for (int nt = nt0; nt < nt1; ++nt, ++tcount) {
          const int buf = (int)(tcount & 1);
          const int64_t use_b = tcount >> 1;
          if (use_b > 0) {
            SKP_T0();
            mbar_wait(&tfree[buf], (uint32_t)((use_b - 1) & 1));
            if (lane == 0) SKP_ADD(1);
          }
          tc_fence_after();
          const int64_t rem = p.ncols - (int64_t)nt * NW;
          const int N = (int)std::min<int64_t>(NW, (rem + 15) / 16 * 16);
          const uint32_t idesc = make_idesc(N, 0, 0);
          const uint32_t d = tmem + (uint32_t)(buf * NW);
          for (int kc = 0; kc < p.nk; ++kc, ++g) {
            const int s = (int)(g % S);
            const int64_t use = g / S;
            {
              SKP_T0();
              mbar_wait(&split[s], (uint32_t)(use & 1));
              if (lane == 0) SKP_ADD(2);
            }
            tc_fence_after();
            const bool leader = elect_one();
            const uint32_t ahi = smem_u32(base + s * STAGE), alo = ahi + ABYTES;
            const uint32_t bhi = alo + ABYTES, blo = bhi + BBYTES;
            const uint64_t dah = make_desc(ahi, 16, 1024), dal = make_desc(alo, 16, 1024);
            const uint64_t dbh = make_desc(bhi, 16, 1024), dbl = make_desc(blo, 16, 1024);
#pragma unroll
            for (int ks = 0; ks < BK / 8; ++ks) {
              const uint32_t acc0 = (kc == 0 && ks == 0) ? 0u : 1u;
              if (leader) {
                mma_tf32(d, dah + 2 * ks, dbh + 2 * ks, idesc, acc0);
                mma_tf32(d, dah + 2 * ks, dbl + 2 * ks, idesc, 1u);
                mma_tf32(d, dal + 2 * ks, dbh + 2 * ks, idesc, 1u);
              }
            }
            __syncwarp();
            if (leader) mma_commit(&empty[s]);
            __syncwarp();
          }
          if (elect_one()) mma_commit(&done[buf]);
          __syncwarp();
        }
      }
    }
  } else if (warp < 4 || warp >= 8) {
    // split warps: A lo parts
    const int st_id = warp < 4 ? threadIdx.x - 64 : threadIdx.x - 256 + 64;
    int64_t g = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int nt0 = (int)(it % p.nsplit) * per, nt1 = min(p.ntn, nt0 + per);
      for (int nt = nt0; nt < nt1; ++nt) {
        for (int kc = 0; kc < p.nk; ++kc, ++g) {
          const int s = (int)(g % S);
          const int64_t use = g / S;
          {
            SKP_T0();
            mbar_wait(&full[s], (uint32_t)(use & 1));
            if (st_id == 0) SKP_ADD(3);
          }
          float4 *raw = reinterpret_cast<float4 *>(base + s * STAGE);
          float4 *lo = raw + ABYTES / 16;
          for (int i = st_id; i < ABYTES / 16; i += kSplit) {
            const float4 x = raw[i];
            lo[i] = make_float4(x.x - tf32_trunc(x.x), x.y - tf32_trunc(x.y), x.z - tf32_trunc(x.z),
                                x.w - tf32_trunc(x.w));
          }
          fence_async_smem();
          mbar_arrive(&split[s]);
        }
      }
    }
  } else {
    // epilogue warps 4-7: TMEM lane quadrant q, row r of the M tile per thread
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const bool zmode = p.row_sign != nullptr;
    int64_t tcount = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int64_t mt = it / p.nsplit;
      const int nt0 = (int)(it % p.nsplit) * per, nt1 = min(p.ntn, nt0 + per);
      const int64_t row = mt * 128 + r;
      const float rsign = (zmode && row < p.m) ? __ldg(p.row_sign + row) : 1.f;
      for (int nt = nt0; nt < nt1; ++nt, ++tcount) {
        const int buf = (int)(tcount & 1);
        {
          SKP_T0();
          mbar_wait(&done[buf], (uint32_t)((tcount >> 1) & 1));
          if (r == 0) SKP_ADD(4);
        }
        tc_fence_after();
        SKP_T0();
        const uint32_t tb = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * NW);
        epi_tile<ZP, ZM, L1P>(p, tb, nt, row, rsign, lane);
        tc_fence_before();
        mbar_arrive(&tfree[buf]);
        if (r == 0) SKP_ADD(5);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// Y mode with fp16-split operands.  Both operands are pre-split in global
// memory: x·2^e = hi + lo with hi = fp16(x·2^e), lo = fp16(x·2^e − hi), the
// power-of-two scale 2^e per row of A (max |A_i| in [2^14, 2^15)) and one
// for all of B, so hi + lo carries ~22 significant bits like tf32 hi + lo,
// and C = A_hi·B_hi + A_hi·B_lo + A_lo·B_hi (tcgen05.mma.kind::f16, fp32
// accumulation) is within ~2^-22 relative of the fp32 product, as 3xTF32.
// An fp16 MMA does twice the K of a tf32 one in the same time, and with the
// split done once per operand no stage waits for split warps:
//   warp 0      TMA: A hi/lo (128 rows × 64 fp16), B hi/lo (NW rows × 64)
//   warp 1      tcgen05.mma kind::f16 ×3 per 16-deep K step
//   warps 2-9   epilogue, two warps per TMEM lane quadrant (warp % 4), each
//               on one half of the N tile's columns; the row's scale
//               2^-e_i · 2^-e_B folded into the f(scale·x) multiply (with the
//               MMA work halved, four epilogue warps were the bottleneck)
// ---------------------------------------------------------------------------
constexpr int HT = 320;
constexpr int kEpiH = 256;  // epilogue threads: warps 2-9, two per TMEM lane quadrant
constexpr int HBK = 64;                 // fp16 K per stage: one 128-B swizzled row
constexpr int HABYTES = 128 * 128;      // A hi (or lo) chunk
constexpr int HBBYTES = NW * 128;       // B hi (or lo) chunk
constexpr int HSTAGE = 2 * HABYTES + 2 * HBBYTES;
constexpr int HS = 2;
// kind::f16 (fp16 A, B), D = f32, M = 128, both K-major
__host__ __device__ constexpr uint32_t make_idesc_f16(int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

template <int ZP, bool ZM, bool L1P>
__global__ void __launch_bounds__(HT, 1) k_sketch_h(const __grid_constant__ CUtensorMap tmAh,
                                                    const __grid_constant__ CUtensorMap tmAl,
                                                    const __grid_constant__ CUtensorMap tmBh,
                                                    const __grid_constant__ CUtensorMap tmBl, const SkP p,
                                                    const float *__restrict__ rinv, const int *__restrict__ bexp) {
  grid_dep_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = align1024(smem_raw);
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + HS * HSTAGE);
  uint64_t *full = bars, *empty = bars + HS;
  uint64_t *done = bars + 2 * HS, *tfree = bars + 2 * HS + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * HS + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nitems = p.nmt * p.nsplit;
  const int per = (p.ntn + p.nsplit - 1) / p.nsplit;
  if (threadIdx.x == 0) {
    for (int s = 0; s < HS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&done[b], 1);
      mbar_init(&tfree[b], kEpiH);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmAh);
      tma_prefetch_desc(&tmAl);
      tma_prefetch_desc(&tmBh);
      tma_prefetch_desc(&tmBl);
    }
    int64_t g = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int64_t mt = it / p.nsplit;
      const int nt0 = (int)(it % p.nsplit) * per, nt1 = min(p.ntn, nt0 + per);
      for (int nt = nt0; nt < nt1; ++nt) {
        for (int kc = 0; kc < p.nk; ++kc, ++g) {
          const int s = (int)(g % HS);
          const int64_t use = g / HS;
          if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
          uint8_t *st = base + s * HSTAGE;
          if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)HSTAGE);
          __syncwarp();
          if (lane == 0) tma_load_2d(st, &tmAh, kc * HBK, (int)(mt * 128), &full[s]);
          if (lane == 1) tma_load_2d(st + HABYTES, &tmAl, kc * HBK, (int)(mt * 128), &full[s]);
          if (lane == 2) tma_load_2d(st + 2 * HABYTES, &tmBh, kc * HBK, nt * NW, &full[s]);
          if (lane == 3) tma_load_2d(st + 2 * HABYTES + HBBYTES, &tmBl, kc * HBK, nt * NW, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    int64_t g = 0, tcount = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int nt0 = (int)(it % p.nsplit) * per, nt1 = min(p.ntn, nt0 + per);
      for (int nt = nt0; nt < nt1; ++nt, ++tcount) {
        const int buf = (int)(tcount & 1);
        const int64_t use_b = tcount >> 1;
        if (use_b > 0) mbar_wait(&tfree[buf], (uint32_t)((use_b - 1) & 1));
        tc_fence_after();
        const int64_t rem = p.ncols - (int64_t)nt * NW;
        const int N = (int)std::min<int64_t>(NW, (rem + 15) / 16 * 16);
        const uint32_t idesc = make_idesc_f16(N);
        const uint32_t d = tmem + (uint32_t)(buf * NW);
        for (int kc = 0; kc < p.nk; ++kc, ++g) {
          const int s = (int)(g % HS);
          const int64_t use = g / HS;
          mbar_wait(&full[s], (uint32_t)(use & 1));
          tc_fence_after();
          const bool leader = elect_one();
          const uint32_t ah = smem_u32(base + s * HSTAGE), al = ah + HABYTES;
          const uint32_t bh = al + HABYTES, bl = bh + HBBYTES;
          const uint64_t dah = make_desc(ah, 16, 1024), dal = make_desc(al, 16, 1024);
          const uint64_t dbh = make_desc(bh, 16, 1024), dbl = make_desc(bl, 16, 1024);
#pragma unroll
          for (int ks = 0; ks < HBK / 16; ++ks) {
            const uint32_t acc0 = (kc == 0 && ks == 0) ? 0u : 1u;
            if (leader) {
              mma_f16(d, dah + 2 * ks, dbh + 2 * ks, idesc, acc0);
              mma_f16(d, dah + 2 * ks, dbl + 2 * ks, idesc, 1u);
              mma_f16(d, dal + 2 * ks, dbh + 2 * ks, idesc, 1u);
            }
          }
          __syncwarp();
          if (leader) mma_commit(&empty[s]);
          __syncwarp();
        }
        if (elect_one()) mma_commit(&done[buf]);
        __syncwarp();
      }
    }
  } else {
    // epilogue warps 2-9: TMEM lane quadrant q = warp % 4, column half hf
    const int q = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int r = 32 * q + lane;
    const float bsc = ldexpf(1.f, -(14 - *bexp));
    int64_t tcount = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int64_t mt = it / p.nsplit;
      const int nt0 = (int)(it % p.nsplit) * per, nt1 = min(p.ntn, nt0 + per);
      const int64_t row = mt * 128 + r;
      const float xs = row < p.m ? __ldg(rinv + row) * bsc : 0.f;
      const float rsign = (ZM && row < p.m) ? __ldg(p.row_sign + row) : 1.f;
      for (int nt = nt0; nt < nt1; ++nt, ++tcount) {
        const int buf = (int)(tcount & 1);
        mbar_wait(&done[buf], (uint32_t)((tcount >> 1) & 1));
        tc_fence_after();
        const uint32_t tb = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * NW + hf * (NW / 2));
        epi_tile<ZP, ZM, L1P, NW / 2, false>(p, tb, nt, row, rsign, lane, xs, hf * (NW / 2));
        tc_fence_before();
        mbar_arrive(&tfree[buf]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// max over rows of ilogb(max_k |x|) (B's common exponent)
__global__ void k_rows_maxexp(const float *__restrict__ src, int64_t rows, int k, int64_t lds, int *__restrict__ gexp) {
  grid_dep_enter();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float m = 0.f;
  if (idx < rows * k) m = fabsf(src[(idx / k) * lds + idx % k]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(gexp, ilogbf(m));
}
// fp16 hi/lo split of a row-major fp32 block (rows × k, stride lds) into
// rows × kp (zero padded): a warp per row; the row's scale 2^e puts its
// largest |x| in [2^14, 2^15) (gexp == nullptr) or uses the common exponent
// *gexp; rinv[row] = 2^-e (per-row mode)
__global__ void k_split_f16(const float *__restrict__ src, int64_t rows, int k, int64_t lds, int kp,
                            __half *__restrict__ hi, __half *__restrict__ lo, float *__restrict__ rinv,
                            const int *__restrict__ gexp) {
  grid_dep_enter();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  // lane owns 8 consecutive entries per 256: two 16-B loads, one 16-B store per plane
  const bool vec = (k % 8) == 0 && (lds % 4) == 0 && ((uintptr_t)src & 15) == 0;
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < rows; i += nw) {
    const float *x = src + i * lds;
    int e;
    if (gexp) {
      e = 14 - *gexp;
    } else {
      float m = 0.f;
      if (vec) {
        for (int c = 8 * lane; c < k; c += 256) {
          const float4 a = *reinterpret_cast<const float4 *>(x + c), b = *reinterpret_cast<const float4 *>(x + c + 4);
          m = fmaxf(m, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
          m = fmaxf(m, fmaxf(fmaxf(fabsf(b.x), fabsf(b.y)), fmaxf(fabsf(b.z), fabsf(b.w))));
        }
      } else {
        for (int c = lane; c < k; c += 32) m = fmaxf(m, fabsf(x[c]));
      }
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      e = m > 0.f ? 14 - ilogbf(m) : 0;
      if (lane == 0) rinv[i] = ldexpf(1.f, -e);
    }
    for (int c = 8 * lane; c < kp; c += 256) {
      float v[8];
      if (vec && c + 8 <= k) {
        const float4 a = *reinterpret_cast<const float4 *>(x + c), b = *reinterpret_cast<const float4 *>(x + c + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) v[t] = c + t < k ? x[c + t] : 0.f;
      }
      __align__(16) __half h[8], l[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float y = ldexpf(v[t], e);
        h[t] = __float2half_rn(y);
        l[t] = __float2half_rn(y - __half2float(h[t]));
      }
      *reinterpret_cast<uint4 *>(hi + i * kp + c) = *reinterpret_cast<const uint4 *>(h);
      *reinterpret_cast<uint4 *>(lo + i * kp + c) = *reinterpret_cast<const uint4 *>(l);
    }
  }
}

// rows of X at the sparse-sign coordinates, one zp-group per column c:
// out row c·zp + t = X[rows[c·z + t]] for t < z, zero for the padding (sign 0);
// optional tf32 lo part and the sign vector
__global__ void k_gather_groups(const float *__restrict__ X, int64_t ldx, int64_t row0, int64_t nloc,
                                const int32_t *__restrict__ rows, const float *__restrict__ signs, int64_t h, int z,
                                int zp, int k, int64_t ldb, float *__restrict__ hi, float *__restrict__ lo,
                                float *__restrict__ sgn) {
  grid_dep_enter();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nr = h * zp;
  if (idx >= nr * ldb) return;
  const int64_t j = idx / ldb, kk = idx % ldb;
  const int64_t c = j / zp;
  const int t = (int)(j % zp);
  float x = 0.f;
  if (t < z && kk < k) {
    const int64_t r = (int64_t)rows[c * z + t] - row0;  // rows of other ranks contribute 0
    if (r >= 0 && r < nloc) x = X[r * ldx + kk];
  }
  hi[idx] = x;
  if (lo) lo[idx] = x - tc::tf32_trunc(x);
  if (kk == 0) sgn[j] = t < z ? signs[c * z + t] : 0.f;
}

// sign → bit masks, 32 columns per word (NW/32 words per N tile, zero padded)
__global__ void k_sign_bits(const float *__restrict__ sg, int64_t ncols, int64_t nwords, uint32_t *__restrict__ neg,
                            uint32_t *__restrict__ val) {
  grid_dep_enter();
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= nwords) return;
  uint32_t nb = 0, vb = 0;
  for (int i = 0; i < 32; ++i) {
    const int64_t j = w * 32 + i;
    const float v = j < ncols ? sg[j] : 0.f;
    if (v < 0.f) nb |= 1u << i;
    if (v != 0.f) vb |= 1u << i;
  }
  neg[w] = nb;
  val[w] = vb;
}

}  // namespace tcs

static int pow2_at_least(int z) {
  int zp = 1;
  while (zp < z) zp <<= 1;
  return zp;
}

static void launch_sketch(Ctx &c, const CUtensorMap &ma, const CUtensorMap &mh, const CUtensorMap &ml,
                          tcs::SkP &prm, const float *col_sign) {
  using namespace tcs;
  const int64_t nwords = (int64_t)prm.ntn * (NW / 32);
  DBuf<uint32_t> bits((size_t)2 * nwords, c.stream);
  NM_LAUNCH(c, "sign_bits", launch_pdl(c.stream, k_sign_bits, ceil_div(nwords, 128), 128, 0, col_sign, prm.ncols, nwords, bits.p,
                                                                                    bits.p + nwords));
  prm.neg_bits = bits.p;
  prm.val_bits = bits.p + nwords;
  prm.epi = prm.zp * 4 + (prm.row_sign ? 2 : 0) + (prm.logmode ? 1 : 0);
  const size_t smem = 1024 + (size_t)S * STAGE + (3 * S + 4) * 8 + 16;
  auto kern = k_sketch_tc<8, false, false>;
  switch (prm.epi) {
#define SK_CASE(ZP, ZM, L1P) \
  case (ZP) * 4 + (ZM) * 2 + (L1P): kern = k_sketch_tc<ZP, ZM, L1P>; break;
    SK_CASE(2, 0, 0) SK_CASE(4, 0, 0) SK_CASE(8, 0, 0) SK_CASE(16, 0, 0) SK_CASE(32, 0, 0) SK_CASE(64, 0, 0)
    SK_CASE(2, 1, 0) SK_CASE(4, 1, 0) SK_CASE(8, 1, 0) SK_CASE(16, 1, 0) SK_CASE(32, 1, 0) SK_CASE(64, 1, 0)
    SK_CASE(2, 0, 1) SK_CASE(4, 0, 1) SK_CASE(8, 0, 1) SK_CASE(16, 0, 1) SK_CASE(32, 0, 1) SK_CASE(64, 0, 1)
    SK_CASE(2, 1, 1) SK_CASE(4, 1, 1) SK_CASE(8, 1, 1) SK_CASE(16, 1, 1) SK_CASE(32, 1, 1) SK_CASE(64, 1, 1)
#undef SK_CASE
    default: NM_REQUIRE(false, "tc_sketch: unsupported group size");
  }
  smem_attr(kern, smem);
  // enough items for every SM: split the N tiles of an M tile when M tiles are few
  prm.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(prm.ntn, ceil_div(2 * (int64_t)c.num_sms, prm.nmt)));
  const int per = (prm.ntn + prm.nsplit - 1) / prm.nsplit;
  prm.nsplit = (prm.ntn + per - 1) / per;
  const int64_t items = prm.nmt * prm.nsplit;
  const unsigned grid = (unsigned)std::min<int64_t>(items, c.num_sms);
  NM_LAUNCH(c, "sketch_tc", launch_pdl(c.stream, kern, grid, THREADS, smem, ma, mh, ml, prm));
}

// fp16-split sketches (k_sketch_h); NETMFP_SKETCH_F16=0 keeps 3xTF32 (A/B measurements)
static bool sketch_f16() {
  static const bool on = [] {
    const char *v = getenv("NETMFP_SKETCH_F16");
    return !v || atoi(v) != 0;
  }();
  return on;
}

static void launch_sketch_h(Ctx &c, const CUtensorMap &mah, const CUtensorMap &mal, const CUtensorMap &mbh,
                            const CUtensorMap &mbl, tcs::SkP &prm, const float *col_sign, const float *rinv,
                            const int *bexp) {
  using namespace tcs;
  const int64_t nwords = (int64_t)prm.ntn * (NW / 32);
  DBuf<uint32_t> bits((size_t)2 * nwords, c.stream);
  NM_LAUNCH(c, "sign_bits", launch_pdl(c.stream, k_sign_bits, ceil_div(nwords, 128), 128, 0, col_sign, prm.ncols, nwords,
                                       bits.p, bits.p + nwords));
  prm.neg_bits = bits.p;
  prm.val_bits = bits.p + nwords;
  const size_t smem = 1024 + (size_t)HS * HSTAGE + (2 * HS + 4) * 8 + 16;
  auto kern = k_sketch_h<8, false, false>;
  switch (prm.zp * 4 + (prm.row_sign ? 2 : 0) + (prm.logmode ? 1 : 0)) {
#define SKH_CASE(ZP, ZM, L1P) \
  case (ZP) * 4 + (ZM) * 2 + (L1P): kern = k_sketch_h<ZP, ZM, L1P>; break;
    SKH_CASE(2, 0, 0) SKH_CASE(4, 0, 0) SKH_CASE(8, 0, 0) SKH_CASE(16, 0, 0) SKH_CASE(32, 0, 0) SKH_CASE(64, 0, 0)
    SKH_CASE(2, 0, 1) SKH_CASE(4, 0, 1) SKH_CASE(8, 0, 1) SKH_CASE(16, 0, 1) SKH_CASE(32, 0, 1) SKH_CASE(64, 0, 1)
    SKH_CASE(2, 1, 0) SKH_CASE(4, 1, 0) SKH_CASE(8, 1, 0) SKH_CASE(16, 1, 0) SKH_CASE(32, 1, 0) SKH_CASE(64, 1, 0)
    SKH_CASE(2, 1, 1) SKH_CASE(4, 1, 1) SKH_CASE(8, 1, 1) SKH_CASE(16, 1, 1) SKH_CASE(32, 1, 1) SKH_CASE(64, 1, 1)
#undef SKH_CASE
    default: NM_REQUIRE(false, "tc_sketch: unsupported group size");
  }
  smem_attr(kern, smem);
  prm.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(prm.ntn, ceil_div(2 * (int64_t)c.num_sms, prm.nmt)));
  const int per = (prm.ntn + prm.nsplit - 1) / prm.nsplit;
  prm.nsplit = (prm.ntn + per - 1) / per;
  const int64_t items = prm.nmt * prm.nsplit;
  const unsigned grid = (unsigned)std::min<int64_t>(items, c.num_sms);
  NM_LAUNCH(c, "sketch_tc", launch_pdl(c.stream, kern, grid, HT, smem, mah, mal, mbh, mbl, prm, rinv, bexp));
}

namespace tcs {
// hi = x, lo = x - trunc_tf32(x) of an r × k block (row stride ld; padding columns stay 0)
__global__ void k_split_hilo(const float *__restrict__ src, int64_t rows, int k, int64_t ld, float *__restrict__ hi,
                             float *__restrict__ lo) {
  grid_dep_enter();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * ld) return;
  const float x = (idx % ld) < k ? src[idx] : 0.f;
  hi[idx] = x;
  if (lo) lo[idx] = x - tc::tf32_trunc(x);
}
__global__ void k_transpose64(const double *__restrict__ C, int64_t k, int64_t ldc, double *__restrict__ Ct) {
  grid_dep_enter();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx < k * k) Ct[(idx % k) * k + idx / k] = C[(idx / k) * ldc + idx % k];
}
}  // namespace tcs

// Gathered rows G (nr × k, ld ldb; fp32) times the small fp64 matrix Bs (k × k):
// out = G Bs (tensor cores for nr >= 128), then hi / lo split into (hi, lo)
static void rows_times(Ctx &c, float *G, int64_t nr, int k, int64_t ldb, const double *Bs, float *hi, float *lo) {
  DBuf<float> out((size_t)nr * ldb, c.stream);
  Mat Gm{G, nr, k, ldb}, Om{out.p, nr, k, ldb};
  gemm_tall(c, Gm, Bs, k, k, nullptr, 0.f, Om);
  NM_LAUNCH(c, "split_hilo", launch_pdl(c.stream, tcs::k_split_hilo, ceil_div(nr * ldb, 256), 256, 0, out.p, nr, k, ldb, hi, lo));
}

// Y[n × h] = f(scale · F C F(rows)ᵀ) Ψ  (Y mode; Ψ = (rows, signs) with z per column).
// M̂ = (F C) F_rᵀ = F (F_r Cᵀ)ᵀ: the A operand is F itself and the gathered
// rows F_r are multiplied by Cᵀ (an h·zp × k × k product) — no n × k F·C block.
bool sketch_uses_split() { return sketch_f16(); }

void sketch_split_a(Ctx &c, const Mat &F, SketchA &A) {
  using namespace tcs;
  A.n = F.rows;
  A.k = (int)F.cols;
  A.kp = (int)((A.k + HBK - 1) / HBK * HBK);
  A.hi.alloc((size_t)A.n * A.kp, c.stream);
  A.lo.alloc((size_t)A.n * A.kp, c.stream);
  A.rinv.alloc(A.n, c.stream);
  if (A.n == 0) return;
  NM_LAUNCH(c, "split_f16", launch_pdl(c.stream, k_split_f16,
                                       (unsigned)std::min<int64_t>(ceil_div(A.n, 8), (int64_t)c.num_sms * 16), 256, 0,
                                       F.p, A.n, A.k, F.ld, A.kp, reinterpret_cast<__half *>(A.hi.p),
                                       reinterpret_cast<__half *>(A.lo.p), A.rinv.p, nullptr));
}

void tc_sketch_y(Ctx &c, const Mat &F, const double *C, int64_t ldc, const int32_t *rows, const float *signs,
                 int64_t h, int z, float scale, int logmode, const Mat &Y, int64_t row0, const SketchA *pre) {
  using namespace tcs;
  NM_REQUIRE(Y.rows == F.rows && Y.cols == h, "tc_sketch_y: shapes");
  NM_REQUIRE(z >= 2 && z <= 64, "tc_sketch_y: 2 <= z <= 64");
  const int64_t n = F.rows;
  const int k = (int)F.cols;
  if (n == 0 || h == 0) return;
  const int zp = pow2_at_least(z);
  const int64_t ncols = h * zp;
  const int64_t ldb = pad32(k);
  DBuf<float> g((size_t)ncols * ldb, c.stream), bh((size_t)ncols * ldb, c.stream), bl((size_t)ncols * ldb, c.stream),
      sg(pad4(ncols) + NW, c.stream);
  DBuf<double> Ct((size_t)k * k, c.stream);
  NM_CUDA(cudaMemsetAsync(sg.p, 0, sg.n * 4, c.stream));
  NM_LAUNCH(c, "gather_groups", launch_pdl(c.stream, k_gather_groups, ceil_div(ncols * ldb, 256), 256, 0, F.p, F.ld, row0, F.rows, rows, signs, h, z, zp, k, ldb, g.p, nullptr, sg.p));
  // each gathered row lives on exactly one rank: the sum over ranks is exact
  dist_allreduce(c, g.p, (size_t)ncols * ldb, DType::F32);
  NM_LAUNCH(c, "transpose64", launch_pdl(c.stream, k_transpose64, ceil_div((int64_t)k * k, 256), 256, 0, C, k, ldc, Ct.p));
  if (sketch_f16()) {
    // fp16-split operands (k_sketch_h): B rows = F_r Cᵀ in fp32, then both
    // operands split once into hi/lo fp16 planes
    DBuf<float> bt((size_t)ncols * ldb, c.stream);
    {
      Mat Gm{g.p, ncols, k, ldb}, Om{bt.p, ncols, k, ldb};
      gemm_tall(c, Gm, Ct.p, k, k, nullptr, 0.f, Om);
    }
    const int kp = (int)((k + HBK - 1) / HBK * HBK);
    SketchA own;
    if (!pre) sketch_split_a(c, F, own);
    const SketchA &A = pre ? *pre : own;
    NM_REQUIRE(A.n == n && A.k == k && A.kp == kp, "tc_sketch_y: pre-split operand does not match F");
    const __half *ah = reinterpret_cast<const __half *>(A.hi.p), *al = reinterpret_cast<const __half *>(A.lo.p);
    const float *rinv = A.rinv.p;
    DBuf<__half> bhh((size_t)ncols * kp, c.stream), blh((size_t)ncols * kp, c.stream);
    DBuf<int> bexp(1, c.stream);
    NM_CUDA(cudaMemsetAsync(bexp.p, 0x80, sizeof(int), c.stream));
    NM_LAUNCH(c, "rows_maxexp", launch_pdl(c.stream, k_rows_maxexp, ceil_div(ncols * k, 256), 256, 0, bt.p, ncols, k,
                                           ldb, bexp.p));
    NM_LAUNCH(c, "split_f16", launch_pdl(c.stream, k_split_f16, ceil_div(ncols, 8), 256, 0, bt.p, ncols, k, ldb, kp,
                                         bhh.p, blh.p, nullptr, bexp.p));
    CUtensorMap mah = make_map_f16(ah, n, kp, kp, 128), mal = make_map_f16(al, n, kp, kp, 128);
    CUtensorMap mbh = make_map_f16(bhh.p, ncols, kp, kp, NW), mbl = make_map_f16(blh.p, ncols, kp, kp, NW);
    SkP prm{};
    prm.m = n;
    prm.k = kp;
    prm.nk = kp / HBK;
    prm.ncols = ncols;
    prm.ntn = (int)ceil_div(ncols, NW);
    prm.nmt = ceil_div(n, 128);
    prm.zp = zp;
    prm.lzp = __builtin_ctz(zp);
    prm.h = h;
    prm.scale = scale;
    prm.logmode = logmode;
    prm.row_sign = nullptr;
    prm.out = Y.p;
    prm.ldo = Y.ld;
    launch_sketch_h(c, mah, mal, mbh, mbl, prm, sg.p, rinv, bexp.p);
    return;
  }
  rows_times(c, g.p, ncols, k, ldb, Ct.p, bh.p, bl.p);  // B rows = F_r Cᵀ
  CUtensorMap ma = make_map(F.p, n, k, F.ld, 128, SW128, BK);
  CUtensorMap mh = make_map(bh.p, ncols, k, ldb, NW, SW128, BK);
  CUtensorMap ml = make_map(bl.p, ncols, k, ldb, NW, SW128, BK);
  SkP prm{};
  prm.m = n;
  prm.k = k;
  prm.nk = (int)ceil_div(k, BK);
  prm.ncols = ncols;
  prm.ntn = (int)ceil_div(ncols, NW);
  prm.nmt = ceil_div(n, 128);
  prm.zp = zp;
  prm.lzp = __builtin_ctz(zp);
  prm.h = h;
  prm.scale = scale;
  prm.logmode = logmode;
  prm.row_sign = nullptr;
  prm.out = Y.p;
  prm.ldo = Y.ld;
  launch_sketch(c, ma, mh, ml, prm, sg.p);
}

// Z[h × h] = Πᵀ f(scale · (F C)(rows) F(rows)ᵀ) Π  (Z mode), fp32 output with ldz;
// the gathered rows of F times C are the A operand
void tc_sketch_z(Ctx &c, const Mat &F, const double *C, int64_t ldc, const int32_t *rows, const float *signs,
                 int64_t h, int z, float scale, int logmode, float *Zf, int64_t ldz, int64_t row0) {
  using namespace tcs;
  NM_REQUIRE(z >= 2 && z <= 64, "tc_sketch_z: 2 <= z <= 64");
  const int k = (int)F.cols;
  const int zp = pow2_at_least(z);
  const int64_t nr = h * zp;
  const int64_t ldb = pad32(k);
  DBuf<float> ah((size_t)nr * ldb, c.stream), rs(pad4(nr) + NW, c.stream);
  DBuf<float> bh((size_t)nr * ldb, c.stream), bl((size_t)nr * ldb, c.stream), sg(pad4(nr) + NW, c.stream);
  NM_CUDA(cudaMemsetAsync(sg.p, 0, sg.n * 4, c.stream));
  NM_CUDA(cudaMemsetAsync(rs.p, 0, rs.n * 4, c.stream));
  NM_LAUNCH(c, "gather_groups", launch_pdl(c.stream, k_gather_groups, ceil_div(nr * ldb, 256), 256, 0, F.p, F.ld, row0, F.rows, rows, signs, h, z, zp, k, ldb, bh.p, bl.p, sg.p));
  dist_allreduce(c, bh.p, (size_t)nr * ldb, DType::F32);
  dist_allreduce(c, bl.p, (size_t)nr * ldb, DType::F32);
  // A = F(rows) C (the gathered raw rows times C); row signs = the column signs
  {
    Mat Gm{bh.p, nr, k, ldb}, Om{ah.p, nr, k, ldb};
    gemm_tall(c, Gm, C, ldc, k, nullptr, 0.f, Om);
  }
  NM_CUDA(cudaMemcpyAsync(rs.p, sg.p, rs.n * 4, cudaMemcpyDeviceToDevice, c.stream));
  if (zp > 32) NM_CUDA(cudaMemset2DAsync(Zf, ldz * 4, 0, h * 4, h, c.stream));
  if (sketch_f16()) {
    // fp16-split operands as in tc_sketch_y: A = F(rows) C per-row scaled, B = F(rows) one common scale
    const int kp = (int)((k + HBK - 1) / HBK * HBK);
    DBuf<__half> a16h((size_t)nr * kp, c.stream), a16l((size_t)nr * kp, c.stream);
    DBuf<__half> b16h((size_t)nr * kp, c.stream), b16l((size_t)nr * kp, c.stream);
    DBuf<float> rinv(nr, c.stream);
    DBuf<int> bexp(1, c.stream);
    NM_CUDA(cudaMemsetAsync(bexp.p, 0x80, sizeof(int), c.stream));
    NM_LAUNCH(c, "rows_maxexp", launch_pdl(c.stream, k_rows_maxexp, ceil_div(nr * k, 256), 256, 0, bh.p, nr, k, ldb,
                                           bexp.p));
    NM_LAUNCH(c, "split_f16", launch_pdl(c.stream, k_split_f16, ceil_div(nr, 8), 256, 0, bh.p, nr, k, ldb, kp,
                                         b16h.p, b16l.p, nullptr, bexp.p));
    NM_LAUNCH(c, "split_f16", launch_pdl(c.stream, k_split_f16, ceil_div(nr, 8), 256, 0, ah.p, nr, k, ldb, kp,
                                         a16h.p, a16l.p, rinv.p, nullptr));
    CUtensorMap mah = make_map_f16(a16h.p, nr, kp, kp, 128), mal = make_map_f16(a16l.p, nr, kp, kp, 128);
    CUtensorMap mbh = make_map_f16(b16h.p, nr, kp, kp, NW), mbl = make_map_f16(b16l.p, nr, kp, kp, NW);
    SkP prm{};
    prm.m = nr;
    prm.k = kp;
    prm.nk = kp / HBK;
    prm.ncols = nr;
    prm.ntn = (int)ceil_div(nr, NW);
    prm.nmt = ceil_div(nr, 128);
    prm.zp = zp;
    prm.lzp = __builtin_ctz(zp);
    prm.h = h;
    prm.scale = scale;
    prm.logmode = logmode;
    prm.row_sign = rs.p;
    prm.out = Zf;
    prm.ldo = ldz;
    launch_sketch_h(c, mah, mal, mbh, mbl, prm, sg.p, rinv.p, bexp.p);
    return;
  }
  CUtensorMap ma = make_map(ah.p, nr, k, ldb, 128, SW128, BK);
  CUtensorMap mh = make_map(bh.p, nr, k, ldb, NW, SW128, BK);
  CUtensorMap ml = make_map(bl.p, nr, k, ldb, NW, SW128, BK);
  SkP prm{};
  prm.m = nr;
  prm.k = k;
  prm.nk = (int)ceil_div(k, BK);
  prm.ncols = nr;
  prm.ntn = (int)ceil_div(nr, NW);
  prm.nmt = ceil_div(nr, 128);
  prm.zp = zp;
  prm.lzp = __builtin_ctz(zp);
  prm.h = h;
  prm.scale = scale;
  prm.logmode = logmode;
  prm.row_sign = rs.p;
  prm.out = Zf;
  prm.ldo = ldz;
  launch_sketch(c, ma, mh, ml, prm, sg.p);
}

}  // namespace netmfp
