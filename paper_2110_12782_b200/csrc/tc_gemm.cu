// tc_gemm.cu — tall-skinny dense contractions on the 5th-gen tensor cores.
//
// C = A·Bᵀ with fp32 operands at fp32-level accuracy via 3xTF32: every operand
// x is split into tf32 parts x = hi + lo (hi = rna_tf32(x), lo = x - hi) and
// C = A_hi B_hiᵀ + A_hi B_loᵀ + A_lo B_hiᵀ (the dropped lo·lo term is ~2^-22
// relative), accumulated in fp32 in TMEM by tcgen05.mma.kind::tf32.
//
//   * one CTA computes a 128-row tile of C for up to 2×256 columns (two MMA
//     N-subtiles side by side in TMEM), looping over K in 32-element chunks;
//   * 256 threads stage each K-chunk: global fp32 -> hi/lo split -> the
//     K-major SWIZZLE_128B canonical layout in shared memory (8-row × 128-B
//     atoms, 16-B chunk c of row r at c ^ (r & 7)); two stages, mbarrier-
//     tracked (tcgen05.commit) so the next chunk loads while the tensor core
//     works on the current one;
//   * one elected thread issues the MMAs; the epilogue reads TMEM with
//     tcgen05.ld (warp w%4 owns TMEM lanes = tile rows 32(w%4)..+31).
//
// Producers: ROWS  — operand element (row, k) = P[row*ld + k] (K contiguous):
//                    A of gemm_tall / sketch, Bᵀ of gemm_tall;
//            TRANS — element (row, k) = P[k*ld + row] (the Gram's Aᵀ, Bᵀ:
//                    rows of the n×c block are the contraction index).
// Epilogues: STORE — C = rs_i · acc (fp32, row-major, optional row scale d_i^-e)
//            PART  — fp32 partial tile of a K-slab (Gram, reduced in fp64 later)
#include <cuda.h>

#include "common.cuh"
#include "kernels.cuh"

namespace netmfp {
namespace tc {

constexpr int BM = 128;       // tile rows (UMMA M)
constexpr int BK = 32;        // fp32 elements per K-chunk = one 128-B swizzle row
constexpr int NT = 256;       // threads
constexpr int MAXN = 288;     // max columns per CTA (2 subtiles of <= 144.. 256)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// byte offset of the 16-B chunk (row r, chunk c) inside a K-major SW128 tile
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// SM100 shared-memory matrix descriptor: K-major, SWIZZLE_128B, SBO = 1024 B
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                          // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                // SBO: 8-row core-matrix stride
  d |= (uint64_t)1 << 46;                          // version 1 (sm_100)
  d |= (uint64_t)2 << 61;                          // layout: SWIZZLE_128B
  return d;
}

// instruction descriptor: kind::tf32, D f32, A/B tf32, both K-major, M=128, N
__host__ __device__ constexpr uint32_t make_idesc(int N) {
  return (1u << 4)                 // c_format = F32
         | (2u << 7)               // a_format = TF32
         | (2u << 10)              // b_format = TF32
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :
      : "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

enum Prod { ROWS = 0, TRANS = 1 };
enum Epi { STORE = 0, PART = 1 };

struct Operand {
  const float *p;
  int64_t ld;
  int64_t rows;   // valid rows (MN extent) of the operand
  int64_t kdim;   // valid K extent
  const int32_t *gather;  // ROWS: optional row index map
  const int32_t *wdeg;    // TRANS: optional K-row weight d_k^-wexp
  float wexp;
};

// stage one K-chunk of `rows_tile` operand rows starting at row0 into hi/lo tiles
template <int PROD>
__device__ __forceinline__ void stage_operand(const Operand &op, int64_t row0, int rows_tile, int64_t k0,
                                              uint8_t *hi, uint8_t *lo) {
  if (PROD == ROWS) {
    // chunk id = r*8 + c (c: 16-B chunk within the 32-float K row)
    for (int idx = threadIdx.x; idx < rows_tile * 8; idx += NT) {
      const int r = idx >> 3, c = idx & 7;
      const int64_t gr = row0 + r;
      const int64_t kk = k0 + c * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < op.rows && kk < op.kdim) {
        const int64_t src = op.gather ? (int64_t)op.gather[gr] : gr;
        const float *ptr = op.p + src * op.ld + kk;
        if (kk + 4 <= op.kdim) {
          v = __ldg(reinterpret_cast<const float4 *>(ptr));
        } else {
          v.x = ptr[0];
          if (kk + 1 < op.kdim) v.y = ptr[1];
          if (kk + 2 < op.kdim) v.z = ptr[2];
        }
      }
      float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
      float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      const uint32_t off = sw128(r, c);
      *reinterpret_cast<float4 *>(hi + off) = h;
      *reinterpret_cast<float4 *>(lo + off) = l;
    }
  } else {
    // element (row r, k) = P[(k0+k)*ld + row0 + r]; thread t of a warp takes
    // k = t (one global row each), float4 along r: conflict-free scatter
    const int nr4 = rows_tile / 4;
    for (int idx = threadIdx.x; idx < nr4 * BK; idx += NT) {
      const int k = idx % BK, r4 = idx / BK;
      const int64_t gk = k0 + k;
      const int64_t gr = row0 + r4 * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gk < op.kdim && gr < op.rows) {
        const float *ptr = op.p + gk * op.ld + gr;
        if (gr + 4 <= op.rows) {
          v = __ldg(reinterpret_cast<const float4 *>(ptr));
        } else {
          v.x = ptr[0];
          if (gr + 1 < op.rows) v.y = ptr[1];
          if (gr + 2 < op.rows) v.z = ptr[2];
        }
        if (op.wdeg) {
          const int dg = op.wdeg[gk];
          const float w = dg <= 0 ? 0.f : (op.wexp == 0.f ? 1.f : powf((float)dg, -op.wexp));
          v.x *= w; v.y *= w; v.z *= w; v.w *= w;
        }
      }
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = r4 * 4 + i;
        const uint32_t off = sw128(r, k >> 2) + (k & 3) * 4;
        const float h = tf32_rna(e[i]);
        *reinterpret_cast<float *>(hi + off) = h;
        *reinterpret_cast<float *>(lo + off) = e[i] - h;
      }
    }
  }
}

struct EpiArgs {
  float *C;        // STORE: C[row*ldc + col]; PART: partial tile base for this slab
  int64_t ldc;
  int64_t rows;    // valid output rows
  int64_t cols;    // valid output cols
  const int32_t *deg;
  float rexp;
};

// C tile (BM × ntot) = A(m0.., k-range) · B(0..ntot, k-range)ᵀ
template <int PA, int PB, int EPI>
__global__ void __launch_bounds__(NT, 1) k_tc_gemm(Operand A, Operand B, int ntot, int n_sub, int nsub_w,
                                                   int64_t kslab, EpiArgs ep) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned carve-up
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int a_bytes = BM * 128;               // 16 KB per part
  const int b_bytes = ((ntot + 7) / 8) * 1024;  // rows rounded to 8-row atoms
  const int stage_bytes = 2 * a_bytes + 2 * b_bytes;
  uint8_t *st[2] = {base, base + stage_bytes};
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + 2 * stage_bytes);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2);

  const int warp = threadIdx.x / 32;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t kbeg = (int64_t)blockIdx.y * kslab;
  const int64_t kend = min(kbeg + kslab, A.kdim);
  const int nk = (int)((kend - kbeg + BK - 1) / BK);

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const uint32_t tcols = ntot <= 32 ? 32u : ntot <= 64 ? 64u : ntot <= 128 ? 128u : ntot <= 256 ? 256u : 512u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = make_idesc(nsub_w);

  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt & 1;
    if (kt >= 2) mbar_wait(&bars[s], (uint32_t)(((kt - 2) >> 1) & 1));
    const int64_t k0 = kbeg + (int64_t)kt * BK;
    uint8_t *ahi = st[s], *alo = st[s] + a_bytes, *bhi = st[s] + 2 * a_bytes, *blo = bhi + b_bytes;
    stage_operand<PA>(A, m0, BM, k0, ahi, alo);
    stage_operand<PB>(B, 0, (ntot + 7) / 8 * 8, k0, bhi, blo);
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t a_hi = smem_u32(ahi), a_lo = smem_u32(alo);
      const uint32_t b_hi = smem_u32(bhi), b_lo = smem_u32(blo);
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint32_t koff = ks * 32;  // 8 tf32 = 32 B along K inside the swizzle row
        for (int sb = 0; sb < n_sub; ++sb) {
          const uint32_t boff = (uint32_t)sb * (uint32_t)(nsub_w / 8) * 1024u;
          const uint32_t d = tmem + (uint32_t)(sb * nsub_w);
          const uint32_t acc0 = (kt > 0 || ks > 0) ? 1u : 0u;
          mma_tf32(d, make_desc(a_hi + koff), make_desc(b_hi + boff + koff), idesc, acc0);
          mma_tf32(d, make_desc(a_hi + koff), make_desc(b_lo + boff + koff), idesc, 1u);
          mma_tf32(d, make_desc(a_lo + koff), make_desc(b_hi + boff + koff), idesc, 1u);
        }
      }
      mma_commit(&bars[s]);
    }
    __syncwarp();
  }
  // wait for the last chunk's MMAs (commit covers all earlier MMAs of the thread)
  if (nk > 0) mbar_wait(&bars[(nk - 1) & 1], (uint32_t)(((nk - 1) >> 1) & 1));
  tc_fence_after();

  // epilogue: warp w reads lanes 32(w%4).. ; warps 0-3 and 4-7 split the columns
  const int lane_base = (warp & 3) * 32;
  const int row_in_tile = lane_base + (threadIdx.x & 31);
  const int64_t row = m0 + row_in_tile;
  const int ncols16 = (ntot + 15) / 16;
  const int half = (ncols16 + 1) / 2;
  const int c16_beg = (warp < 4) ? 0 : half, c16_end = (warp < 4) ? half : ncols16;
  float scale = 1.f;
  if (EPI == STORE && ep.deg && row < ep.rows) {
    const int dg = ep.deg[row];
    scale = dg <= 0 ? 0.f : (ep.rexp == 0.f ? 1.f : powf((float)dg, -ep.rexp));
  }
  for (int c16 = c16_beg; c16 < c16_end; ++c16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)lane_base << 16) + (uint32_t)(c16 * 16), v);
    const int col0 = c16 * 16;
    if (nk == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.f;
    }
    if (EPI == STORE) {
      if (row < ep.rows) {
        float *dst = ep.C + row * ep.ldc + col0;
        if (col0 + 16 <= ep.cols) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4 *>(dst + i) =
                make_float4(scale * v[i], scale * v[i + 1], scale * v[i + 2], scale * v[i + 3]);
        } else {
          for (int i = 0; i < 16 && col0 + i < ep.cols; ++i) dst[i] = scale * v[i];
        }
      }
    } else {
      // PART: dense (BM_pad × ntot_pad) fp32 tile at ep.C + slab*stride; ldc = padded cols
      float *dst = ep.C + (int64_t)blockIdx.y * ep.rows * ep.ldc + row * ep.ldc + col0;
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        *reinterpret_cast<float4 *>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tcols));
}

static size_t smem_for(int ntot) {
  const int a_bytes = BM * 128;
  const int b_bytes = ((ntot + 7) / 8) * 1024;
  return (size_t)2 * (2 * a_bytes + 2 * b_bytes) + 64 + 1024;
}

// split ntot (<= 512) into 1-2 MMA subtiles of equal width (multiple of 16, <= 256)
static void subtiles(int64_t cols, int &ntot, int &n_sub, int &nsub_w) {
  const int c16 = (int)((cols + 15) / 16) * 16;
  n_sub = c16 <= 256 ? 1 : 2;
  nsub_w = (int)(((c16 / n_sub) + 15) / 16 * 16);
  ntot = nsub_w * n_sub;
}

template <int PA, int PB, int EPI>
static void launch(Ctx &c, const Operand &A, const Operand &B, int64_t mtiles, int64_t nslab, int64_t kslab,
                   int ntot, int n_sub, int nsub_w, const EpiArgs &ep) {
  const size_t smem = smem_for(ntot);
  NM_REQUIRE(smem <= 227 * 1024, "tc_gemm: tile too wide for shared memory");
  static bool attr = false;
  if (!attr) {
    NM_CUDA(cudaFuncSetAttribute(k_tc_gemm<PA, PB, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  dim3 grid((unsigned)mtiles, (unsigned)nslab);
  NM_LAUNCH(c, EPI == STORE ? "tc_gemm_tall" : "tc_gram",
            k_tc_gemm<PA, PB, EPI><<<grid, NT, smem, c.stream>>>(A, B, ntot, n_sub, nsub_w, kslab, ep));
}

// ---------------------------------------------------------------------------
// Gram kernel: G tile (128 × 128) of Aᵀ W B over one K-slab of the n rows.
// The tensor core's fp32 accumulation truncates, so a long K chain biases sums
// of squares by ~1e-8 per row; the TMEM accumulator is therefore drained into
// fp32 registers (round-to-nearest adds) every GD K-chunks (256 rows) and the
// chain restarts.  CTAs of the same K-slab are adjacent in launch order so the
// slab's rows are read from HBM once and shared through L2.
// ---------------------------------------------------------------------------
constexpr int GN = 128;
constexpr int GD = 4;

__device__ __forceinline__ void gram_drain(uint32_t tmem, int lane_base, int cbase, float (&rs)[64]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)lane_base << 16) + (uint32_t)(cbase + 16 * j), v);
#pragma unroll
    for (int i = 0; i < 16; ++i) rs[16 * j + i] += v[i];
  }
}

__global__ void __launch_bounds__(NT, 1) k_tc_gram(Operand A, Operand B, int nta, int ntb, bool sym,
                                                   int64_t kslab, float *__restrict__ part, int64_t rows_pad,
                                                   int64_t ldp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int TB = BM * 128;  // 16 KB: one 128-row × 32-fp32 tile part
  uint8_t *st[2] = {base, base + 4 * TB};
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + 8 * TB);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2);

  // tile (ta, tb) of this CTA; CTAs of one slab are consecutive
  const int ntiles = sym ? nta * (nta + 1) / 2 : nta * ntb;
  int t = blockIdx.x % ntiles;
  const int64_t slab = blockIdx.x / ntiles;
  int ta = 0, tb = 0;
  if (sym) {
    while (t >= nta - ta) { t -= nta - ta; ++ta; }
    tb = ta + t;
  } else {
    ta = t / ntb;
    tb = t % ntb;
  }
  const int64_t m0 = (int64_t)ta * BM, n0 = (int64_t)tb * GN;
  const int64_t kbeg = slab * kslab;
  const int64_t kend = min(kbeg + kslab, A.kdim);
  const int nk = (int)((kend - kbeg + BK - 1) / BK);
  const int warp = threadIdx.x / 32;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(GN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = make_idesc(GN);
  const int lane_base = (warp & 3) * 32;
  const int cbase = (warp < 4) ? 0 : 64;
  float rs[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) rs[i] = 0.f;

  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt & 1;
    if (kt >= 2) mbar_wait(&bars[s], (uint32_t)(((kt - 2) >> 1) & 1));
    const int64_t k0 = kbeg + (int64_t)kt * BK;
    uint8_t *ahi = st[s], *alo = st[s] + TB, *bhi = st[s] + 2 * TB, *blo = st[s] + 3 * TB;
    stage_operand<TRANS>(A, m0, BM, k0, ahi, alo);
    stage_operand<TRANS>(B, n0, GN, k0, bhi, blo);
    fence_async_smem();
    __syncthreads();
    const bool chain_start = (kt % GD) == 0;
    if (chain_start && kt > 0) {
      // close the previous chain: its MMAs are complete, fold TMEM into registers
      mbar_wait(&bars[(kt - 1) & 1], (uint32_t)(((kt - 1) >> 1) & 1));
      tc_fence_after();
      gram_drain(tmem, lane_base, cbase, rs);
      tc_fence_before();
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t a_hi = smem_u32(ahi), a_lo = smem_u32(alo);
      const uint32_t b_hi = smem_u32(bhi), b_lo = smem_u32(blo);
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint32_t koff = ks * 32;
        const uint32_t acc0 = (!chain_start || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, make_desc(a_hi + koff), make_desc(b_hi + koff), idesc, acc0);
        mma_tf32(tmem, make_desc(a_hi + koff), make_desc(b_lo + koff), idesc, 1u);
        mma_tf32(tmem, make_desc(a_lo + koff), make_desc(b_hi + koff), idesc, 1u);
      }
      mma_commit(&bars[s]);
    }
    __syncwarp();
  }
  if (nk > 0) {
    mbar_wait(&bars[(nk - 1) & 1], (uint32_t)(((nk - 1) >> 1) & 1));
    tc_fence_after();
    gram_drain(tmem, lane_base, cbase, rs);
  }
  const int64_t row = m0 + lane_base + (threadIdx.x & 31);
  float *dst = part + slab * rows_pad * ldp + row * ldp + n0 + cbase;
#pragma unroll
  for (int i = 0; i < 64; i += 4) *reinterpret_cast<float4 *>(dst + i) = make_float4(rs[i], rs[i + 1], rs[i + 2], rs[i + 3]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(GN));
}

}  // namespace tc

// Bt[j][k] = (float)Bs[k][j] for the tall GEMM's B operand (K-major), zero padded
__global__ void k_transpose64to32(const double *__restrict__ Bs, int64_t ldb, int64_t K, int64_t N,
                                  float *__restrict__ Bt, int64_t ldt) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= N * ldt) return;
  int64_t j = idx / ldt, k = idx % ldt;
  Bt[idx] = (k < K) ? (float)Bs[k * ldb + j] : 0.f;
}

// C[n×b] = rs ⊙ (A[n×a] · Bs[a×b]) on tensor cores (b <= 512)
void tc_gemm_tall(Ctx &c, const Mat &A, const double *Bs, int64_t ldb, int64_t bcols, const int32_t *deg,
                  float rexp, const Mat &C) {
  using namespace tc;
  NM_REQUIRE(bcols <= 512 && A.cols <= 4096, "tc_gemm_tall: shape out of range");
  int ntot, n_sub, nsub_w;
  subtiles(bcols, ntot, n_sub, nsub_w);
  if (n_sub == 2 && smem_for(ntot) > 227 * 1024) NM_REQUIRE(false, "tc_gemm_tall: too wide");
  const int64_t K = A.cols, ldt = pad32(K);
  DBuf<float> Bt((size_t)ntot * ldt, c.stream);
  NM_CUDA(cudaMemsetAsync(Bt.p, 0, (size_t)ntot * ldt * 4, c.stream));
  NM_LAUNCH(c, "transpose64", k_transpose64to32<<<ceil_div(bcols * ldt, 256), 256, 0, c.stream>>>(Bs, ldb, K, bcols, Bt, ldt));
  Operand oa{A.p, A.ld, A.rows, K, nullptr, nullptr, 0.f};
  Operand ob{Bt.p, ldt, bcols, K, nullptr, nullptr, 0.f};
  EpiArgs ep{C.p, C.ld, C.rows, bcols, deg, rexp};
  launch<ROWS, ROWS, STORE>(c, oa, ob, ceil_div(A.rows, BM), 1, K, ntot, n_sub, nsub_w, ep);
}

__global__ void k_tc_gram_reduce(const float *__restrict__ part, int nslab, int64_t a, int64_t b,
                                 int64_t rows_pad, int64_t ldp, bool sym, double *__restrict__ G, int64_t ldg) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= a * b) return;
  int64_t i = idx / b, j = idx % b;
  if (sym && (i / tc::BM) > (j / tc::GN)) {  // lower tile: mirror of the computed upper one
    const int64_t t = i;
    i = j;
    j = t;
  }
  double s = 0.0;
  for (int t = 0; t < nslab; ++t) s += (double)part[(size_t)t * rows_pad * ldp + i * ldp + j];
  G[(idx / b) * ldg + idx % b] = s;
}

// G[a×b] (fp64) = Aᵀ W B over n rows on tensor cores (W = diag(d^-wexp) if deg)
void tc_gram(Ctx &c, const Mat &A, const Mat &B, const int32_t *deg, float wexp, double *G, int64_t ldg) {
  using namespace tc;
  NM_REQUIRE(A.rows == B.rows, "tc_gram: row mismatch");
  const int64_t n = A.rows;
  const bool sym = (A.p == B.p && A.cols == B.cols && A.ld == B.ld && deg == nullptr);
  const int nta = (int)ceil_div(A.cols, BM), ntb = (int)ceil_div(B.cols, GN);
  const int ntiles = sym ? nta * (nta + 1) / 2 : nta * ntb;
  int64_t nslab = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 2048), ceil_div((int64_t)c.num_sms * 2, ntiles)));
  int64_t kslab = (ceil_div(n, nslab) + BK - 1) / BK * BK;
  nslab = ceil_div(n, kslab);
  const int64_t rows_pad = (int64_t)nta * BM, ldp = (int64_t)ntb * GN;
  DBuf<float> part((size_t)nslab * rows_pad * ldp, c.stream);
  // operand element (row = column index of the n×c block, k = its row index)
  Operand oa{A.p, A.ld, A.cols, n, nullptr, deg, wexp};
  Operand ob{B.p, B.ld, B.cols, n, nullptr, nullptr, 0.f};
  const size_t smem = 8 * (size_t)BM * 128 + 64 + 1024;
  static bool attr = false;
  if (!attr) {
    NM_CUDA(cudaFuncSetAttribute(k_tc_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  NM_LAUNCH(c, "tc_gram", k_tc_gram<<<(unsigned)(ntiles * nslab), NT, smem, c.stream>>>(oa, ob, nta, ntb, sym, kslab,
                                                                                     part, rows_pad, ldp));
  NM_LAUNCH(c, "tc_gram_reduce", k_tc_gram_reduce<<<ceil_div(A.cols * B.cols, 256), 256, 0, c.stream>>>(
                                     part, (int)nslab, A.cols, B.cols, rows_pad, ldp, sym, G, ldg));
}

}  // namespace netmfp
