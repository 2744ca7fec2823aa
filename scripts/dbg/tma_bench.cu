// TMA streaming throughput microbenchmark: one CTA per SM pulls boxes of a
// [rows][cols] fp32 matrix (L2-resident or not) into an S-stage smem ring.
#include "../../paper_2110_12782_b200/csrc/tc_gemm.cu"
#include <cstdio>
using namespace netmfp;
namespace netmfp { void set_last_error(const std::string &) {} }
using namespace netmfp::tc;

__device__ __forceinline__ void mbar_wait_test(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAITT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAITT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_relaxed(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
template <bool WHOLE>
__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap tm, int box_bytes, int boxes_per_stage,
                                                int S, int iters, int box_cols, int box_rows, int nbox_r, int nbox_c,
                                                unsigned long long *cycles, const float *src) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = align1024(smem_raw);
  const int stage_bytes = box_bytes * boxes_per_stage;
  uint64_t *full = reinterpret_cast<uint64_t *>(base + S * stage_bytes);
  uint64_t *empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (WHOLE && warp == 0 && lane == 0) {
    for (int g = 0; g < iters + S; ++g) {
      const int s = g % S, use = g / S;
      if (use > 0) mbar_wait(&full[s], (use - 1) & 1);
      if (g >= iters) continue;
      mbar_expect_tx(&full[s], stage_bytes);
      for (int b = 0; b < boxes_per_stage; ++b) {
        const int idx = (blockIdx.x * 7 + g * boxes_per_stage + b);
        const int bc = idx % nbox_c, br = (idx / nbox_c) % nbox_r;
        tma_load_2d(base + s * stage_bytes + b * box_bytes, &tm, bc * box_cols, br * box_rows, &full[s]);
      }
    }
    cycles[blockIdx.x] = clock64() - t0;
  } else if (!WHOLE && warp == 0 && lane == 0) {
    for (int g = 0; g < iters; ++g) {
      const int s = g % S, use = g / S;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      if (lane == 0) {
        mbar_expect_tx(&full[s], stage_bytes);
        for (int b = 0; b < boxes_per_stage; ++b) {
          const int idx = (blockIdx.x * 7 + g * boxes_per_stage + b);
          {
            const int bc = idx % nbox_c, br = (idx / nbox_c) % nbox_r;
            if (WHOLE) tma_load_2d_hint(base + s * stage_bytes + b * box_bytes, &tm, bc * box_cols, br * box_rows, &full[s]);
            else tma_load_2d(base + s * stage_bytes + b * box_bytes, &tm, bc * box_cols, br * box_rows, &full[s]);
          }
        }
      }
      
    }
  } else if (!WHOLE && warp == 1 && lane == 0) {
    for (int g = 0; g < iters; ++g) {
      const int s = g % S, use = g / S;
      if (false) {
        uint32_t ok = 0;
        while (true) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                       : "=r"(ok) : "r"(smem_u32(&full[s])), "r"((uint32_t)(use & 1)) : "memory");
          if (ok) break;
          __nanosleep(64);
        }
      } else {
        mbar_wait(&full[s], use & 1);
      }
      if (lane == 0) mbar_arrive(&empty[s]);
      
    }
    if (lane == 0) cycles[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
}

int main() {
  Ctx c; cudaStreamCreate(&c.stream);
  const int64_t rows = 1 << 16, cols = 256;  // 64 MB, L2 resident
  float *A; cudaMalloc(&A, rows * cols * 4); cudaMemset(A, 0, rows * cols * 4);
  unsigned long long *cyc; cudaMalloc(&cyc, 148 * 8);
  struct Cfg { int bc, br; MapSwizzle sw; int bps; int S; const char *name; } cfgs[] = {
      {32, 128, SW128, 1, 1, "32x128 x1 S1"}, {32, 128, SW128, 1, 2, "32x128 x1 S2"},
      {32, 128, SW128, 1, 4, "32x128 x1 S4"}, {32, 128, SW128, 1, 8, "32x128 x1 S8"},
      {32, 128, SW128, 1, 12, "32x128 x1 S12"}, {32, 64, SW128, 1, 16, "32x64 x1 S16"},
      {32, 128, SW128, 4, 2, "32x128 x4 S2"}, {32, 256, SW128, 2, 3, "32x256 x2 S3"},
      {32, 256, SW128, 3, 2, "32x256 x3 S2"}, {32, 128, SW128, 1, 8, "c32x128 x1 S8"}};
  cudaFuncSetAttribute(k_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int whole = 0; whole < 2; ++whole)
  for (int resident = 1; resident < 2; ++resident) {
  const int64_t rws = resident ? rows : rows * 16;
  float *B = A;
  if (!resident) { cudaMalloc(&B, rws * cols * 4); cudaMemset(B, 0, rws * cols * 4); }
  printf("--- %s %s\n", resident ? "L2-resident 64 MB" : "1 GB (HBM)", whole ? "single-thread ring (no consumer)" : "producer/consumer");
  for (auto &cf : cfgs) {
    const bool contig = cf.name[0] == 'c';
    CUtensorMap m = contig ? make_map(B, rws * cols / 32, 32, 32, cf.br, cf.sw, cf.bc)
                           : make_map(B, rws, cols, cols, cf.br, cf.sw, cf.bc);
    const int box_bytes = cf.bc * cf.br * 4;
    const int iters = 4000 / cf.bps;
    size_t smem = 1024 + (size_t)cf.S * box_bytes * cf.bps + 256;
    if (smem > 227 * 1024) continue;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, c.stream);
      if (whole == 3) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(148); lc.blockDim = dim3(128); lc.dynamicSmemBytes = smem; lc.stream = c.stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        lc.attrs = at; lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, k_tma<false>, m, box_bytes, cf.bps, cf.S, iters, cf.bc, cf.br,
                           contig ? (int)(rws * cols / 32 / cf.br) : (int)(rws / cf.br), contig ? 1 : (int)(cols / cf.bc), cyc,
                           (const float *)B);
      } else
      if (whole) k_tma<true><<<148, 128, smem, c.stream>>>(m, box_bytes, cf.bps, cf.S, iters, cf.bc, cf.br, (int)(rws / cf.br),
                                          (int)(cols / cf.bc), cyc, B);
      else k_tma<false><<<148, 128, smem, c.stream>>>(m, box_bytes, cf.bps, cf.S, iters, cf.bc, cf.br,
                                          contig ? (int)(rws * cols / 32 / cf.br) : (int)(rws / cf.br),
                                          contig ? 1 : (int)(cols / cf.bc), cyc, B);
      cudaEventRecord(e1, c.stream);
      cudaStreamSynchronize(c.stream);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long hc[148]; cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    double bytes = (double)148 * iters * box_bytes * cf.bps;
    printf("%-22s %s  %.3f ms  %.2f TB/s  %.1f B/cyc/SM  %.0f cyc/box\n", cf.name, cudaGetErrorString(cudaGetLastError()),
           ms, bytes / ms / 1e9, (double)iters * box_bytes * cf.bps / hc[0], (double)hc[0] / (iters * cf.bps));
  }
  }
  return 0;
}
