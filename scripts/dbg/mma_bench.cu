// tcgen05.mma kind::tf32 issue-rate microbenchmark: one CTA per SM issues NI MMAs
// (M=128, N given, K=8) from resident operands (smem B, smem or TMEM A), commit, wait.
#include "../../paper_2110_12782_b200/csrc/tc_gemm.cu"
#include <cstdio>
using namespace netmfp;
using namespace netmfp::tc;
namespace netmfp { void set_last_error(const std::string &) {} }

__global__ void __launch_bounds__(128, 1) k_mma(int N, int NI, int ts, int nacc, unsigned long long *cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = align1024(smem_raw);
  uint64_t *bar = reinterpret_cast<uint64_t *>(base + 128 * 1024);
  uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 1);
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<float *>(base)[i] = 1.0f;
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  if (threadIdx.x < 32) tmem_alloc(slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    // lean loop: all descriptors / addresses precomputed, 4 MMAs per iteration
    const uint32_t a = smem_u32(base), b = smem_u32(base + 32768);
    const uint32_t idesc = ts == 2 ? make_idesc(N, 1, 1) : make_idesc(N, 0, 0);
    uint64_t da[4], db[4];
    uint32_t dd[4];
    for (int t = 0; t < 4; ++t) {
      da[t] = ts == 2 ? make_desc_mn32(a + t * 1024, 4096) : make_desc(a + t * 32, 16, 1024);
      db[t] = ts == 2 ? make_desc_mn32(b + t * 1024, 4096) : make_desc(b + t * 32, 16, 1024);
      dd[t] = tmem + (uint32_t)((t % (nacc < 0 ? -nacc : nacc)) * (N <= 128 ? 128 : 192)) % 384;
    }
    unsigned long long t0 = clock64();
    const uint32_t ta = tmem + 384;
    if (ts == 1) {
      for (int i = 0; i < NI; i += 4) {
        mma_tf32_ts(dd[0], ta, db[0], idesc, i > 0);
        mma_tf32_ts(dd[1], ta + 8, db[1], idesc, i > 0);
        mma_tf32_ts(dd[2], ta + 16, db[2], idesc, i > 0);
        mma_tf32_ts(dd[3], ta + 24, db[3], idesc, i > 0);
      }
    } else {
      for (int i = 0; i < NI; i += 4) {
        mma_tf32(dd[0], da[0], db[0], idesc, i > 0);
        mma_tf32(dd[1], da[1], db[1], idesc, i > 0);
        mma_tf32(dd[2], da[2], db[2], idesc, i > 0);
        mma_tf32(dd[3], da[3], db[3], idesc, i > 0);
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long *cyc; cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  struct C { int ts, N, nacc; } cs[] = {{0, 144, 1}, {1, 144, 1}, {1, 144, 2}, {0, 128, 1}, {1, 128, 1},
                                      {1, 64, 1}, {0, 256, 1}, {1, 256, 1}, {1, 32, 1},
                                      {2, 256, 1}, {2, 160, 1}, {2, 32, 1}, {2, 128, 1}, {0, 32, 1}, {0, 160, 1},
                                      {2, 128, 2}, {2, 128, 4}, {2, 256, 2}, {0, 128, 4}, {0, 256, 2}};
  for (auto &cc : cs) {
    const int NI = 4096;
    for (int rep = 0; rep < 2; ++rep) k_mma<<<148, 128, 140 * 1024>>>(cc.N, NI, cc.ts, cc.nacc, cyc);
    cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double flops = 2.0 * 128 * cc.N * 8 * NI * 148;
    printf("%s N=%3d nacc=%d: %.1f cycles/MMA (%s) %.0f TFLOP/s tf32 @1.9GHz\n", cc.ts == 1 ? "TS" : cc.ts == 2 ? "MN" : "SS", cc.N, cc.nacc,
           (double)h[0] / NI, cudaGetErrorString(cudaGetLastError()), flops / ((double)h[0] / 1.9e9) / 1e12);
  }
  return 0;
}
