// TMA issue/completion microbenchmark: one thread issues NB box loads (16 KB each,
// distinct smem slots of 4) either all on one mbarrier or one mbarrier per box.
#include "../../paper_2110_12782_b200/csrc/tc_gemm.cu"
#include <cstdio>
using namespace netmfp;
namespace netmfp { void set_last_error(const std::string &) {} }
using namespace netmfp::tc;

__global__ void k_issue(const __grid_constant__ CUtensorMap tm, int NB, int per_bar, unsigned long long *out, int pf,
                        const CUtensorMap *gtm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = align1024(smem_raw);
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + 8 * 16384);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap *tp = &tm;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(tp);
    for (int i = 0; i < 2000; ++i) __nanosleep(10);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    const int nbar = NB / per_bar;
    if (pf != 1) for (int b = 0; b < nbar; ++b) mbar_expect_tx(&bars[b], per_bar * 16384);
    unsigned long long t1 = clock64();
    for (int i = 0; i < NB; ++i) {
      if (pf == 1 && i % per_bar == 0) mbar_expect_tx(&bars[i / per_bar], per_bar * 16384);
      tma_load_2d(base + (i % 8) * 16384, tp, 0, (blockIdx.x * 64 + i) * 128, &bars[i / per_bar]);
    }
    unsigned long long t2 = clock64();
    for (int b = 0; b < nbar; ++b) mbar_wait(&bars[b], 0);
    unsigned long long t3 = clock64();
    out[blockIdx.x * 4 + 0] = t1 - t0;
    out[blockIdx.x * 4 + 1] = t2 - t1;
    out[blockIdx.x * 4 + 2] = t3 - t2;
  }
}

int main() {
  Ctx c; cudaStreamCreate(&c.stream);
  const int64_t rows = 148 * 64 * 128, cols = 32;
  float *A; cudaMalloc(&A, rows * cols * 4); cudaMemset(A, 0, rows * cols * 4);
  unsigned long long *o; cudaMalloc(&o, 148 * 4 * 8);
  CUtensorMap m = make_map(A, rows, cols, cols, 128, SW128, 32);
  cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int cfg[][3] = {{32, 16, 1}, {32, 1, 1}, {32, 4, 1}, {16, 16, 1}, {16, 1, 1}, {32, 16, 148}, {32, 1, 148}, {32, 8, 148}};
  CUtensorMap *gm; cudaMalloc(&gm, sizeof(CUtensorMap)); cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  for (int pf = 0; pf < 2; ++pf)
  for (auto &cf : cfg) {
    printf("pf=%d ", pf);
    for (int rep = 0; rep < 2; ++rep) {
      k_issue<<<cf[2], 32, 8 * 16384 + 1024 + 1024, c.stream>>>(m, cf[0], cf[1], o, pf, gm);
      cudaStreamSynchronize(c.stream);
    }
    unsigned long long h[4];
    cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
    printf("NB=%d per_bar=%d ctas=%d: expect %llu  issue %llu (%.0f/box)  wait %llu (%.0f/box)  %s\n", cf[0], cf[1],
           cf[2], h[0], h[1], (double)h[1] / cf[0], h[2], (double)(h[1] + h[2]) / cf[0],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
