// Latency of the primitives on the tridiagonalisation's critical path (cycles, one CTA).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ long long g_out[16];
__global__ void __cluster_dims__(2, 1, 1) k_lat(double x, int n) {
  __shared__ double sh[64];
  const int tid = threadIdx.x;
  long long t0, t1;
  double a = x + tid;
  // dependent DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, 1.0000001, 0.5);
  t1 = clock64();
  if (tid == 0) g_out[0] = (t1 - t0) / n;
  // sqrt + div chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = 2.0 / sqrt(a + 1.0);
  t1 = clock64();
  if (tid == 0) g_out[1] = (t1 - t0) / n;
  // __syncthreads
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) g_out[2] = (t1 - t0) / n;
  // smem store -> sync -> load chain (block broadcast)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (tid == (i & 255)) sh[i & 63] = a;
    __syncthreads();
    a += sh[i & 63];
  }
  t1 = clock64();
  if (tid == 0) g_out[3] = (t1 - t0) / n;
  // warp_sum (5 dependent shuffles)
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  t1 = clock64();
  if (tid == 0) g_out[4] = (t1 - t0) / n;
  // cluster barrier
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  t1 = clock64();
  if (tid == 0 && cl.block_rank() == 0) g_out[5] = (t1 - t0) / n;
  // DSMEM push + cluster barrier + read
  double *peer = cl.map_shared_rank(sh, cl.block_rank() ^ 1);
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (tid < 32) peer[tid] = a;
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    a += sh[tid & 31];
  }
  t1 = clock64();
  if (tid == 0 && cl.block_rank() == 0) g_out[6] = (t1 - t0) / n;
  if (a == 12345.0) g_out[15] = 1;
}
int main() {
  for (int nt : {256, 512, 1024}) {
    k_lat<<<2, nt>>>(1.5, 200);
    cudaDeviceSynchronize();
    long long o[16];
    cudaMemcpyFromSymbol(o, g_out, sizeof(o));
    printf("threads %d: dfma %lld  sqrt+div %lld  syncthreads %lld  sts-sync-lds %lld  warp_sum %lld  cluster barrier %lld  dsmem push+barrier %lld  (%s)\n",
           nt, o[0], o[1], o[2], o[3], o[4], o[5], o[6], cudaGetErrorString(cudaGetLastError()));
  }
}
