// Random row-gather throughput: every warp reads 512-B rows (one float4 per
// lane) at pseudo-random row indices of an rows x 128 fp32 table, 4 rows in
// flight per warp.  Reports delivered bytes/s (the SpMM's gather roofline).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int ILP>
__global__ void k_gather(const float4 *__restrict__ X, uint32_t rows, int iters, float4 *out) {
  const int lane = threadIdx.x & 31;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = 0; i < iters; ++i) {
    float4 v[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      const uint32_t r = hash32(w * 7919u + (uint32_t)(i * ILP + u) * 104729u) % rows;
      v[u] = __ldg(X + (size_t)r * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < ILP; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  if (acc.x == 12345.f) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t maxrows = 1 << 20;  // 512 MB table
  float4 *X, *out;
  cudaMalloc(&X, maxrows * 512); cudaMemset(X, 0, maxrows * 512); cudaMalloc(&out, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int ilp, uint32_t rows, int bps) {
    const int grid = sms * bps, iters = 1600 / ilp;
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      kern<<<grid, 256>>>(X, rows, iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)grid * 8 * iters * ilp * 512;
    printf("table %7.1f MB  ILP %2d blocks/SM %d: %.2f TB/s %s\n", rows * 512.0 / 1e6, ilp, bps, bytes / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  // table sizes of profiles/r01_gather_roofline.txt (8.4 MB .. 537 MB; 406727 rows =
  // one 128-column pass of configs[2]'s compacted X), then the ILP sweep at 208 MB
  for (uint32_t rows : {16384u, 65536u, 131072u, 200000u, 262144u, 406727u, 1048576u})
    for (int bps : {4, 8}) run(k_gather<4>, 4, rows, bps);
  for (int bps : {2, 4, 8}) {
    run(k_gather<8>, 8, 406727u, bps);
    run(k_gather<16>, 16, 406727u, bps);
  }
  return 0;
}
