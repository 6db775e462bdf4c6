// Microbenchmark: tcgen05.ld throughput per SM (32x32b.x32: 32 lanes x 32
// columns x 4 B = 4 KB per warp instruction).  W warps (W/4 per lane quarter)
// each issue N loads of 32 columns (cycling over 512 columns) with a wait
// after every G loads; prints clocks and bytes/clk per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_22234_b200/csrc/sm100.cuh"
using namespace bd;

template <int G>
__global__ void __launch_bounds__(512, 1) k_tmem(long long* out, int n, float* sink) {
  __shared__ uint32_t slot;
  if (warp_id() == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot + ((uint32_t)((warp_id() & 3) * 32) << 16);
  uint32_t r[G][32];
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; i += G) {
#pragma unroll
    for (int g = 0; g < G; ++g) tmem_ld32(t + (((i + g) * 32) & 511), r[g]);
    tmem_ld_wait();
#pragma unroll
    for (int g = 0; g < G; ++g) acc += __uint_as_float(r[g][g & 31]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(slot);
}

template <int G>
void run(int warps) {
  long long* d; float* s;
  cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4096);
  const int n = 4096;
  k_tmem<G><<<148, 32 * warps>>>(d, n, s);
  k_tmem<G><<<148, 32 * warps>>>(d, n, s);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes = (double)warps * n * 4096;
  printf("warps %2d, %d loads per wait: %lld clk, %.1f B/clk/SM (%s)\n", warps, G, h[0], bytes / h[0],
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d); cudaFree(s);
}

int main() {
  for (int w : {4, 8, 16}) { run<1>(w); run<4>(w); }
  return 0;
}
