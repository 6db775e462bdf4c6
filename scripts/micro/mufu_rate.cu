// MUFU ex2 throughput per SM (dev microbenchmark): each thread runs N
// independent chains of ex2.approx.ftz.f32 (8 chains keep the pipe full);
// clock64 around the loop, ops / clk / SM reported for several warp counts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu && ./mufu_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void k(float* out, long long* clk, int iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ex2(a[i]) - 1.0f;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&clk, 1 << 16);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    k<<<148, 32 * warps>>>(out, clk, iters);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i];
    mean /= 148;
    const double ops = 32.0 * warps * iters * 8;  // ex2 per SM (one CTA per SM)
    printf("warps/SM %2d: %.1f ex2 / clk / SM (FADD in the chain too)\n", warps, ops / mean);
  }
  return 0;
}
