// MUFU ex2 throughput per SM by operand type (dev microbenchmark): f32,
// f16x2 and bf16x2 (two results per lane per instruction), 8 independent
// chains per thread, one CTA per SM; results counted per element.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate2 mufu_rate2.cu && ./mufu_rate2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__device__ __forceinline__ uint32_t ex2op(uint32_t x) {
  uint32_t y;
  if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=r"(y) : "r"(x));
  if (KIND == 1) asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  if (KIND == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int KIND>
__global__ void k(uint32_t* out, long long* clk, int iters) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 0x3c00bc00u ^ (threadIdx.x + i);  // modest values
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ex2op<KIND>(a[i]) ^ 0x80008000u;  // sign flip keeps values bounded
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, int warps) {
  uint32_t* out;
  long long* clk;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&clk, 1 << 16);
  const int iters = 4096;
  k<KIND><<<148, 32 * warps>>>(out, clk, iters);
  k<KIND><<<148, 32 * warps>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += h[i];
  mean /= 148;
  const double elems = 32.0 * warps * iters * 8 * (KIND ? 2 : 1);
  printf("%-8s warps/SM %2d: %.1f exp results / clk / SM (%.1f instr / clk / SM)  [%s]\n", name, warps, elems / mean,
         elems / mean / (KIND ? 2 : 1), cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("f32", w);
    run<1>("f16x2", w);
    run<2>("bf16x2", w);
  }
  return 0;
}
