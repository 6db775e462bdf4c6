// Microbenchmark: the forward softmax's exp phase for ONE warp per SM
// sub-partition (and two), with the row read from and the packed P written
// to shared memory each iteration (standing in for tcgen05.ld / st).  Per
// pair of scores:
//   V0: x = FFMA2(s, sl2, -m); p = 2 x MUFU ex2; sum FADD2; pack F2FP  (the kernel)
//   V1: x = FADD2(s, -m)      (log2 e / sqrt(d) folded into Q upstream)
//   V2: x = s                 (no argument op: the MUFU / pack / sum floor)
//   V3: V0 with every 4th pair on the FMA-pipe polynomial (the kernel's split)
// Prints clocks per row per warp and per MUFU instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o softmax_mix softmax_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_22234_b200/csrc/sm100.cuh"
using namespace bd;

template <int V>
__global__ void k(long long* out, int iters, float mshift) {
  extern __shared__ __align__(16) uint8_t dyn[];
  auto sS = reinterpret_cast<float (*)[128 + 4]>(dyn);                          // one row per thread
  auto sP = reinterpret_cast<uint32_t (*)[64 + 4]>(dyn + 256 * (128 + 4) * 4);  // (8 warps max)
  const int t = threadIdx.x;
  for (int c = 0; c < 128; ++c) sS[t][c] = -0.01f * (float)((t * 7 + c * 13) & 255);
  __syncthreads();
  const float2 sl2v = make_float2(1.0f, 1.0f), nm = make_float2(-mshift, -mshift);
  float tot = 0.f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float s[128];
#pragma unroll
    for (int c = 0; c < 128; c += 4) {
      const float4 v = *reinterpret_cast<const float4*>(&sS[t][c]);
      s[c] = v.x; s[c + 1] = v.y; s[c + 2] = v.z; s[c + 3] = v.w;
    }
    float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    uint32_t pk[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      float2 x;
      if (V == 0 || V == 3) x = ffma2(make_float2(s[2 * c], s[2 * c + 1]), sl2v, nm);
      if (V == 1) x = fadd2(make_float2(s[2 * c], s[2 * c + 1]), nm);
      if (V == 2) x = make_float2(s[2 * c], s[2 * c + 1]);
      float2 p;
      if (V == 3 && (c % 4) == 3) p = ex2_poly2(x);
      else p = make_float2(ex2_approx(x.x), ex2_approx(x.y));
      acc[c & 3] = fadd2(acc[c & 3], p);
      pk[c] = pack_bf16x2(p.x, p.y);
    }
#pragma unroll
    for (int c = 0; c < 64; c += 4)
      *reinterpret_cast<uint4*>(&sP[t][c]) = make_uint4(pk[c], pk[c + 1], pk[c + 2], pk[c + 3]);
    const float2 a01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    tot += a01.x + a01.y;
    __syncwarp();
  }
  const long long t1 = clock64();
  if (tot == 1.2345f) sP[t][0] = 1;
  if ((t & 31) == 0) out[blockIdx.x * 32 + (t >> 5)] = t1 - t0;
}

template <int V>
void run(const char* name, int warps) {
  long long* d;
  cudaMalloc(&d, 148 * 32 * 8);
  const int iters = 256;
  const int smem = 256 * (128 + 4) * 4 + 256 * (64 + 4) * 4;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 2; ++r) k<V><<<148, 32 * warps, smem>>>(d, iters, 0.5f);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < warps; ++w) mean += (double)h[b * 32 + w] / (148.0 * warps);
  const double mufu = V == 3 ? 96.0 : 128.0;
  printf("%-44s warps/SM %d: %7.1f clk per row per warp, %5.2f clk per MUFU instr  [%s]\n", name, warps,
         mean / iters, mean / iters / mufu, cudaGetErrorString(e));
}

int main() {
  for (int w : {4, 8}) {
    run<0>("V0 FFMA2 -> 2 MUFU, FADD2 sum, F2FP", w);
    run<1>("V1 FADD2 -> 2 MUFU (scale folded in Q)", w);
    run<2>("V2 no argument op", w);
    run<3>("V3 V0 + 1/4 polynomial", w);
  }
  return 0;
}
