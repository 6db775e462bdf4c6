// Microbenchmark: does a warp issuing tcgen05.mma slow down the other warps
// on its SM sub-partition?  One CTA per SM, 8 warps: warp 0 (sub-partition 0)
// either idles, spins on an mbarrier try_wait, or issues back-to-back
// tcgen05.mma (kind::f16, M = 128, N = 128, K = 16, A from TMEM, B from smem)
// until told to stop; warps 4-7 (one per sub-partition 0-3) each run the same
// fixed ALU loop (FFMA2 + MUFU ex2, a softmax-like mix) and record its
// clock64 duration.  Prints the mean duration per sub-partition.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_issue_cost mma_issue_cost.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_22234_b200/csrc/sm100.cuh"
using namespace bd;

constexpr int kSmem = 65536 + 1024 + 64;

__global__ void __launch_bounds__(32 * 8, 1) k(long long* out, int mode, int iters, float* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  volatile int* done = reinterpret_cast<volatile int*>(slot + 1);  // ALU warps finished
  const int warp = warp_id(), lane = lane_id();
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tmem_alloc<512>(slot);
  if (threadIdx.x == 32) {
    mbar_init(bar, 1);
    *done = 0;
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = *slot;
  if (warp == 0) {
    if (elect_one()) {
      if (mode == 1) {
        // spin on a barrier that never completes until stop
        while (*done < 4) {
          mbar_test(bar, 0);
        }
      } else if (mode == 2) {
        constexpr uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
        const uint32_t b = smem_u32(sm);
        int i = 0;
        while (*done < 4) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t bd = umma_desc_sw128(b + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
            umma_ts(tb + 256, tb + 128 + k * 8, bd, idesc, (i | k) > 0);
          }
          ++i;
        }
        umma_commit(bar);
        mbar_wait(bar, 0);
      }
    }
  } else if (warp >= 4) {
    float2 a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = make_float2(0.001f * (lane + j), 0.002f * j);
    const float2 m = make_float2(0.999f, 0.999f), c = make_float2(0.0001f, 0.0001f);
    float s = 0.f;
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a[j] = ffma2(a[j], m, c);
        s += ex2_approx(a[j].x);
      }
    }
    const long long t1 = clock64();
    float t = s;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += a[j].x + a[j].y;
    if (t == 1.2345f) sink[threadIdx.x] = t;
    if (lane == 0) {
      out[blockIdx.x * 4 + (warp - 4)] = t1 - t0;
      atomicAdd(const_cast<int*>(done), 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  long long* d;
  float* s;
  cudaMalloc(&d, 148 * 4 * 8);
  cudaMalloc(&s, 4096 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  const char* names[3] = {"idle issuer", "spinning issuer (test_wait)", "issuing tcgen05.mma"};
  for (int mode = 0; mode < 3; ++mode) {
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) k<<<148, 256, kSmem>>>(d, mode, iters, s);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148 * 4];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double per[4] = {0, 0, 0, 0};
    for (int b = 0; b < 148; ++b)
      for (int w = 0; w < 4; ++w) per[w] += (double)h[b * 4 + w] / 148;
    printf("%-30s ALU warp clocks per sub-partition: %8.0f %8.0f %8.0f %8.0f  [%s]\n", names[mode], per[0], per[1],
           per[2], per[3], cudaGetErrorString(e));
  }
  return 0;
}
