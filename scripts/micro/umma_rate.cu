// Microbenchmark: tcgen05.mma (kind::f16, bf16 in, fp32 accumulate,
// cta_group::1, M = 128) issue-to-completion rate per SM for the operand
// placements the attention kernels use:
//   SS   A and B from shared memory (128B-swizzled, K-major)
//   TS   A from TMEM, B from shared memory (K-major or MN-major)
// for N in {64, 128, 256}, optionally with W "noise" warps streaming LDS.128
// from another 64 KB smem region (the compute warps' shared-memory traffic)
// or with a TMA-like bulk copy stream into smem.  One CTA per SM (148 CTAs);
// prints clocks per MMA (the floor is 128 N / 256 clk) and the implied
// shared-memory operand bytes per clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_rate umma_rate.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_22234_b200/csrc/sm100.cuh"
using namespace bd;

constexpr int kA = 0;             // A tile: 128 rows x 128 K (2 x 16 KB)
constexpr int kB = 32768;         // B tile: 256 rows x 128 K (2 x 32 KB) -- N <= 256
constexpr int kNoise = 98304;     // 64 KB read by the noise warps
constexpr int kSmem = kNoise + 65536 + 1024 + 64;

template <int N, bool TS, bool BMN>
__global__ void __launch_bounds__(32 * 9, 1) k_umma(long long* out, int n_mma, int noise_warps, float* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kNoise + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  volatile uint32_t* stop = slot + 1;
  const int warp = warp_id(), lane = lane_id();
  for (int i = threadIdx.x; i < (kNoise + 65536) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tmem_alloc<512>(slot);
  if (threadIdx.x == 32) {
    mbar_init(bar, 1);
    *stop = 0;
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = *slot;
  if (warp == 0) {
    if (elect_one()) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, BMN);
      const uint32_t a = smem_u32(sm + kA), b = smem_u32(sm + kB);
      long long t0 = clock64();
      for (int i = 0; i < n_mma; ++i) {
        const int k = i & 7;
        const uint64_t bd = BMN ? umma_desc_sw128(b + k * 2048, 16384, 1024)
                                : umma_desc_sw128(b + (k >> 2) * 32768 + (k & 3) * 32, 16, 1024);
        if (TS)
          umma_ts(tb + 256, tb + 128 + k * 8, bd, idesc, i > 0);  // D at 256.., A at 128..191
        else
          umma_ss(tb + 256, umma_desc_sw128(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), bd, idesc, i > 0);
      }
      umma_commit(bar);
      mbar_wait(bar, 0);
      long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
      *stop = 1;
    }
  } else if (warp <= noise_warps) {
    // shared-memory traffic: LDS.128 over 64 KB, conflict-free
    float acc = 0.f;
    const uint4* src = reinterpret_cast<const uint4*>(sm + kNoise);
    int it = 0;
    while (*stop == 0) {
#pragma unroll 8
      for (int u = 0; u < 32; ++u) {
        const uint4 v = src[((it * 32 + u) * 32 + lane) & 4095];
        acc += __uint_as_float(v.x ^ v.w);
      }
      ++it;
    }
    if (acc == 1.2345f) sink[threadIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int N, bool TS, bool BMN>
void run(const char* name, int noise) {
  long long* d;
  float* s;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&s, 4096 * 4);
  cudaFuncSetAttribute(k_umma<N, TS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) k_umma<N, TS, BMN><<<148, 32 * 9, kSmem>>>(d, n, noise, s);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0, sum = 0;
  for (int i = 0; i < 148; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    sum += h[i];
  }
  const double cyc = (double)sum / 148 / n;
  const double floor_ = 128.0 * N / 256.0;
  const double bytes = (TS ? 0 : 128 * 16 * 2) + N * 16 * 2;
  printf("%-22s N=%3d noise_warps=%d: %6.1f clk/MMA (floor %5.1f, %.2fx), smem operands %.1f B/clk  [%s]\n", name,
         N, noise, cyc, floor_, cyc / floor_, bytes / cyc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  cudaFree(s);
}

int main() {
  for (int noise : {0, 4, 8}) {
    run<64, false, false>("SS", noise);
    run<128, false, false>("SS", noise);
    run<256, false, false>("SS", noise);
    run<64, true, false>("TS (A in TMEM)", noise);
    run<128, true, false>("TS (A in TMEM)", noise);
    run<256, true, false>("TS (A in TMEM)", noise);
    run<128, true, true>("TS, B MN-major", noise);
    run<128, false, true>("SS, B MN-major", noise);
  }
  return 0;
}
