// Hardware self-test of the UMMA / TMEM / TMA conventions used by the
// attention kernels (see sm100.cuh header comment).  One CTA, 128 threads:
//   C    = A . B^T                      (SS, both K-major; B via TMA)
//   O_ts = bf16(C) . V                  (A = P in TMEM, V MN-major via TMA)
//   O_ss = bf16(C) . V                  (A = P in smem, K-major, thread-written)
//   O_mn = bf16(C) . V                  (A = P^T in smem, i.e. MN-major A)
// A, B, V are [128][128] bf16 row-major.  Exported as bd_selftest_mma.
#include "sm100.cuh"
#include "tma_host.h"
#include "abi_common.h"

#include <cuda_bf16.h>

namespace bd {
namespace {

constexpr uint32_t kTile = 128 * 128 * 2;  // 32 KB

__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __nv_bfloat16* __restrict__ A, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmV, float* __restrict__ C, float* __restrict__ Ots,
                    float* __restrict__ Oss, float* __restrict__ Omn) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kTile;
  uint8_t* sV = smem + 2 * kTile;
  uint8_t* sP = smem + 3 * kTile;
  uint8_t* sPt = smem + 4 * kTile;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 5 * kTile);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  const uint32_t tid = threadIdx.x, w = warp_id();

  if (w == 0) tmem_alloc<512>(tslot);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  // A -> smem, K-major SW128, written by threads (row = tid)
  for (int kb = 0; kb < 2; ++kb)
    for (int c = 0; c < 8; ++c) {
      const uint4 v = *reinterpret_cast<const uint4*>(A + tid * 128 + kb * 64 + c * 8);
      *reinterpret_cast<uint4*>(sA + kb * 16384 + sw128_offset(tid, c)) = v;
    }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (tid == 0) {
    mbar_expect_tx(&bars[0], 2 * kTile);
    for (int kb = 0; kb < 2; ++kb) {
      tma_load_2d(sB + kb * 16384, &tmB, &bars[0], kb * 64, 0);
      tma_load_2d(sV + kb * 16384, &tmV, &bars[0], kb * 64, 0);
    }
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    const uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
    for (int k = 0; k < 8; ++k) {
      const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
      umma_ss(tbase, umma_desc_sw128(smem_u32(sA) + off, 16, 1024), umma_desc_sw128(smem_u32(sB) + off, 16, 1024),
              idesc, k > 0);
    }
    umma_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[1], 0);
  tc_fence_after();

  const uint32_t row = tid;
  const uint32_t lane_base = (w * 32) << 16;
  float p[128];
  for (int cb = 0; cb < 4; ++cb) {
    uint32_t r[32];
    tmem_ld32(tbase + lane_base + cb * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) {
      const float f = __uint_as_float(r[j]);
      C[row * 128 + cb * 32 + j] = f;
      p[cb * 32 + j] = f;
    }
  }
  uint32_t pk[64];
  for (int j = 0; j < 64; ++j) pk[j] = pack_bf16x2(p[2 * j], p[2 * j + 1]);
  // P -> TMEM columns [128, 192)
  for (int cb = 0; cb < 4; ++cb) tmem_st16(tbase + lane_base + 128 + cb * 16, pk + cb * 16);
  tmem_st_wait();
  // P -> smem K-major (row = m)
  for (int kb = 0; kb < 2; ++kb)
    for (int c = 0; c < 8; ++c) {
      uint4 v = make_uint4(pk[kb * 32 + c * 4 + 0], pk[kb * 32 + c * 4 + 1], pk[kb * 32 + c * 4 + 2],
                           pk[kb * 32 + c * 4 + 3]);
      *reinterpret_cast<uint4*>(sP + kb * 16384 + sw128_offset(row, c)) = v;
    }
  // P^T -> smem MN-major: element (m=row, k) at row k of M-block row/64
  {
    const uint32_t mb = row >> 6, mc = (row & 63) >> 3, me = row & 7;
    for (int k = 0; k < 128; ++k) {
      const uint16_t bits = (k & 1) ? (pk[k >> 1] >> 16) : (pk[k >> 1] & 0xFFFF);
      *reinterpret_cast<uint16_t*>(sPt + mb * 16384 + sw128_offset(k, mc) + me * 2) = bits;
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (tid == 0) {
    const uint32_t idesc_ts = umma_idesc_bf16(128, 128, false, true);
    for (int k = 0; k < 8; ++k)
      umma_ts(tbase + 256, tbase + 128 + k * 8, umma_desc_sw128(smem_u32(sV) + k * 2048, 16384, 1024), idesc_ts,
              k > 0);
    for (int k = 0; k < 8; ++k) {
      const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
      umma_ss(tbase + 384, umma_desc_sw128(smem_u32(sP) + off, 16, 1024),
              umma_desc_sw128(smem_u32(sV) + k * 2048, 16384, 1024), idesc_ts, k > 0);
    }
    const uint32_t idesc_mn = umma_idesc_bf16(128, 128, true, true);
    for (int k = 0; k < 8; ++k)
      umma_ss(tbase, umma_desc_sw128(smem_u32(sPt) + k * 2048, 16384, 1024),
              umma_desc_sw128(smem_u32(sV) + k * 2048, 16384, 1024), idesc_mn, k > 0);
    umma_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[1], 1);
  tc_fence_after();
  for (int cb = 0; cb < 4; ++cb) {
    uint32_t r[32];
    tmem_ld32(tbase + lane_base + 256 + cb * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) Ots[row * 128 + cb * 32 + j] = __uint_as_float(r[j]);
    tmem_ld32(tbase + lane_base + 384 + cb * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) Oss[row * 128 + cb * 32 + j] = __uint_as_float(r[j]);
    tmem_ld32(tbase + lane_base + cb * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) Omn[row * 128 + cb * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tbase);
}

}  // namespace
}  // namespace bd

extern "C" int bd_selftest_mma(const void* a, const void* b, const void* v, float* c, float* o_ts, float* o_ss,
                               float* o_mn, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  using namespace bd;
  if (!a || !b || !v || !c || !o_ts || !o_ss || !o_mn) return BD_ERR_INVALID_ARG;
  CUtensorMap tmB, tmV;
  const uint64_t dims[2] = {128, 128}, strides[1] = {256};
  const uint32_t box[2] = {64, 128};
  if (!make_tmap_bf16(&tmB, b, 2, dims, strides, box) || !make_tmap_bf16(&tmV, v, 2, dims, strides, box))
    return BD_ERR_CUDA;
  const int smem = 5 * kTile + 64 + 1024;
  if (cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return BD_ERR_CUDA;
  selftest_kernel<<<1, 128, smem, stream>>>(reinterpret_cast<const __nv_bfloat16*>(a), tmB, tmV, c, o_ts, o_ss,
                                            o_mn);
  note_launches(1);
  return cudaGetLastError() == cudaSuccess ? BD_OK : BD_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// Diagnostic: TMA ingest bandwidth.  Every CTA streams 32 KB tiles (two
// 64x128 bf16 boxes of a [rows, 128] tensor, 4-D map like the attention
// operands: row stride `row_stride_elems`) through `stages` smem slots;
// cycles[blockIdx] = clock64 span, bytes per CTA = iters * 32 KB.
namespace bd {
namespace {
__global__ void __launch_bounds__(64, 1)
    tma_bw_kernel(const __grid_constant__ CUtensorMap tm, int n_tiles, int iters, int stages, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 6 * 32768);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    const int start = (blockIdx.x * 7) % n_tiles;
    for (int s = 0; s < stages && s < iters; ++s) {
      mbar_expect_tx(&full[s], 32768);
      const int t = (start + s) % n_tiles;
      tma_load_4d(smem + s * 32768, &tm, &full[s], 0, 0, t * 128, 0);
      tma_load_4d(smem + s * 32768 + 16384, &tm, &full[s], 64, 0, t * 128, 0);
    }
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      const int nx = i + stages;
      if (nx < iters) {
        mbar_expect_tx(&full[s], 32768);
        const int t = (start + nx) % n_tiles;
        tma_load_4d(smem + s * 32768, &tm, &full[s], 0, 0, t * 128, 0);
        tma_load_4d(smem + s * 32768 + 16384, &tm, &full[s], 64, 0, t * 128, 0);
      }
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
}
}  // namespace
}  // namespace bd

extern "C" int bd_bench_tma(const void* src, int64_t rows, int heads, int grid, int iters, int stages,
                            long long* cycles, void* stream_) {
  using namespace bd;
  CUtensorMap tm;
  // [rows, heads, 128] bf16 viewed as dims (128, heads, rows, 1), box (64, 1, 128, 1)
  const uint64_t dims[4] = {128, (uint64_t)heads, (uint64_t)rows, 1};
  const uint64_t strides[3] = {256, (uint64_t)heads * 256, (uint64_t)rows * heads * 256};
  const uint32_t box[4] = {64, 1, 128, 1};
  if (!make_tmap_bf16(&tm, src, 4, dims, strides, box)) return BD_ERR_CUDA;
  if (stages < 1 || stages > 6) return BD_ERR_INVALID_ARG;
  const int smem = 6 * 32768 + 64 + 1024;
  cudaFuncSetAttribute(tma_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tma_bw_kernel<<<grid, 64, smem, static_cast<cudaStream_t>(stream_)>>>(tm, (int)(rows / 128), iters, stages,
                                                                          cycles);
  return cudaGetLastError() == cudaSuccess ? BD_OK : BD_ERR_CUDA;
}
