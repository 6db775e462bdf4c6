// bd_lmhead_logprob / bd_lmhead_logprob_bwd: the LM head fused with the
// per-token log-softmax gather (the numerators
// pi_theta(o_k | .) of Eqs. 6-8, are the softmax of the logits
// z = h W^T).  The forward never materialises z [N, V]; the backward
// materialises only a bounded row chunk of dz (bf16).
//
// One GEMM engine, four epilogues:
//   * gemm2sm_kernel: CTA pair (cluster of 2, tcgen05.mma.cta_group::2,
//     UMMA 256 x 256 x 16 bf16 -> fp32).  CTA r of the pair owns rows
//     [256 mp + 128 r, +128) of D and loads half of every B tile (rows
//     [256 t + 128 r, +128)); both halves feed one MMA issued by the leader.
//     Operands arrive by TMA (128B swizzle) into a 6-stage ring (32 KB per
//     CTA per stage); the two accumulator buffers (2 x 256 TMEM columns) let
//     the epilogue of tile t overlap the MMAs of tile t+1.  A pair walks a
//     contiguous chunk of N tiles, so row-wise state (the online softmax)
//     lives in the epilogue's registers across the whole chunk.
//   * warp 0: TMA producer (both CTAs; completion counted on the leader's
//     barrier), warp 1: MMA issuer (leader only; commits multicast to both
//     CTAs), warps 2-5: epilogue (thread = TMEM lane = one row of D).
//   * Epilogues: LSE (online max / sum 2^x per row over the chunk + target
//     logit gather -> per-chunk partials), DZ (dz = w (1[v = t] - e^{z - LSE})
//     -> bf16), BF16 (store), F32 (store or accumulate).
//   * Operands may be K-major ([rows][K]) or MN-major ([K][rows]); the
//     backward's dh = dz W and dW = dz^T h read W, dz and h in place as
//     MN-major operands (no transposes).
//   * Grid raster: clusters are grouped so that ~74 co-resident pairs cover
//     `group` row pairs x all N chunks: the live A panels and B tiles fit in
//     L2 (each W tile is read from HBM once per group, not once per pair).
#include "abi_common.h"
#include "sm100.cuh"
#include "tma_host.h"

#include <cuda_bf16.h>
#include <algorithm>

namespace bd {
namespace {

constexpr int kBK = 64;
constexpr int kStages = 6;
constexpr int kStageA = 128 * kBK * 2;  // 16 KB: this CTA's 128 rows of A
constexpr int kStageB = 128 * kBK * 2;  // 16 KB: this CTA's half of the 256-row B tile
constexpr int kStageBytes = kStageA + kStageB;
constexpr int kThreadsG = 192;
constexpr uint32_t kTmemCols = 512;
constexpr int kSmemG = kStages * kStageBytes + 1024 + 256;
constexpr int kPairsPerWave = 74;  // 148 SMs / 2
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.69314718055994531f;

enum { EPI_LSE = 0, EPI_DZ = 1, EPI_BF16 = 2, EPI_F32 = 3 };

struct GemmParams {
  int M, N, K;
  int n_tiles, n_chunks, tiles_per_chunk;
  int m_pairs, group;
  const int32_t* targets;  // LSE, DZ: [M]
  float2* part;            // LSE: [n_chunks][M] (running max in log2 units, sum of 2^(x - max))
  float* zt;               // LSE: [M] target logit
  const float* lse;        // DZ: [M] natural-log LSE
  const float* w;          // DZ: [M] upstream gradient dL/dlogp
  void* out;               // DZ / BF16: bf16 [M][ldo]; F32: fp32 [M][ldo]
  long long ldo;
  int beta;                // F32: 1 = accumulate into out
};

// cluster / 2-SM PTX helpers: sm100.cuh

__device__ __forceinline__ void st_global_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ------------------------------------------------------------------- kernel
template <int EPI, bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsG, 1)
    gemm2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2] accumulator ready (both CTAs)
  uint64_t* tempty = tfull + 2;       // [2] accumulator drained (leader: 4 warps x 2 CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t rank = cluster_rank();
  const int warp = (int)warp_id(), lane = (int)lane_id();

  // grid raster: cluster id -> (row pair, N chunk)
  const int cid = blockIdx.x >> 1;
  const int gsz = p.group * p.n_chunks;
  const int grp = cid / gsz, rr = cid % gsz;
  const int g_m = min(p.group, p.m_pairs - grp * p.group);
  const int chunk = rr / g_m, mp = grp * p.group + rr % g_m;
  const int t0 = chunk * p.tiles_per_chunk, t1 = min(p.n_tiles, t0 + p.tiles_per_chunk);
  const int m0 = mp * 256 + (int)rank * 128;
  const int nk = (p.K + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      const uint32_t full_leader = mapa_shared(smem_u32(&full[0]), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t0; t < t1; ++t) {
        const int n0 = t * 256 + (int)rank * 128;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + kStageA;
          const uint32_t bar = full_leader + stage * 8;
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * kStageBytes);
          const int k0 = kb * kBK;
          if (!A_MN) {
            tma_load_2d_2sm(sa, &tmA, bar, k0, m0);
          } else {
            tma_load_2d_2sm(sa, &tmA, bar, m0, k0);
            tma_load_2d_2sm(sa + 8192, &tmA, bar, m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d_2sm(sb, &tmB, bar, k0, n0);
          } else {
            tma_load_2d_2sm(sb, &tmB, bar, n0, k0);
            tma_load_2d_2sm(sb + 8192, &tmB, bar, n0 + 64, k0);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, 256, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = t0; t < t1; ++t, ++it) {
        const int ab = it & 1;
        mbar_wait(&tempty[ab], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + ab * 256;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint32_t sb = sa + kStageA;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = A_MN ? umma_desc_sw128(sa + kk * 2048, 8192, 1024) : umma_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(sb + kk * 2048, 8192, 1024) : umma_desc_sw128(sb + kk * 32, 16, 1024);
            umma2_ss(d, ad, bd, idesc, (kb | kk) != 0);
          }
          umma2_commit_both(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma2_commit_both(&tfull[ab]);
      }
    }
  } else {
    // --------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_l = q * 32 + lane;
    const int row = m0 + row_l;
    const bool row_ok = row < p.M;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
    // per-row state
    int tgt = -1;
    float wr = 0.f, l2 = 0.f;
    if constexpr (EPI == EPI_LSE || EPI == EPI_DZ) tgt = row_ok ? p.targets[row] : -1;
    if constexpr (EPI == EPI_DZ) {
      wr = row_ok ? p.w[row] : 0.f;
      l2 = row_ok ? p.lse[row] * kLog2e : 0.f;
    }
    float m = -INFINITY, s = 0.f, ztv = 0.f;
    int it = 0;
    for (int t = t0; t < t1; ++t, ++it) {
      const int ab = it & 1;
      mbar_wait(&tfull[ab], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + ab * 256 + c * 32, r);
        tmem_ld_wait();
        const int col0 = t * 256 + c * 32;
        if constexpr (EPI == EPI_LSE) {
          float y[32];
          float cm = -INFINITY;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            y[j] = (col0 + j < p.N) ? __uint_as_float(r[j]) * kLog2e : -INFINITY;
            cm = fmaxf(cm, y[j]);
          }
          if (cm > m) {
            s *= ex2_approx(m - cm);
            m = cm;
          }
          if (m != -INFINITY) {
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              acc.x += ex2_approx(y[j] - m);
              acc.y += ex2_approx(y[j + 1] - m);
            }
            s += acc.x + acc.y;
          }
          const int tt = tgt - col0;
          if ((unsigned)tt < 32u) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j == tt) ztv = __uint_as_float(r[j]);
          }
        } else if constexpr (EPI == EPI_DZ) {
          if (row_ok && col0 < p.N) {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              float d0 = -wr * ex2_approx(fmaf(__uint_as_float(r[j]), kLog2e, -l2));
              float d1 = -wr * ex2_approx(fmaf(__uint_as_float(r[j + 1]), kLog2e, -l2));
              if (col0 + j == tgt) d0 += wr;
              if (col0 + j + 1 == tgt) d1 += wr;
              pk[j / 2] = pack_bf16x2(d0, d1);
            }
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + (size_t)row * p.ldo + col0;
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (col0 + 8 * g < p.N) st_global_v4(dst + 8 * g, pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
          }
        } else if constexpr (EPI == EPI_BF16) {
          if (row_ok && col0 < p.N) {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = pack_bf16x2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + (size_t)row * p.ldo + col0;
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (col0 + 8 * g < p.N) st_global_v4(dst + 8 * g, pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
          }
        } else {  // EPI_F32
          if (row_ok && col0 < p.N) {
            float* dst = reinterpret_cast<float*>(p.out) + (size_t)row * p.ldo + col0;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              if (col0 + 4 * g < p.N) {
                float4 v = make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                                       __uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3]));
                if (p.beta) {
                  const float4 o = *reinterpret_cast<const float4*>(dst + 4 * g);
                  v.x += o.x;
                  v.y += o.y;
                  v.z += o.z;
                  v.w += o.w;
                }
                *reinterpret_cast<float4*>(dst + 4 * g) = v;
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + ab * 8);
    }
    if constexpr (EPI == EPI_LSE) {
      if (row_ok) {
        p.part[(size_t)chunk * p.M + row] = make_float2(m, s);
        if (tgt >= t0 * 256 && tgt < t1 * 256 && tgt < p.N) p.zt[row] = ztv;
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2<kTmemCols>(tmem);
  }
}

// Combine the per-chunk (max, sum) partials of each row: LSE, logp.
__global__ void lse_combine_kernel(int M, int V, int n_chunks, const float2* __restrict__ part,
                                   const float* __restrict__ zt, const int32_t* __restrict__ targets,
                                   float* __restrict__ logp, float* __restrict__ lse) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= M) return;
  float mm = -INFINITY;
  for (int c = 0; c < n_chunks; ++c) mm = fmaxf(mm, part[(size_t)c * M + row].x);
  float ss = 0.f;
  for (int c = 0; c < n_chunks; ++c) {
    const float2 v = part[(size_t)c * M + row];
    if (v.x != -INFINITY) ss += v.y * exp2f(v.x - mm);
  }
  const float l = (mm + log2f(ss)) * kLn2;
  if (lse) lse[row] = l;
  const int t = targets[row];
  logp[row] = (t >= 0 && t < V) ? zt[row] - l : __int_as_float(0x7fc00000);
}

// ------------------------------------------------------------------- host
struct Plan {
  int n_tiles, n_chunks, tpc, m_pairs, group;
};

Plan plan_for(int M, int N, int max_chunks) {
  Plan pl;
  pl.n_tiles = (N + 255) / 256;
  pl.m_pairs = (M + 255) / 256;
  int want = std::max(1, (4 * kPairsPerWave + pl.m_pairs - 1) / pl.m_pairs);
  want = std::min(std::max(want, std::min(max_chunks, pl.n_tiles)), pl.n_tiles);
  pl.tpc = (pl.n_tiles + want - 1) / want;
  pl.n_chunks = (pl.n_tiles + pl.tpc - 1) / pl.tpc;
  pl.group = std::max(1, kPairsPerWave / pl.n_chunks);
  return pl;
}

// 2-D bf16 tensor map, dims {inner, outer}, outer stride in elements.
bool tmap2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld, bool mn_major) {
  const uint64_t dims[2] = {inner, outer};
  const uint64_t strides[1] = {ld * 2};
  const uint32_t box[2] = {64u, mn_major ? 64u : 128u};
  return make_tmap_bf16(m, base, 2, dims, strides, box);
}

template <int EPI, bool A_MN, bool B_MN>
int launch_gemm(const CUtensorMap& tA, const CUtensorMap& tB, GemmParams p, const Plan& pl, cudaStream_t stream) {
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(gemm2sm_kernel<EPI, A_MN, B_MN>), kSmemG,
                                "cudaFuncSetAttribute(gemm2sm)"))
    return rc;
  p.n_tiles = pl.n_tiles;
  p.n_chunks = pl.n_chunks;
  p.tiles_per_chunk = pl.tpc;
  p.m_pairs = pl.m_pairs;
  p.group = pl.group;
  const long long grid = 2LL * pl.m_pairs * pl.n_chunks;
  if (grid > 0x7FFFFFFF) return set_error(BD_ERR_UNSUPPORTED, "grid too large");
  gemm2sm_kernel<EPI, A_MN, B_MN><<<(unsigned)grid, kThreadsG, kSmemG, stream>>>(tA, tB, p);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "gemm2sm_kernel launch");
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int kFwdMaxChunks = 8;

size_t fwd_ws_bytes(int64_t n, int32_t V) {
  const Plan pl = plan_for((int)n, V, kFwdMaxChunks);
  return align256((size_t)pl.n_chunks * n * sizeof(float2)) + align256((size_t)n * sizeof(float));
}

int check_dims(int64_t n, int32_t C, int32_t V) {
  if (n <= 0 || C <= 0 || V <= 0) return set_error(BD_ERR_INVALID_ARG, "non-positive dimension");
  if (n > (1LL << 30)) return set_error(BD_ERR_UNSUPPORTED, "n_rows %lld too large", (long long)n);
  if (C % 8 || V % 8)
    return set_error(BD_ERR_UNSUPPORTED, "hidden (%d) and vocab (%d) must be multiples of 8 (16-byte rows)", C, V);
  return BD_OK;
}

int check_ptrs(std::initializer_list<const void*> ps) {
  for (const void* x : ps) {
    if (!x) return set_error(BD_ERR_INVALID_ARG, "null tensor pointer");
    if (!aligned16(x)) return set_error(BD_ERR_ALIGNMENT, "tensor pointer not 16-byte aligned");
  }
  return BD_OK;
}

}  // namespace
}  // namespace bd

extern "C" size_t bd_lmhead_workspace_bytes(int64_t n_rows, int32_t hidden, int32_t vocab, int backward,
                                            int64_t chunk_rows) {
  using namespace bd;
  if (check_dims(n_rows, hidden, vocab)) return 0;
  if (!backward) return fwd_ws_bytes(n_rows, vocab);
  if (chunk_rows <= 0) chunk_rows = n_rows;
  chunk_rows = std::min<int64_t>(chunk_rows, n_rows);
  return align256((size_t)chunk_rows * vocab * 2);
}

extern "C" int bd_lmhead_logprob(int64_t n_rows, int32_t hidden, int32_t vocab, const void* h, const void* w,
                                 const int32_t* targets, float* logp, float* lse, void* ws, size_t ws_bytes,
                                 void* stream_) {
  using namespace bd;
  int rc = check_dims(n_rows, hidden, vocab);
  if (rc) return rc;
  if ((rc = check_ptrs({h, w, targets, logp, ws}))) return rc;
  const size_t need = fwd_ws_bytes(n_rows, vocab);
  if (ws_bytes < need) return set_error(BD_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const Plan pl = plan_for((int)n_rows, vocab, kFwdMaxChunks);
  CUtensorMap tA, tB;
  if (!tmap2d(&tA, h, hidden, n_rows, hidden, false) || !tmap2d(&tB, w, hidden, vocab, hidden, false))
    return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  GemmParams p{};
  p.M = (int)n_rows;
  p.N = vocab;
  p.K = hidden;
  p.targets = targets;
  p.part = reinterpret_cast<float2*>(ws);
  p.zt = reinterpret_cast<float*>(static_cast<char*>(ws) + align256((size_t)pl.n_chunks * n_rows * sizeof(float2)));
  if ((rc = launch_gemm<EPI_LSE, false, false>(tA, tB, p, pl, stream))) return rc;
  lse_combine_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, stream>>>((int)n_rows, vocab, pl.n_chunks, p.part,
                                                                           p.zt, targets, logp, lse);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "lse_combine_kernel launch");
}

extern "C" int bd_lmhead_logprob_bwd(int64_t n_rows, int32_t hidden, int32_t vocab, const void* h, const void* w,
                                     const int32_t* targets, const float* lse, const float* dlogp, void* dh,
                                     float* dw, int64_t chunk_rows, void* ws, size_t ws_bytes, void* stream_) {
  using namespace bd;
  int rc = check_dims(n_rows, hidden, vocab);
  if (rc) return rc;
  if ((rc = check_ptrs({h, w, targets, lse, dlogp, dh, dw, ws}))) return rc;
  if (chunk_rows <= 0) chunk_rows = n_rows;
  chunk_rows = std::min<int64_t>(chunk_rows, n_rows);
  const size_t need = bd_lmhead_workspace_bytes(n_rows, hidden, vocab, 1, chunk_rows);
  if (ws_bytes < need) return set_error(BD_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const __nv_bfloat16* hb = static_cast<const __nv_bfloat16*>(h);
  __nv_bfloat16* dz = static_cast<__nv_bfloat16*>(ws);
  for (int64_t r0 = 0; r0 < n_rows; r0 += chunk_rows) {
    const int nc = (int)std::min<int64_t>(chunk_rows, n_rows - r0);
    const __nv_bfloat16* hc = hb + (size_t)r0 * hidden;
    // 1. dz = w (1[v = t] - softmax(h W^T)) for rows [r0, r0 + nc)   (recomputed logits)
    {
      CUtensorMap tA, tB;
      if (!tmap2d(&tA, hc, hidden, nc, hidden, false) || !tmap2d(&tB, w, hidden, vocab, hidden, false))
        return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
      GemmParams p{};
      p.M = nc;
      p.N = vocab;
      p.K = hidden;
      p.targets = targets + r0;
      p.lse = lse + r0;
      p.w = dlogp + r0;
      p.out = dz;
      p.ldo = vocab;
      if ((rc = launch_gemm<EPI_DZ, false, false>(tA, tB, p, plan_for(nc, vocab, kFwdMaxChunks), stream))) return rc;
    }
    // 2. dh[r0:] = dz W       (A = dz K-major over V; B = W read MN-major: N = hidden)
    {
      CUtensorMap tA, tB;
      if (!tmap2d(&tA, dz, vocab, nc, vocab, false) || !tmap2d(&tB, w, hidden, vocab, hidden, true))
        return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
      GemmParams p{};
      p.M = nc;
      p.N = hidden;
      p.K = vocab;
      p.out = static_cast<__nv_bfloat16*>(dh) + (size_t)r0 * hidden;
      p.ldo = hidden;
      if ((rc = launch_gemm<EPI_BF16, false, true>(tA, tB, p, plan_for(nc, hidden, 1 << 20), stream))) return rc;
    }
    // 3. dW (+)= dz^T h[r0:]  (A = dz read MN-major: M = V; B = h MN-major: N = hidden; K = rows)
    {
      CUtensorMap tA, tB;
      if (!tmap2d(&tA, dz, vocab, nc, vocab, true) || !tmap2d(&tB, hc, hidden, nc, hidden, true))
        return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
      GemmParams p{};
      p.M = vocab;
      p.N = hidden;
      p.K = nc;
      p.out = dw;
      p.ldo = hidden;
      p.beta = r0 > 0;
      if ((rc = launch_gemm<EPI_F32, true, true>(tA, tB, p, plan_for(vocab, hidden, 1 << 20), stream))) return rc;
    }
  }
  return BD_OK;
}

// Self-test of the GEMM engine: out[M][N] fp32 = sum_k A[m,k] B[n,k] with A
// K-major ([M][K]) or MN-major ([K][M]), likewise B.
extern "C" int bd_selftest_gemm(int32_t M, int32_t N, int32_t K, const void* a, int a_mn, const void* b, int b_mn,
                                float* out, void* stream_) {
  using namespace bd;
  if (M <= 0 || N <= 0 || K <= 0 || M % 8 || N % 8 || K % 8) return set_error(BD_ERR_INVALID_ARG, "bad dims");
  int rc = check_ptrs({a, b, out});
  if (rc) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  CUtensorMap tA, tB;
  const bool okA = a_mn ? tmap2d(&tA, a, M, K, M, true) : tmap2d(&tA, a, K, M, K, false);
  const bool okB = b_mn ? tmap2d(&tB, b, N, K, N, true) : tmap2d(&tB, b, K, N, K, false);
  if (!okA || !okB) return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.out = out;
  p.ldo = N;
  const Plan pl = plan_for(M, N, 4);
  if (!a_mn && !b_mn) return launch_gemm<EPI_F32, false, false>(tA, tB, p, pl, stream);
  if (!a_mn && b_mn) return launch_gemm<EPI_F32, false, true>(tA, tB, p, pl, stream);
  if (a_mn && b_mn) return launch_gemm<EPI_F32, true, true>(tA, tB, p, pl, stream);
  return launch_gemm<EPI_F32, true, false>(tA, tB, p, pl, stream);
}
