// bd_decode_attn / bd_decode_select: blockwise KV-cache decoding for the
// rollout.
//
// Attention (Eq. 2, p(b^k_0 | b^k_t, b^{<k}); KV cache P:83; SPEC
// inference mask S:201-205): the active block's B query rows of every head
// attend to the first kv_len[b] keys of their sequence's cache -- the clean
// blocks < k followed by the active block's own keys -- with no mask inside.
// It is HBM-bound (each cached K/V byte is read once per call) with a tiny
// contraction per byte, so the kernel is organised around streaming the cache:
//  * CTA = (key split, kv head [x head part], sequence).  Its query rows are
//    the hs heads x B positions sharing that kv head (GQA), NQ <= 32 rows.
//  * 128-key K/V tiles stream through a 3-stage TMA ring (64 KB per stage).
//  * The contraction is transposed so the tensor core sees a full 128-row
//    operand: S^T [128 keys x NQ] = K Q^T (tcgen05, M = 128, N = NQ) and
//    O^T [128 d x NQ] += V^T P^T (V read MN-major straight from the TMA tile,
//    P^T written by the softmax warps into a swizzled smem operand).
//  * Softmax warps: thread = key (S^T lane); column max by warp shuffles and
//    a 4-warp smem exchange; running max with lazy rescaling of O^T (thread
//    = d lane in TMEM); thread-partial row sums reduced once at the end.
//  * Keys >= kv_len in the tail tile get p = 0 and their V rows are zeroed
//    in smem (the cache past kv_len may hold anything, even NaN).
//  * Each CTA writes an unnormalised partial (O, m, l); a combine kernel
//    merges the splits into O (bf16) and LSE.
// Token selection (P:312 dynamic decoding, reading c20): per row
// argmax (lowest index on ties) and confidence 1 / sum exp(z - max) in fp32;
// per sequence commit every masked position above the threshold, else the
// most confident one.
#include "abi_common.h"
#include "sm100.cuh"
#include "tma_host.h"
#include "attn_common.h"

#include <cuda_bf16.h>
#include <algorithm>
#include <initializer_list>

namespace bd {
namespace {

constexpr int kD = 128;
constexpr int kTile = 128;
constexpr int kTileBytes = kTile * kD * 2;  // 32 KB
constexpr int kDStages = 3;
constexpr int kDThreads = 192;  // warps 0-3 softmax, 4 TMA, 5 MMA
constexpr float kLog2eD = 1.4426950408889634f;
constexpr float kLn2D = 0.69314718055994531f;
constexpr float kRescaleThr = 8.f;

template <int NQ>
struct DecCfg {
  static constexpr int kQBytes = NQ * kD * 2;     // two 64-column halves of NQ rows
  static constexpr int kPBytes = NQ * kTile * 2;  // two 64-key halves of NQ rows
  // smem: Q | P[2] | K,V stages | red[4][NQ] | bars
  static constexpr int kOffP = kQBytes;
  static constexpr int kOffKV = ((kOffP + 2 * kPBytes + 1023) / 1024) * 1024;
  static constexpr int kOffRed = kOffKV + kDStages * 2 * kTileBytes;
  static constexpr int kOffBar = kOffRed + 4 * NQ * 4;
  static constexpr int kNumBars = 3 * kDStages + 2 + 2 + 2;  // k_full, v_full, empty; s_full[2], p_full[2], o_done[2]
  static constexpr int kSmem = kOffBar + kNumBars * 8 + 16 + 1024;
};

struct DecArgs {
  const __nv_bfloat16* q;  // [b, B, Hq, d]
  const int32_t* kv_len;   // [b]
  float* part_o;           // [splits][b][Hq][B][d]
  float2* part_ml;         // [splits][b][Hq][B]
  int batch, B, Hq, Hkv, G, hs, n_parts, n_splits, cap;
  float scale_log2;
};

template <int NQ>
__global__ void __launch_bounds__(kDThreads, 1)
    decode_attn_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const DecArgs a) {
  using C = DecCfg<NQ>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sP = smem + C::kOffP;
  uint8_t* sKV = smem + C::kOffKV;  // stage s: K at 2s, V at 2s+1
  float* red = reinterpret_cast<float*>(smem + C::kOffRed);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* k_full = bars;
  uint64_t* v_full = k_full + kDStages;
  uint64_t* empty = v_full + kDStages;
  uint64_t* s_full = empty + kDStages;  // [2]
  uint64_t* p_full = s_full + 2;        // [2]
  uint64_t* o_done = p_full + 2;        // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  const int split = blockIdx.x;
  const int kvh = blockIdx.y / a.n_parts, part = blockIdx.y % a.n_parts;
  const int b = blockIdx.z;
  const int h0 = kvh * a.G + part * a.hs;  // first query head of this CTA
  const int rows = a.hs * a.B;             // valid query rows (<= NQ)
  const int kv_len = a.kv_len[b];
  const int n_t = (kv_len + kTile - 1) / kTile;
  const int j0 = (int)((long long)split * n_t / a.n_splits);
  const int j1 = (int)((long long)(split + 1) * n_t / a.n_splits);
  const int nj = j1 - j0;

  // Q -> swizzled K-major smem operand [NQ rows x 128 d]; row r = hl * B + i
  for (int idx = threadIdx.x; idx < NQ * 16; idx += kDThreads) {
    const int r = idx >> 4, c = idx & 15;  // 16-byte chunk c of row r
    uint4 val = make_uint4(0, 0, 0, 0);
    if (r < rows) {
      const int hl = r / a.B, i = r - hl * a.B;
      val = *reinterpret_cast<const uint4*>(a.q + (((size_t)b * a.B + i) * a.Hq + h0 + hl) * kD + c * 8);
    }
    *reinterpret_cast<uint4*>(sQ + (c >> 3) * (NQ * 128) + sw128_offset(r, c & 7)) = val;
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  if (threadIdx.x == 32 * 4) {
    for (int s = 0; s < kDStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_done[i], 1);
    }
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // TMEM: S^T buffers at columns [0, NQ) and [NQ, 2 NQ); O^T at [128, 128 + NQ)
  const uint32_t tO = tbase + 128;

  if (warp == 4) {
    // ---------------------------------------------------------------- TMA
    if (lane == 0 && nj > 0) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      for (int jj = 0; jj < nj; ++jj) {
        const int s = jj % kDStages;
        const uint32_t ph = (jj / kDStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const int k0 = (j0 + jj) * kTile;
        uint8_t* dk = sKV + (2 * s) * kTileBytes;
        uint8_t* dv = dk + kTileBytes;
        mbar_expect_tx(&k_full[s], kTileBytes);
        for (int kb = 0; kb < 2; ++kb) tma_load_4d(dk + kb * 16384, &tmK, &k_full[s], kb * 64, kvh, k0, b);
        mbar_expect_tx(&v_full[s], kTileBytes);
        for (int kb = 0; kb < 2; ++kb) tma_load_4d(dv + kb * 16384, &tmV, &v_full[s], kb * 64, kvh, k0, b);
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA
    if (lane == 0 && nj > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, NQ, false, false);  // S^T = K Q^T
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, NQ, true, false);   // O^T = V^T P^T
      const uint32_t qaddr = smem_u32(sQ);
      auto issue_s = [&](int jj) {
        const int s = jj % kDStages;
        mbar_wait(&k_full[s], (jj / kDStages) & 1);
        tc_fence_after();
        const uint32_t kaddr = smem_u32(sKV + (2 * s) * kTileBytes);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint32_t ka = kaddr + (k >> 2) * 16384 + (k & 3) * 32;
          const uint32_t qa = qaddr + (k >> 2) * (NQ * 128) + (k & 3) * 32;
          umma_ss(tbase + (jj & 1) * NQ, umma_desc_sw128(ka, 16, 1024), umma_desc_sw128(qa, 16, 1024), idesc_s,
                  k > 0);
        }
        umma_commit(&s_full[jj & 1]);
      };
      issue_s(0);
      if (nj > 1) issue_s(1);
      for (int jj = 0; jj < nj; ++jj) {
        const int s = jj % kDStages;
        mbar_wait(&p_full[jj & 1], (jj >> 1) & 1);
        mbar_wait(&v_full[s], (jj / kDStages) & 1);
        tc_fence_after();
        const uint32_t vaddr = smem_u32(sKV + (2 * s + 1) * kTileBytes);
        const uint32_t paddr = smem_u32(sP + (jj & 1) * C::kPBytes);
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k) {
          const uint32_t va = vaddr + k * 2048;  // 16 keys of the MN-major V^T operand
          const uint32_t pa = paddr + (k >> 2) * (NQ * 128) + (k & 3) * 32;
          umma_ss(tO, umma_desc_sw128(va, 16384, 1024), umma_desc_sw128(pa, 16, 1024), idesc_o,
                  (jj > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&o_done[jj & 1]);
        umma_commit(&empty[s]);
        if (jj + 2 < nj) issue_s(jj + 2);  // S^T buffer jj&1 was read before p_full(jj)
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int key_l = warp * 32 + lane;  // TMEM lane: key (S^T) / d (O^T)
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    float m[NQ], l[NQ];
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      m[c] = -INFINITY;
      l[c] = 0.f;
    }
    for (int jj = 0; jj < nj; ++jj) {
      const int key = (j0 + jj) * kTile + key_l;
      const bool valid = key < kv_len;
      const bool tail = (j0 + jj + 1) * kTile > kv_len;
      mbar_wait(&s_full[jj & 1], (jj >> 1) & 1);
      tc_fence_after();
      uint32_t sr[NQ];
      if constexpr (NQ == 16) {
        tmem_ld16(tbase + lane_off + (jj & 1) * NQ, sr);
      } else {
        tmem_ld32(tbase + lane_off + (jj & 1) * NQ, sr);
      }
      tmem_ld_wait();
      float x[NQ];
#pragma unroll
      for (int c = 0; c < NQ; ++c) x[c] = valid ? __uint_as_float(sr[c]) * a.scale_log2 : -INFINITY;
      // column max over the 128 keys: warp butterfly, then 4-warp exchange
      float cm[NQ];
#pragma unroll
      for (int c = 0; c < NQ; ++c) {
        float v = x[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        cm[c] = v;
      }
      if (lane < NQ) {
        float mine = cm[0];
#pragma unroll
        for (int c = 1; c < NQ; ++c)
          if (lane == c) mine = cm[c];
        red[warp * NQ + lane] = mine;
      }
      named_bar_sync(1, 128);
      bool resc = false;
      float alpha[NQ];
#pragma unroll
      for (int c = 0; c < NQ; ++c) {
        const float t = fmaxf(fmaxf(red[c], red[NQ + c]), fmaxf(red[2 * NQ + c], red[3 * NQ + c]));
        // lazy: keep the running max unless the tile exceeds it by > 2^8
        if (t > m[c] + kRescaleThr || m[c] == -INFINITY) {
          alpha[c] = ex2_approx(m[c] - t);  // m = -inf -> 0
          m[c] = t;
          resc = true;
        } else {
          alpha[c] = 1.f;
        }
      }
      named_bar_sync(1, 128);  // red[] may be overwritten next tile
      // P^T (bf16) into the free P buffer: O(jj-2) consumed it
      if (jj >= 2) mbar_wait(&o_done[jj & 1], ((jj - 2) >> 1) & 1);
      uint8_t* pb = sP + (jj & 1) * C::kPBytes + (key_l >> 6) * (NQ * 128);
      const uint32_t kc = (key_l & 63) >> 3, kb2 = (key_l & 7) * 2;
#pragma unroll
      for (int c = 0; c < NQ; ++c) {
        const float p = ex2_approx(x[c] - m[c]);
        l[c] = fmaf(l[c], alpha[c], p);
        *reinterpret_cast<__nv_bfloat16*>(pb + sw128_offset(c, kc) + kb2) = __float2bfloat16_rn(p);
      }
      if (tail) {
        // zero V rows of keys >= kv_len (0 * garbage must not reach O)
        const int s = jj % kDStages;
        mbar_wait(&v_full[s], (jj / kDStages) & 1);
        if (!valid) {
          uint8_t* vr = sKV + (2 * s + 1) * kTileBytes + key_l * 128;
#pragma unroll
          for (int kb = 0; kb < 2; ++kb)
#pragma unroll
            for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(vr + kb * 16384 + c * 16) = make_uint4(0, 0, 0, 0);
        }
      }
      // O^T columns *= alpha (O(jj-1) must have landed)
      if (jj > 0 && __any_sync(0xffffffffu, resc)) {
        mbar_wait(&o_done[(jj - 1) & 1], ((jj - 1) >> 1) & 1);
        tc_fence_after();
        uint32_t ov[NQ];
        if constexpr (NQ == 16) {
          tmem_ld16(tO + lane_off, ov);
        } else {
          tmem_ld32(tO + lane_off, ov);
        }
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < NQ; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * alpha[c]);
        if constexpr (NQ == 16) {
          tmem_st16(tO + lane_off, ov);
        } else {
          tmem_st32(tO + lane_off, ov);
        }
        tmem_st_wait();
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[jj & 1]);
    }
    // ---- partial epilogue: l column sums, O^T (unnormalised), m
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      float v = l[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      l[c] = v;
    }
    if (lane < NQ) {
      float mine = l[0];
#pragma unroll
      for (int c = 1; c < NQ; ++c)
        if (lane == c) mine = l[c];
      red[warp * NQ + lane] = mine;
    }
    named_bar_sync(1, 128);
    const size_t seq_head = ((size_t)split * a.batch + b) * a.Hq;
    if (nj > 0) {
      mbar_wait(&o_done[(nj - 1) & 1], ((nj - 1) >> 1) & 1);
      tc_fence_after();
    }
    uint32_t ov[NQ];
    if (nj > 0) {
      if constexpr (NQ == 16) {
        tmem_ld16(tO + lane_off, ov);
      } else {
        tmem_ld32(tO + lane_off, ov);
      }
      tmem_ld_wait();
    }
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      if (c < rows) {
        const int hl = c / a.B, i = c - hl * a.B;
        const size_t rix = (seq_head + h0 + hl) * a.B + i;
        a.part_o[rix * kD + key_l] = nj > 0 ? __uint_as_float(ov[c]) : 0.f;
        if (key_l == 0) {
          const float lsum = red[c] + red[NQ + c] + red[2 * NQ + c] + red[3 * NQ + c];
          a.part_ml[rix] = make_float2(nj > 0 ? m[c] : -INFINITY, nj > 0 ? lsum : 0.f);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

// Merge the key splits: one CTA per (sequence, head), thread = d.
__global__ void decode_combine_kernel(const float* __restrict__ part_o, const float2* __restrict__ part_ml,
                                      int n_splits, int batch, int Hq, int B, __nv_bfloat16* __restrict__ o,
                                      float* __restrict__ lse) {
  const int b = blockIdx.x / Hq, h = blockIdx.x % Hq;
  const int d = threadIdx.x;
  for (int i = 0; i < B; ++i) {
    float M = -INFINITY;
    for (int s = 0; s < n_splits; ++s) M = fmaxf(M, part_ml[(((size_t)s * batch + b) * Hq + h) * B + i].x);
    float L = 0.f, acc = 0.f;
    for (int s = 0; s < n_splits; ++s) {
      const size_t rix = (((size_t)s * batch + b) * Hq + h) * B + i;
      const float2 ml = part_ml[rix];
      if (ml.x == -INFINITY) continue;
      const float w = exp2f(ml.x - M);
      L += ml.y * w;
      acc += part_o[rix * kD + d] * w;
    }
    o[(((size_t)b * B + i) * Hq + h) * kD + d] = __float2bfloat16_rn(acc / L);
    if (d == 0) lse[((size_t)b * Hq + h) * B + i] = (M + log2f(L)) * kLn2D;
  }
}

// ---- token selection: per row (argmax, confidence), then per-sequence rule
constexpr int kSelThreads = 256;

__global__ void __launch_bounds__(kSelThreads) select_row_kernel(int V, const __nv_bfloat16* __restrict__ z,
                                                                 int32_t* __restrict__ token,
                                                                 float* __restrict__ conf) {
  const size_t row = blockIdx.x;
  const __nv_bfloat16* zr = z + row * V;
  float mx = -INFINITY;
  int arg = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += kSelThreads) {
    const float x = __bfloat162float(zr[v]);
    if (x > mx) {  // increasing v: first maximal index per thread
      mx = x;
      arg = v;
    }
  }
  __shared__ float smx[kSelThreads / 32];
  __shared__ int sarg[kSelThreads / 32];
  __shared__ float sfin;
  __shared__ float ssum[kSelThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, arg, o);
    if (m2 > mx || (m2 == mx && a2 < arg)) {
      mx = m2;
      arg = a2;
    }
  }
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (ln == 0) {
    smx[w] = mx;
    sarg[w] = arg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float bm = smx[0];
    int ba = sarg[0];
    for (int i = 1; i < kSelThreads / 32; ++i)
      if (smx[i] > bm || (smx[i] == bm && sarg[i] < ba)) {
        bm = smx[i];
        ba = sarg[i];
      }
    sfin = bm;
    token[row] = ba;
  }
  __syncthreads();
  const float m2 = sfin * kLog2eD;
  float s = 0.f;
  for (int v = threadIdx.x; v < V; v += kSelThreads) s += exp2f(fmaf(__bfloat162float(zr[v]), kLog2eD, -m2));
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (ln == 0) ssum[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < kSelThreads / 32; ++i) t += ssum[i];
    conf[row] = 1.f / t;
  }
}

__global__ void select_commit_kernel(int batch, int B, const uint8_t* __restrict__ masked,
                                     const float* __restrict__ conf, float threshold, uint8_t* __restrict__ commit) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  int any = 0, best = -1;
  float bc = -1.f;
  for (int i = 0; i < B; ++i) {
    const size_t r = (size_t)b * B + i;
    const bool mk = masked[r] != 0;
    const bool hit = mk && conf[r] > threshold;
    commit[r] = hit ? 1 : 0;
    any |= hit;
    if (mk && conf[r] > bc) {
      bc = conf[r];
      best = i;
    }
  }
  if (!any && best >= 0) commit[(size_t)b * B + best] = 1;
}

template <int NQ>
int launch_decode(const CUtensorMap& tK, const CUtensorMap& tV, const DecArgs& a, cudaStream_t stream) {
  using C = DecCfg<NQ>;
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(decode_attn_kernel<NQ>), C::kSmem,
                                "cudaFuncSetAttribute(decode)"))
    return rc;
  dim3 grid(a.n_splits, a.Hkv * a.n_parts, a.batch);
  decode_attn_kernel<NQ><<<grid, kDThreads, C::kSmem, stream>>>(tK, tV, a);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "decode_attn_kernel launch");
}

struct DecPlan {
  int hs, n_parts, nq, n_splits;
};

bool plan_decode(int batch, int B, int Hq, int Hkv, int cap, DecPlan& pl) {
  if (B > 32) return false;
  const int G = Hq / Hkv;
  pl.hs = 1;
  for (int h = G; h >= 1; --h)
    if (G % h == 0 && h * B <= 32) {
      pl.hs = h;
      break;
    }
  pl.n_parts = G / pl.hs;
  pl.nq = pl.hs * B <= 16 ? 16 : 32;
  const int units = batch * Hkv * pl.n_parts;
  const int tiles = (cap + kTile - 1) / kTile;
// Key splits only until ~4 CTAs per SM exist: each CTA's prologue (TMEM
// alloc, barriers, Q load, ring fill) costs more than the tail imbalance
// that finer splits would remove (SDAR-8B rollout, 128 x 8 kv heads: 4 per
// SM -> no split, 0.478 ms; 8 -> 0.494; 16 -> 0.527; 32 -> 0.620).
#ifndef BD_DEC_CTAS_PER_SM
#define BD_DEC_CTAS_PER_SM 4
#endif
  pl.n_splits = std::max(1, std::min(tiles, (BD_DEC_CTAS_PER_SM * 148 + units - 1) / units));
  return true;
}

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace bd

extern "C" size_t bd_decode_workspace_bytes(int32_t batch, int32_t block, int32_t n_q_heads, int32_t n_kv_heads,
                                            int32_t head_dim, int32_t cap) {
  using namespace bd;
  if (batch <= 0 || block <= 0 || n_kv_heads <= 0 || n_q_heads % n_kv_heads || head_dim != 128 || cap < block)
    return 0;
  DecPlan pl;
  if (!plan_decode(batch, block, n_q_heads, n_kv_heads, cap, pl)) return 0;
  const size_t rows = (size_t)pl.n_splits * batch * n_q_heads * block;
  return al256(rows * kD * sizeof(float)) + al256(rows * sizeof(float2));
}

extern "C" int bd_decode_attn(int32_t batch, int32_t block, int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                              int32_t cap, float softmax_scale, const void* q, const void* k_cache,
                              const void* v_cache, const int32_t* kv_len, void* o, float* lse, void* ws,
                              size_t ws_bytes, void* stream_) {
  using namespace bd;
  if (batch <= 0 || block <= 0 || n_q_heads <= 0 || n_kv_heads <= 0 || cap <= 0)
    return set_error(BD_ERR_INVALID_ARG, "non-positive dimension");
  if (n_q_heads % n_kv_heads) return set_error(BD_ERR_INVALID_ARG, "Hq %% Hkv != 0");
  if (head_dim != 128) return set_error(BD_ERR_UNSUPPORTED, "decode head_dim %d != 128", head_dim);
  if (block > 32) return set_error(BD_ERR_UNSUPPORTED, "decode block size %d > 32", block);
  if (cap < block) return set_error(BD_ERR_INVALID_ARG, "cache capacity < block size");
  for (const void* x : std::initializer_list<const void*>{q, k_cache, v_cache, kv_len, o, lse, ws}) {
    if (!x) return set_error(BD_ERR_INVALID_ARG, "null pointer");
    if (!aligned16(x)) return set_error(BD_ERR_ALIGNMENT, "pointer not 16-byte aligned");
  }
  const size_t need = bd_decode_workspace_bytes(batch, block, n_q_heads, n_kv_heads, head_dim, cap);
  if (ws_bytes < need) return set_error(BD_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  DecPlan pl;
  plan_decode(batch, block, n_q_heads, n_kv_heads, cap, pl);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  CUtensorMap tK, tV;
  if (!make_qkv_tmap(&tK, k_cache, batch, cap, n_kv_heads, kD) || !make_qkv_tmap(&tV, v_cache, batch, cap, n_kv_heads, kD))
    return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  DecArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.kv_len = kv_len;
  const size_t rows = (size_t)pl.n_splits * batch * n_q_heads * block;
  a.part_o = static_cast<float*>(ws);
  a.part_ml = reinterpret_cast<float2*>(static_cast<char*>(ws) + al256(rows * kD * sizeof(float)));
  a.batch = batch;
  a.B = block;
  a.Hq = n_q_heads;
  a.Hkv = n_kv_heads;
  a.G = n_q_heads / n_kv_heads;
  a.hs = pl.hs;
  a.n_parts = pl.n_parts;
  a.n_splits = pl.n_splits;
  a.cap = cap;
  a.scale_log2 = (softmax_scale > 0.f ? softmax_scale : 1.f / sqrtf((float)head_dim)) * kLog2eD;
  int rc = pl.nq == 16 ? launch_decode<16>(tK, tV, a, stream) : launch_decode<32>(tK, tV, a, stream);
  if (rc) return rc;
  decode_combine_kernel<<<batch * n_q_heads, kD, 0, stream>>>(a.part_o, a.part_ml, pl.n_splits, batch, n_q_heads,
                                                              block, static_cast<__nv_bfloat16*>(o), lse);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "decode_combine_kernel launch");
}

extern "C" int bd_decode_select(int32_t batch, int32_t block, int32_t vocab, const void* logits,
                                const uint8_t* masked, float threshold, int32_t* token, float* conf, uint8_t* commit,
                                void* stream_) {
  using namespace bd;
  if (batch <= 0 || block <= 0 || vocab <= 0) return set_error(BD_ERR_INVALID_ARG, "non-positive dimension");
  if (!logits || !masked || !token || !conf || !commit) return set_error(BD_ERR_INVALID_ARG, "null pointer");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  select_row_kernel<<<(unsigned)((size_t)batch * block), kSelThreads, 0, stream>>>(
      vocab, static_cast<const __nv_bfloat16*>(logits), token, conf);
  select_commit_kernel<<<(batch + 127) / 128, 128, 0, stream>>>(batch, block, masked, conf, threshold, commit);
  note_launches(2);
  return check_cuda(cudaGetLastError(), "select kernels launch");
}
