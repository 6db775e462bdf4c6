// bd_attn_fwd: block-diffusion masked attention forward, sm_100a.
//
// Computes, for every packed query row i of every (sequence, q-head),
//   O_i = sum_j softmax_j(scale q_i.k_j | M_ij) v_j,  LSE_i = ln sum_j exp(scale q_i.k_j | M_ij)
// with M the DiRL block-diffusion mask (Eq. 2).
//
// Design:
//  * One CTA per (q-tile, sequence, pair of q-heads of one kv group): the two
//    query tiles share every K/V tile (GQA packing), so each K/V tile loaded by
//    TMA feeds two S = QK^T and two O += PV tcgen05 MMAs.  When Hq/Hkv is odd
//    a CTA carries one q-head (NQ = 1) and two CTAs share an SM.
//  * Only the k-tiles listed by the tile map for this q-tile are visited
//    (EMPTY tiles are never loaded); the list is LPT-ordered across CTAs.
//  * Warp roles: warps [0, 4 NQ) are softmax warpgroups (one per q-tile, a
//    thread owns one row = one TMEM lane), warp 4 NQ issues TMA, warp 4 NQ + 1
//    issues tcgen05.mma.  S and O accumulate in TMEM (S_q at column 128 q,
//    O_q after the S regions); P (bf16) overwrites S_q in place and feeds the
//    PV MMA straight from TMEM.
//  * Online softmax in the exp2 domain with lazy rescaling: the running max is
//    only raised when a tile's max exceeds it by > 8 (factor 256), so the O
//    correction (TMEM ld/mul/st) is rare.
//  * Mask: on PARTIAL or ragged tiles each row keeps the columns inside its
//    visible interval (tilemap.cuh row_interval); FULL tiles are unmasked.
#include "sm100.cuh"
#include "tma_host.h"
#include "tilemap.cuh"
#include "problem.h"
#include "attn_common.h"

#include <cuda_bf16.h>
#include <cstdlib>

namespace bd {
namespace {

template <int D, int NQ>
struct FwdCfg {
  static constexpr int kTileBytes = 128 * D * 2;
#ifndef BD_FWD_STAGES
#define BD_FWD_STAGES 4
#endif
  static constexpr int kStages = NQ == 2 ? BD_FWD_STAGES : 2;
  static constexpr int kSoftmaxWarps = 4 * NQ;
  static constexpr int kTmaWarp = kSoftmaxWarps;
  static constexpr int kMmaWarp = kSoftmaxWarps + 1;
  static constexpr int kThreads = (kSoftmaxWarps + 2) * 32;
  static constexpr int kSCol = 0;                 // S_q at 128 q
  static constexpr int kOCol = 128 * NQ;          // O_q at kOCol + D q
  static constexpr int kTmemUsed = 128 * NQ + D * NQ;
  static constexpr uint32_t kTmemCols = kTmemUsed <= 256 ? 256 : 512;
  // barriers: q_full, kv_full[S], kv_empty[S], s_full[NQ], p_full[NQ], pv_done[NQ], p_half[NQ]
  static constexpr int kNumBars = 1 + 2 * kStages + 4 * NQ;
  static constexpr int kSmemBytes = NQ * kTileBytes + kStages * kTileBytes + kNumBars * 8 + 16 + 1024;
};

// Opt-in event trace (BD_TRACE=1): CTA 0 records clock64 stamps, read back by
// bd_debug_trace_fwd().
__device__ long long g_trace_fwd[8192];
#define FTRACE(slot, cond)                                        \
  do {                                                            \
    if (a.trace && (cond)) g_trace_fwd[(slot)] = clock64();       \
  } while (0)

struct FwdArgs {
  const int* map;
  int map_stride;  // varlen: words between per-sequence maps
  __nv_bfloat16* o;
  float* lse;
  int batch, n_q_heads, n_hg, group, N, n_kv;
  int q_row_heads;  // heads per token row of o in memory
  Geom g;
  float scale_log2;
  int trace;
};

// One online-softmax step of a 128-column S tile held in TMEM at tS (this
// thread's row): optional interval mask [lo, hi), running max m (log2 units,
// lazily raised by > 8), running sum l, P = 2^(s sl2 - m) written over tS as
// bf16.  Returns the new max, whether O must be rescaled, and by how much.
// Share of the forward's exps moved from the MUFU to the packed FMA-pipe
// polynomial: element pair c uses it iff c % BD_FWD_POLY_MOD == MOD - 1
// (0 = MUFU only).  At d = 128 the MUFU (16 ex2/clk/SM) needs as many clocks
// per tile as the tensor core, so it co-bounds the forward.
#ifndef BD_FWD_POLY_MOD
#define BD_FWD_POLY_MOD 4
#endif

template <bool MASKED, int D>
__device__ __forceinline__ void softmax_tile(uint32_t tS, uint32_t tO, int lo, int hi, float sl2, float m, float& l,
                                             float& m_new, int j, uint64_t* p_half, int lane) {
  uint32_t sr[128];
#pragma unroll
  for (int c = 0; c < 4; ++c) tmem_ld32(tS + 32 * c, sr + 32 * c);
  tmem_ld_wait();
  float* s = reinterpret_cast<float*>(sr);
  if (MASKED) {
#pragma unroll
    for (int c = 0; c < 128; ++c) s[c] = (c >= lo && c < hi) ? s[c] : -INFINITY;
  }
  // row max: 8 independent chains (a single FMNMX3 chain is ~64 dependent
  // instructions with one softmax warp per scheduler to hide them)
  float mx8[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) mx8[i] = s[i];
#pragma unroll
  for (int c = 8; c < 128; c += 8)
#pragma unroll
    for (int i = 0; i < 8; ++i) mx8[i] = fmaxf(mx8[i], s[c + i]);
  const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
  const float tmax = mx * sl2;
  m_new = m;
  bool resc = false;
  if (tmax > m + 8.f) {
    m_new = tmax;
    resc = true;
  }
  const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
  const float alpha = resc ? ex2_approx(m - m_use) : 1.f;
  if (j > 0 && __any_sync(0xffffffffu, resc)) {
    // O_q *= alpha before PV_q(j) accumulates into it (PV_q(j-1) has
    // completed: S_q(j), issued after it, has completed)
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t ov[32];
      tmem_ld32(tO + 32 * c, ov);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
      tmem_st32(tO + 32 * c, ov);
    }
  }
  const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m_use, -m_use);
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  uint32_t pk[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) {
    const float2 x = ffma2(make_float2(s[2 * c], s[2 * c + 1]), sl2v, nm);
    float2 p;
    if (BD_FWD_POLY_MOD > 0 && (c % BD_FWD_POLY_MOD) == BD_FWD_POLY_MOD - 1) {
      p = ex2_poly2(x);  // exactly +0 for a masked (-inf) score, like the MUFU's ex2
    } else {
      p.x = ex2_approx(x.x);  // ex2.approx(-inf) = +0
      p.y = ex2_approx(x.y);
    }
    acc[c & 3] = fadd2(acc[c & 3], p);
    pk[c] = pack_bf16x2(p.x, p.y);
    if (c == 47) {
      // first 96 keys of P out: PV_q(j) k-steps 0-5 may start (p_half)
      tmem_st32(tS, pk);
      tmem_st16(tS + 32, pk + 32);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_half);
    }
  }
  const float2 a01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
  const float sum = a01.x + a01.y;
  l = l * alpha + sum;
  tmem_st16(tS + 48, pk + 48);
}

template <int D, int NQ, bool VARLEN>
__global__ void __launch_bounds__(FwdCfg<D, NQ>::kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const FwdArgs a) {
  using C = FwdCfg<D, NQ>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + NQ * C::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::kStages * C::kTileBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;
  uint64_t* p_full = s_full + NQ;
  uint64_t* pv_done = p_full + NQ;
  uint64_t* p_half = pv_done + NQ;  // first 96 keys of P_q written
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  const Geom& gm = a.g;  // the batch's (maximum) geometry: grid decomposition

  // ---- work unit: LPT rank of the q-tile, then (sequence, head pair)
  // Grid order: (sequence, kv head) outermost, then the q-tile's LPT rank,
  // then the head pairs of the group -- concurrently resident CTAs belong to
  // the same (sequence, kv head) and stream the same K/V tiles (L2 reuse).
  const int hp_per_kv = a.group / NQ;
  const int per_unit = gm.NT * hp_per_kv;
  const int unit = blockIdx.x / per_unit;
  const int rem = blockIdx.x - unit * per_unit;
  const int rank = rem / hp_per_kv;
  const int mi = unit / a.n_kv;  // map slot (varlen: longest sequences first)
  const int kvh = unit - mi * a.n_kv;
  const int h0 = kvh * a.group + (rem - rank * hp_per_kv) * NQ;
  // varlen: this sequence's own map and geometry; ranks past its tile count exit
  const int* mapb = VARLEN ? a.map + (size_t)mi * a.map_stride : a.map;
  const int b = VARLEN ? map_seq(mapb) : mi;
  const Geom gsq = VARLEN ? map_geom(mapb) : gm;
  const Geom& g = VARLEN ? gsq : gm;
  if (VARLEN && rank >= g.NT) return;
  const MapView mv{const_cast<int*>(mapb), g.NT, map_capacity(g)};
  const int qt = mv.fwd_order()[rank];
  const int e0 = mv.row_ptr()[qt];
  const int n_kt = mv.row_ptr()[qt + 1] - e0;
  const int* ents = mv.row_ent() + e0;
  int q0, q1, qseg;
  tile_bounds(g, qt, q0, q1, qseg);

  if (warp == 0) tmem_alloc<C::kTmemCols>(tslot);
  if (warp == C::kTmaWarp && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int q = 0; q < NQ; ++q) {
      mbar_init(&s_full[q], 1);
      mbar_init(&p_full[q], 4);
      mbar_init(&pv_done[q], 1);
      mbar_init(&p_half[q], 4);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    // Q goes out before the CTA-wide barrier and the TMEM allocation (only
    // this thread uses q_full before the barrier)
    mbar_expect_tx(q_full, NQ * C::kTileBytes);
    for (int q = 0; q < NQ; ++q)
      for (int kb = 0; kb < D / 64; ++kb)
        tma_load_4d(sQ + q * C::kTileBytes + kb * 16384, &tmQ, q_full, kb * 64, h0 + q, q0, b);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == C::kTmaWarp) {
    // ================================================================ TMA
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int j = 0; j < n_kt; ++j) {
        const int k0 = tile_start(g, entry_tile(ents[j]));
#pragma unroll
        for (int kv = 0; kv < 2; ++kv) {
          mbar_wait(&kv_empty[stage], phase ^ 1);
          mbar_expect_tx(&kv_full[stage], C::kTileBytes);
          uint8_t* dst = sKV + stage * C::kTileBytes;
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_4d(dst + kb * 16384, kv ? &tmV : &tmK, &kv_full[stage], kb * 64, kvh, k0, b);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == C::kMmaWarp) {
    // ================================================================ MMA
    if (elect_one()) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
      // Ring index of K(j) is 2j, of V(j) 2j+1.  Issue order per tile j and head q:
      // PV_q(j) as soon as P_q(j) is ready, then (after PV_q(j) has consumed P_q,
      // which aliases S_q) S_q(j+1).  Heads are handled independently so the two
      // softmax warpgroups fall into a ping-pong: one runs its exps while the
      // other's PV / S MMAs execute.
      auto slot = [](int idx) { return idx % C::kStages; };
      auto ph = [](int idx) { return (uint32_t)((idx / C::kStages) & 1); };
      auto kv_addr = [&](int idx) { return smem_u32(sKV + slot(idx) * C::kTileBytes); };
      auto issue_s = [&](int q, int j) {
        const uint32_t qaddr = smem_u32(sQ + q * C::kTileBytes), kaddr = kv_addr(2 * j);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          umma_ss(tbase + C::kSCol + 128 * q, umma_desc_sw128(qaddr + off, 16, 1024),
                  umma_desc_sw128(kaddr + off, 16, 1024), idesc_s, k > 0);
        }
        umma_commit(&s_full[q]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&kv_full[slot(0)], ph(0));
      tc_fence_after();
#pragma unroll
      for (int q = 0; q < NQ; ++q) issue_s(q, 0);
      umma_commit(&kv_empty[slot(0)]);
      for (int j = 0; j < n_kt; ++j) {
        mbar_wait(&kv_full[slot(2 * j + 1)], ph(2 * j + 1));
        FTRACE(1024 + 8 * (j & 127) + 0, blockIdx.x == 0);
        const uint32_t vaddr = kv_addr(2 * j + 1);
        const bool has_next = j + 1 < n_kt;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          // PV_q(j) in two parts: keys 0-95 once P_q's first 96 columns are
          // written (p_half), keys 96-127 at p_full -- overlaps the softmax tail
          mbar_wait(&p_half[q], j & 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 6; ++k)
            umma_ts(tbase + C::kOCol + D * q, tbase + C::kSCol + 128 * q + k * 8,
                    umma_desc_sw128(vaddr + k * 2048, 16384, 1024), idesc_o, (j > 0 || k > 0) ? 1u : 0u);
          mbar_wait(&p_full[q], j & 1);
          FTRACE(1024 + 8 * (j & 127) + 1 + q, blockIdx.x == 0);
          tc_fence_after();
#pragma unroll
          for (int k = 6; k < 8; ++k)
            umma_ts(tbase + C::kOCol + D * q, tbase + C::kSCol + 128 * q + k * 8,
                    umma_desc_sw128(vaddr + k * 2048, 16384, 1024), idesc_o, 1u);
          // pv_done is observed only by the epilogue: commit the last tile only
          // (no mbarrier phase completes unobserved; compute-sanitizer synccheck)
          if (!has_next) umma_commit(&pv_done[q]);
          if (q == NQ - 1) umma_commit(&kv_empty[slot(2 * j + 1)]);  // V(j) consumed
          if (has_next) {
            if (q == 0) mbar_wait(&kv_full[slot(2 * j + 2)], ph(2 * j + 2));
            // No wait for PV_q(j): tcgen05.mma ops of one thread execute in
            // issue order, so S_q(j+1) overwrites the S/P columns only after
            // PV_q(j) has read P_q(j) (WAR through the in-order tensor pipe).
            FTRACE(1024 + 8 * (j & 127) + 3 + q, blockIdx.x == 0);
            issue_s(q, j + 1);
            if (q == NQ - 1) umma_commit(&kv_empty[slot(2 * j + 2)]);  // K(j+1) consumed
          }
        }
      }
    }
  } else {
    // ============================================================ softmax
    const int q = warp >> 2;
    const int r = (warp & 3) * 32 + lane;  // row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tbase + lane_off + C::kSCol + 128 * q;
    const uint32_t tO = tbase + lane_off + C::kOCol + D * q;
    const int row = q0 + r;
    int lo0, hi0, lo1, hi1;
    row_interval(g, qseg, row, 0, lo0, hi0);
    row_interval(g, qseg, row, qseg ? qseg : 1, lo1, hi1);  // the row's own noisy copy
    const float sl2 = a.scale_log2;
    float m = -INFINITY, l = 0.f;

    int ent_next = n_kt > 0 ? ents[0] : 0;  // row entries loaded one tile ahead
    for (int j = 0; j < n_kt; ++j) {
      const int ent = ent_next;
      if (j + 1 < n_kt) ent_next = ents[j + 1];
      const int kt = entry_tile(ent);
      const int k0 = tile_start(g, kt), k1 = tile_end(g, kt);
      const bool need_mask = entry_kind(ent) == kKindPartial || (k1 - k0) < 128;
      FTRACE(8 * (j & 127) + 0 + 4 * q, blockIdx.x == 0 && (threadIdx.x & 127) == 0);
      mbar_wait(&s_full[q], j & 1);
      FTRACE(8 * (j & 127) + 1 + 4 * q, blockIdx.x == 0 && (threadIdx.x & 127) == 0);
      tc_fence_after();
      const bool xt = tile_seg(g, kt) != 0;
      const int lo = (xt ? lo1 : lo0) - k0;
      const int hi = min(xt ? hi1 : hi0, k1) - k0;
      float m_new;
      // two separate code paths: the masked one must not be if-converted into
      // every tile (FULL tiles need no per-element work)
      if (need_mask)
        softmax_tile<true, D>(tS, tO, lo, hi, sl2, m, l, m_new, j, &p_half[q], lane);
      else
        softmax_tile<false, D>(tS, tO, lo, hi, sl2, m, l, m_new, j, &p_half[q], lane);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[q]);
      FTRACE(8 * (j & 127) + 2 + 4 * q, blockIdx.x == 0 && (threadIdx.x & 127) == 0);
      m = m_new;
    }
    // ---- epilogue
    mbar_wait(&pv_done[q], 0);
    tc_fence_after();
    const int h = h0 + q;
    const bool valid = row < q1;
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = a.o + (((size_t)b * a.N + row) * a.q_row_heads + h) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t ov[32];
      tmem_ld32(tO + 32 * c, ov);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = pack_bf16x2(__uint_as_float(ov[2 * i]) * inv_l, __uint_as_float(ov[2 * i + 1]) * inv_l);
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(orow + 32 * c);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (valid) {
      const float m_use = (m == -INFINITY) ? 0.f : m;
      a.lse[((size_t)b * a.n_q_heads + h) * a.N + row] =
          l > 0.f ? (m_use + __log2f(l)) * 0.69314718055994531f : -INFINITY;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D, int NQ, bool VARLEN>
int launch_fwd(const bd_problem& p, const Geom& g, const void* q, const void* k, const void* v, void* o,
               float* lse, const int* map, int map_stride, cudaStream_t stream) {
  using C = FwdCfg<D, NQ>;
  CUtensorMap tmQ, tmK, tmV;
  if (!make_qkv_tmap(&tmQ, q, p.batch, g.N, p.n_q_heads, D, 128, q_row_heads(p)) ||
      !make_qkv_tmap(&tmK, k, p.batch, g.N, p.n_kv_heads, D, 128, kv_row_heads(p)) ||
      !make_qkv_tmap(&tmV, v, p.batch, g.N, p.n_kv_heads, D, 128, kv_row_heads(p)))
    return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(attn_fwd_kernel<D, NQ, VARLEN>), C::kSmemBytes,
                                "cudaFuncSetAttribute(fwd)"))
    return rc;
  FwdArgs a;
  a.map = map;
  a.map_stride = map_stride;
  a.o = reinterpret_cast<__nv_bfloat16*>(o);
  a.lse = lse;
  a.batch = p.batch;
  a.n_q_heads = p.n_q_heads;
  a.q_row_heads = q_row_heads(p);
  a.n_hg = p.n_q_heads / NQ;
  a.group = p.n_q_heads / p.n_kv_heads;
  a.n_kv = p.n_kv_heads;
  a.N = g.N;
  a.g = g;
  a.scale_log2 = scale_of(p) * 1.4426950408889634f;
  static const bool trace_on = getenv("BD_TRACE") != nullptr;
  a.trace = trace_on ? 1 : 0;
  const long long grid = (long long)g.NT * p.batch * a.n_hg;
  if (grid > 0x7FFFFFFF) return set_error(BD_ERR_UNSUPPORTED, "grid too large");
  attn_fwd_kernel<D, NQ, VARLEN><<<(unsigned)grid, C::kThreads, C::kSmemBytes, stream>>>(tmQ, tmK, tmV, a);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "attn_fwd_kernel launch");
}

}  // namespace

int run_attn_fwd(const bd_problem& p, const Geom& g, const void* q, const void* k, const void* v, void* o,
                 float* lse, const int* map, int map_stride, cudaStream_t stream) {
  const bool pair = (p.n_q_heads / p.n_kv_heads) % 2 == 0;
  const bool vl = map_stride != 0;
#define BD_FWD_CASE(D_, NQ_)                                                                         \
  return vl ? launch_fwd<D_, NQ_, true>(p, g, q, k, v, o, lse, map, map_stride, stream)             \
            : launch_fwd<D_, NQ_, false>(p, g, q, k, v, o, lse, map, map_stride, stream)
  if (p.head_dim == 128) {
    if (pair) BD_FWD_CASE(128, 2);
    BD_FWD_CASE(128, 1);
  }
  if (p.head_dim == 64) {
    if (pair) BD_FWD_CASE(64, 2);
    BD_FWD_CASE(64, 1);
  }
#undef BD_FWD_CASE
  return set_error(BD_ERR_UNSUPPORTED, "head_dim %d not in {64, 128}", p.head_dim);
}

}  // namespace bd

extern "C" int bd_debug_trace_fwd(int64_t* host_out, int n) {
  if (!host_out || n <= 0 || n > 8192) return BD_ERR_INVALID_ARG;
  return bd::check_cuda(cudaMemcpyFromSymbol(host_out, bd::g_trace_fwd, n * sizeof(long long)), "trace copy");
}
