// bd_attn_bwd: backward of the block-diffusion attention, sm_100a.
//
// Analytic gradient of O = softmax(scale QK^T | M) V:
//   P = exp(scale S - LSE) (masked), dV = P^T dO, dP = dO V^T,
//   dS = P o (dP - D) with D_i = rowsum(dO_i o O_i),
//   dQ = scale dS K, dK = scale dS^T Q (dK, dV summed over the q-heads of a group).
//
// Launches (after the tile map), no atomics:
//  1. zero + bwd_pre: D and the log2-domain LSE in a tile-major workspace
//               layout (a q-tile's 128 values form one aligned 512 B bulk copy).
//  2. dkdv:     one CTA per (k-tile, sequence, kv head), visiting only the
//               q-tiles of the tile map's column list (EMPTY tiles never
//               loaded), for every q-head of the group.  K, V stay in smem;
//               Q, dO stream through a 5-slot TMA ring, LSE / D through a
//               2-slot bulk-copy ring.  TMEM: S^T, dP^T, dV, dK (512 columns).
//               P^T and dS^T (bf16) go back over the dP^T columns just read,
//               in two halves, and feed dV += P^T dO and dK += dS^T Q as TS
//               MMAs.  Issue order: S^T(i+1) once phase 1 has read S^T(i);
//               the even k-steps of dV(i), dK(i) at the first half, the odd
//               ones at the second; dP^T(i+1) right behind them.
//  3. dq:       persistent, one CTA per SM walking (q-tile, sequence, q-head)
//               units over the tile map's row lists: S = QK^T (double-
//               buffered in TMEM), dP = dO V^T, dS (bf16) over S feeds
//               dQ += dS K from TMEM; K through 4 slots, V through 1.  The
//               pipelines run across units (next Q / dO load once the last S
//               and dP of a unit are issued).
// dQ is therefore accumulated in TMEM and written once (deterministic), at
// the price of recomputing S and dP per (q-tile, k-tile) pair -- cheaper on
// B200 than 64 KB of fp32 L2 reductions per tile pair (profiles/r01).
// Compute warps: four warpgroups split the 128 columns of a tile; a thread
// owns one TMEM lane (a key row in dkdv, a query row in dq).
#include "sm100.cuh"
#include "tma_host.h"
#include "tilemap.cuh"
#include "problem.h"
#include "attn_common.h"

#include <cuda_bf16.h>
#include <cstdlib>

namespace bd {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

// ------------------------------------------------------------ preprocess
// -D_i = -rowsum(dO_i o O_i) and -log2-domain LSE, written tile-major.  One
// 16-byte load per thread per tensor; D/8 threads per row; grid
// (ceil(N / rows_per_block), b * Hq).
template <int D, bool VARLEN>
__global__ void __launch_bounds__(256) bwd_pre_kernel(const __nv_bfloat16* __restrict__ o,
                                                      const __nv_bfloat16* __restrict__ dout,
                                                      const float* __restrict__ lse, float* __restrict__ lse2_t,
                                                      float* __restrict__ dsum_t, int N, int Hq, int q_rh, Geom gm,
                                                      const int* __restrict__ map, int map_stride) {
  constexpr int kTpr = D / 8;             // threads per row
  constexpr int kRows = 256 / kTpr;       // rows per block
  // varlen: blockIdx.y / Hq indexes the per-sequence maps, which name their
  // sequence; rows past that sequence's packed length are padding
  const int mi = blockIdx.y / Hq, h = blockIdx.y - mi * Hq;
  const int* mapb = map + (size_t)mi * map_stride;
  const int b = VARLEN ? map_seq(mapb) : mi;
  const int bh = b * Hq + h;
  const int n = blockIdx.x * kRows + threadIdx.x / kTpr;
  const int sub = threadIdx.x % kTpr;
  const Geom g = VARLEN ? map_geom(mapb) : gm;
  const bool valid = n < (VARLEN ? g.N : N);
  float acc = 0.f;
  if (valid) {
    const size_t base = (((size_t)b * N + n) * q_rh + h) * D + sub * 8;  // q_rh: heads per row in memory
    const uint4 a = *reinterpret_cast<const uint4*>(o + base);
    const uint4 c = *reinterpret_cast<const uint4*>(dout + base);
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc = fmaf(__uint_as_float(av[i] << 16), __uint_as_float(cv[i] << 16), acc);
      acc = fmaf(__uint_as_float(av[i] & 0xFFFF0000u), __uint_as_float(cv[i] & 0xFFFF0000u), acc);
    }
  }
#pragma unroll
  for (int off = kTpr / 2; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (valid && sub == 0) {
    const int t = tile_of_row(g, n);
    const int r = n - tile_start(g, t);
    const size_t slot = ((size_t)bh * gm.NT + t) * kTileRows + r;  // stride: the batch's max tile count
    // stored negated: the compute loops add them with packed FFMA2 / FADD2
    dsum_t[slot] = -acc;
    lse2_t[slot] = -lse[(size_t)bh * N + n] * kLog2e;
  }
}

__global__ void zero_kernel(float4* __restrict__ p, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Opt-in event trace (BD_TRACE=1 in the environment): one CTA records clock64
// stamps of its pipeline hand-offs into a static device buffer, read back by
// bd_debug_trace().  Off by default (a warp-uniform predicate per event).
__device__ long long g_trace[8192];
// BD_TRACE=2: per-unit timeline of the dQ kernel (globaltimer ns when the
// compute warps start the unit and after its epilogue, tile count, SM id) for
// the first 32768 units, read by bd_debug_cta_timeline()
__device__ long long g_cta_tl[4 * 32768];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int smid() {
  int r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#define TRACE(slot, cond)                                         \
  do {                                                            \
    if (a.trace == 1 && (cond)) g_trace[(slot)] = clock64();      \
  } while (0)

struct BwdArgs {
  const int* map;
  int map_stride;  // varlen: words between per-sequence maps
  const float* lse2_t;
  const float* dsum_t;
  __nv_bfloat16* dq;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  int batch, n_q_heads, n_kv_heads, group, N;
  int q_row_heads, kv_row_heads;  // heads per token row of dq / dk, dv in memory
  Geom g;
  float scale, scale_log2;
  int trace;  // 1 = record the trace for blockIdx.x == 0
  // stored-dS path: the dK/dV kernel writes every tile's dS^T (bf16,
  // [128 keys][128 q]) at tile slot (b Hq + h) ds_stride + (its row-CSR entry
  // index), the dQ kernel reads each q-tile's row of tiles contiguously
  __nv_bfloat16* ds;  // null: dQ recomputes S and dP (attn_bwd_dqp_kernel)
  long long ds_stride;
};

__device__ __forceinline__ void store_row_bf16(__nv_bfloat16* dst, const uint32_t* v, float mul, bool ok) {
  uint32_t pk[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) pk[j] = pack_bf16x2(__uint_as_float(v[2 * j]) * mul, __uint_as_float(v[2 * j + 1]) * mul);
  if (ok) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int u = 0; u < 4; ++u) d4[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
  }
}

template <int N>
__device__ __forceinline__ void store_row_bf16_n(__nv_bfloat16* dst, const uint32_t* v, float mul, bool ok) {
  uint32_t pk[N / 2];
#pragma unroll
  for (int j = 0; j < N / 2; ++j) pk[j] = pack_bf16x2(__uint_as_float(v[2 * j]) * mul, __uint_as_float(v[2 * j + 1]) * mul);
  if (ok) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int u = 0; u < N / 8; ++u) d4[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
  }
}

// P = 2^(s sl2 - lse2) for NC columns, zeroed outside [ja, jb) when MASKED
// (dK/dV kernel: per-column lse2 from smem).  Masked and unmasked tiles take
// separate code paths so FULL tiles pay no per-element mask work.
// Share of the exps on the packed FMA-pipe polynomial (pair j/2 uses it iff
// (j/2) % MOD == MOD - 1; 0 = MUFU only), per kernel.
#ifndef BD_DKDV_POLY_MOD
#define BD_DKDV_POLY_MOD 0
#endif
#ifndef BD_DKDV_TAIL_GROUPS
#define BD_DKDV_TAIL_GROUPS 4
#endif
#ifndef BD_DQ_POLY_MOD
#define BD_DQ_POLY_MOD 4
#endif

template <int MOD>
__device__ __forceinline__ float2 ex2_pair(int pair, float2 x) {
  if (MOD > 0 && (pair % MOD) == MOD - 1) return ex2_poly2(x);
  return make_float2(ex2_approx(x.x), ex2_approx(x.y));
}

template <bool MASKED, int NC>
__device__ __forceinline__ void p_tile(const uint32_t* sr, const float* sv, float sl2, int ja, int jb, float* pv) {
#pragma unroll
  for (int j = 0; j < NC; j += 2) {  // sv = -lse2 (negated by bwd_pre)
    const float2 x = ffma2(make_float2(__uint_as_float(sr[j]), __uint_as_float(sr[j + 1])), make_float2(sl2, sl2),
                           make_float2(sv[j], sv[j + 1]));
    const float2 p = ex2_pair<BD_DKDV_POLY_MOD>(j / 2, x);
    pv[j] = p.x;
    pv[j + 1] = p.y;
  }
  if (MASKED) {
#pragma unroll
    for (int j = 0; j < NC; ++j) pv[j] = (j >= ja && j < jb) ? pv[j] : 0.f;
  }
}
// Same with a per-row lse2 (dQ kernel), 32 columns.
template <bool MASKED>
__device__ __forceinline__ void p_row(const uint32_t* sr, float nlse2, float sl2, int ja, int jb, float* pv) {
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const float2 x = ffma2(make_float2(__uint_as_float(sr[j]), __uint_as_float(sr[j + 1])), make_float2(sl2, sl2),
                           make_float2(nlse2, nlse2));
    const float2 p = ex2_pair<BD_DQ_POLY_MOD>(j / 2, x);
    pv[j] = p.x;
    pv[j + 1] = p.y;
  }
  if (MASKED) {
#pragma unroll
    for (int j = 0; j < 32; ++j) pv[j] = (j >= ja && j < jb) ? pv[j] : 0.f;
  }
}

// ================================================================== dK/dV
// Smem: K, V resident; Q(i), dO(i) through a 4-slot single-tile ring (Q(i) ->
// ring index 2i, dO(i) -> 2i+1, each released by its last MMA); dS^T (bf16)
// in smem; LSE/D vectors through a 2-slot ring.  TMEM: S^T [0,128),
// dP^T [128,256), dV, dK.  Four compute warpgroups each own 32 q columns
// (a thread = one key row = one TMEM lane).  Per iteration i:
//   phase 1 (needs S^T(i)):  P = exp2(S sl2 - lse2)          -> p1_done
//   phase 2 (needs dP^T(i)): dS = P (dP - D); P^T (bf16) over the dP^T
//            columns just read, dS^T (bf16) beside it        -> pt_done
//   MMA: S^T(i+1) at p1_done(i); dV(i), dK(i) at pt_done(i) (both TS: A = P^T /
//        dS^T from TMEM);
//        dP^T(i+1) once dV(i) has consumed P^T(i).
// (dK(i) before dP^T(i+1) so that storing dS^T(i+1) never waits for dK(i).)
template <int D>
struct DkdvCfg {
  static constexpr int kTileBytes = 128 * D * 2;
  // dS^T lives in TMEM (next to P^T in the dP^T columns), so the 32 KB it
  // took in smem buys a fifth Q/dO ring slot: loads are issued an iteration
  // earlier and the dP^T(i+1) issue no longer waits for dO(i+1)
  static constexpr int kSlots = 5;
  static constexpr int kWGs = 4;
  static constexpr int kCols = 128 / kWGs;  // q columns per warpgroup
  static constexpr int kComputeWarps = 4 * kWGs;
  static constexpr int kTmaWarp = kComputeWarps;
  static constexpr int kMmaWarp = kComputeWarps + 1;
  static constexpr int kThreads = 32 * (kComputeWarps + 2);
  static constexpr int kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + D;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kTileBytes;
  static constexpr int kOffRing = 2 * kTileBytes;
  static constexpr int kOffVec = kOffRing + kSlots * kTileBytes;
  static constexpr int kVecBytes = 2 * 128 * 4;
  static constexpr int kOffBar = kOffVec + 2 * kVecBytes;
  // kv_full, slot_full[S], slot_empty[S], vec_full[2], vec_empty[2], s_full, dp_full, p1_done,
  // pt_done[4], acc_done, pt_half[4] (per warpgroup)
  static constexpr int kNumBars = 1 + 2 * kSlots + 4 + 3 + 2 * kWGs + 1;
  static constexpr int kSmemBytes = kOffBar + kNumBars * 8 + 16;
  static_assert(kSmemBytes <= 232448, "dkdv smem budget");
};

template <int D, bool VARLEN>
__global__ void __launch_bounds__(DkdvCfg<D>::kThreads, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                         const BwdArgs a) {
  using C = DkdvCfg<D>;
  const long long t_entry = (a.trace == 3 && threadIdx.x == 0) ? gtimer() : 0;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + C::kOffK;
  uint8_t* sV = smem + C::kOffV;
  uint8_t* sRing = smem + C::kOffRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* slot_full = bars + 1;
  uint64_t* slot_empty = slot_full + C::kSlots;
  uint64_t* vec_full = slot_empty + C::kSlots;  // [2]
  uint64_t* vec_empty = vec_full + 2;           // [2]
  uint64_t* s_full = vec_empty + 2;
  uint64_t* dp_full = s_full + 1;
  uint64_t* p1_done = dp_full + 1;  // S^T(i) read
  // per warpgroup w: its 32 q columns' P^T(i), dS^T(i) written -- first 16
  // (pt_half[w]) / all (pt_done[w]); the dV / dK k-steps 2w and 2w+1 read
  // exactly those columns, so each issues as soon as its own warpgroup is
  // done instead of waiting for the slowest of the 16 warps
  uint64_t* pt_done = p1_done + 1;  // [4]
  uint64_t* acc_done = pt_done + C::kWGs;
  uint64_t* pt_half = acc_done + 1;  // [4]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

  const int warp = (int)warp_id(), lane = (int)lane_id();
  const Geom& gm = a.g;  // the batch's (maximum) geometry: grid, vector strides
  if ((smem_u32(smem) & 1023u) != 0) __trap();

  // Grid order: (sequence, kv head) outermost, LPT rank of the k-tile inner --
  // concurrently resident CTAs stream the same Q / dO tiles (L2 reuse).  The
  // last BD_DKDV_TAIL_GROUPS groups are merged into one LPT order (their
  // ranks interleaved) so their longest columns start early enough not to
  // leave a tail (list-scheduling model and BD_TRACE=3 timeline: 1.5% tail).
  int unit, rank;
  {
    const int n_units = (int)(gridDim.x / gm.NT);
    const int kt = n_units < BD_DKDV_TAIL_GROUPS ? n_units : BD_DKDV_TAIL_GROUPS;
    const int split = (n_units - kt) * gm.NT;
    if ((int)blockIdx.x < split || kt <= 1) {
      unit = blockIdx.x / gm.NT;
      rank = blockIdx.x - unit * gm.NT;
    } else {
      const int t = blockIdx.x - split;
      rank = t / kt;
      unit = n_units - kt + (t - rank * kt);
    }
  }
  const int mi = unit / a.n_kv_heads;  // map slot (varlen: longest sequences first)
  const int kvh = unit - mi * a.n_kv_heads;
  const int* mapb = VARLEN ? a.map + (size_t)mi * a.map_stride : a.map;
  const int b = VARLEN ? map_seq(mapb) : mi;
  const Geom gsq = VARLEN ? map_geom(mapb) : gm;
  const Geom& g = VARLEN ? gsq : gm;
  if (VARLEN && rank >= g.NT) return;
  const MapView mv{const_cast<int*>(mapb), g.NT, map_capacity(g)};
  const int kt = mv.bwd_order()[rank];
  const int e0 = mv.col_ptr()[kt];
  const int n_qt = mv.col_ptr()[kt + 1] - e0;
  const int* ents = mv.col_ent() + e0;
  const int n_it = n_qt * a.group;
  int k0, k1, kseg;
  tile_bounds(g, kt, k0, k1, kseg);
  auto slot_of = [](int idx) { return idx % C::kSlots; };
  auto phase_of = [](int idx) { return (uint32_t)((idx / C::kSlots) & 1); };

  if (warp == 0) tmem_alloc<C::kTmemCols>(tslot);
  if (warp == C::kTmaWarp && lane == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < C::kSlots; ++s) {
      mbar_init(&slot_full[s], 1);
      mbar_init(&slot_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&vec_full[s], 1);
      mbar_init(&vec_empty[s], C::kComputeWarps);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p1_done, C::kComputeWarps);
    for (int w = 0; w < C::kWGs; ++w) mbar_init(&pt_done[w], 4);
    mbar_init(acc_done, 1);
    for (int w = 0; w < C::kWGs; ++w) mbar_init(&pt_half[w], 4);
    fence_barrier_init();
    // K, V loads go out before the CTA-wide barrier and the TMEM allocation
    // (only this thread uses kv_full before the barrier)
    if (n_it > 0) {
      mbar_expect_tx(kv_full, 2 * C::kTileBytes);
      for (int kb = 0; kb < D / 64; ++kb) {
        tma_load_4d(sK + kb * 16384, &tmK, kv_full, kb * 64, kvh, k0, b);
        tma_load_4d(sV + kb * 16384, &tmV, kv_full, kb * 64, kvh, k0, b);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == C::kTmaWarp) {
    // ================================================================ TMA
    if (elect_one() && n_it > 0) {
      // LSE / D vectors one iteration ahead of Q / dO: vec(i+1) is issued right
      // after dO(i) (its 2-slot ring frees a whole iteration earlier than the
      // Q / dO slots), so its ~1 us load latency is off the compute path
      // iteration i = (column entry n_qt - 1 - i / group, head i % group), walked
      // with counters (no integer division on the issue path)
      auto issue_vec = [&](int i, int qt, int hs) {
        const int h = kvh * a.group + hs;
        const int vs = i & 1;
        mbar_wait(&vec_empty[vs], ((i >> 1) & 1) ^ 1);
        mbar_expect_tx(&vec_full[vs], C::kVecBytes);
        const size_t vec = (((size_t)b * a.n_q_heads + h) * gm.NT + qt) * kTileRows;
        float* sv = reinterpret_cast<float*>(smem + C::kOffVec + vs * C::kVecBytes);
        bulk_load(sv, a.lse2_t + vec, 512, &vec_full[vs]);
        bulk_load(sv + 128, a.dsum_t + vec, 512, &vec_full[vs]);
      };
      int eidx = n_qt - 1, qt = entry_tile(ents[eidx]), hs = 0;  // iteration i
      issue_vec(0, qt, 0);
      for (int i = 0; i < n_it; ++i) {
        const int h = kvh * a.group + hs;  // decreasing q-tile: L2 reuse across CTAs
        const int q0 = tile_start(g, qt);
#pragma unroll
        for (int w = 0; w < 2; ++w) {  // w = 0: Q(i), w = 1: dO(i)
          const int idx = 2 * i + w, s = slot_of(idx);
          mbar_wait(&slot_empty[s], phase_of(idx) ^ 1);
          TRACE(2048 + 8 * (i & 127) + w, blockIdx.x == 0);
          mbar_expect_tx(&slot_full[s], C::kTileBytes);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_4d(sRing + s * C::kTileBytes + kb * 16384, w ? &tmDO : &tmQ, &slot_full[s], kb * 64, h, q0, b);
        }
        if (++hs == a.group) {
          hs = 0;
          if (i + 1 < n_it) qt = entry_tile(ents[--eidx]);
        }
        if (i + 1 < n_it) issue_vec(i + 1, qt, hs);
      }
    }
  } else if (warp == C::kMmaWarp) {
    // ================================================================ MMA
    if (elect_one() && n_it > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);  // S^T, dP^T
      constexpr uint32_t idesc_kv = umma_idesc_bf16(128, D, false, true);    // dV, dK: B MN-major
      const uint32_t kaddr = smem_u32(sK), vaddr = smem_u32(sV);
      auto ring = [&](int idx) { return smem_u32(sRing + slot_of(idx) * C::kTileBytes); };
      auto issue_s = [&](int i) {  // S^T = K Q^T
        const uint32_t qaddr = ring(2 * i);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          umma_ss(tbase + C::kColS, umma_desc_sw128(kaddr + off, 16, 1024), umma_desc_sw128(qaddr + off, 16, 1024),
                  idesc_s, k > 0);
        }
        umma_commit(s_full);
      };
      auto issue_dp = [&](int i) {  // dP^T = V dO^T
        const uint32_t doaddr = ring(2 * i + 1);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          umma_ss(tbase + C::kColDP, umma_desc_sw128(vaddr + off, 16, 1024),
                  umma_desc_sw128(doaddr + off, 16, 1024), idesc_s, k > 0);
        }
        umma_commit(dp_full);
      };
      mbar_wait(kv_full, 0);
      mbar_wait(&slot_full[slot_of(0)], phase_of(0));
      tc_fence_after();
      issue_s(0);
      mbar_wait(&slot_full[slot_of(1)], phase_of(1));
      tc_fence_after();
      issue_dp(0);
      for (int i = 0; i < n_it; ++i) {
        const bool has_next = i + 1 < n_it;
        const uint32_t qaddr = ring(2 * i), doaddr = ring(2 * i + 1);
        mbar_wait(p1_done, i & 1);
        TRACE(1024 + 8 * (i & 127) + 0, blockIdx.x == 0);
        if (has_next) {
          mbar_wait(&slot_full[slot_of(2 * i + 2)], phase_of(2 * i + 2));
          TRACE(1024 + 8 * (i & 127) + 6, blockIdx.x == 0);
          tc_fence_after();
          issue_s(i + 1);
        }
        // P^T / dS^T arrive in two halves (q columns 0-15 and 16-31 of every
        // warpgroup = the even and odd k-steps): the even k-steps of dV(i) and
        // dK(i) run while the compute warps finish the odd half
        // even k-steps (first 16 q columns of warpgroup w), then odd ones; the
        // dV k-step order (0, 2, 4, 6, 1, 3, 5, 7) is unchanged
#pragma unroll
        for (int w = 0; w < C::kWGs; ++w) {
          const int k = 2 * w;
          mbar_wait(&pt_half[w], i & 1);
          tc_fence_after();
          umma_ts(tbase + C::kColDV, tbase + C::kColDP + 32 * w, umma_desc_sw128(doaddr + k * 2048, 16384, 1024),
                  idesc_kv, (i > 0 || k > 0) ? 1u : 0u);
          umma_ts(tbase + C::kColDK, tbase + C::kColDP + 32 * w + 16, umma_desc_sw128(qaddr + k * 2048, 16384, 1024),
                  idesc_kv, (i > 0 || k > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int w = 0; w < C::kWGs; ++w) {
          const int k = 2 * w + 1;
          mbar_wait(&pt_done[w], i & 1);
          if (w == 0) TRACE(1024 + 8 * (i & 127) + 1, blockIdx.x == 0);
          tc_fence_after();
          umma_ts(tbase + C::kColDV, tbase + C::kColDP + 32 * w + 8, umma_desc_sw128(doaddr + k * 2048, 16384, 1024),
                  idesc_kv, 1u);
          umma_ts(tbase + C::kColDK, tbase + C::kColDP + 32 * w + 24, umma_desc_sw128(qaddr + k * 2048, 16384, 1024),
                  idesc_kv, 1u);
        }
        umma_commit(&slot_empty[slot_of(2 * i + 1)]);  // dO(i) consumed
        TRACE(1024 + 8 * (i & 127) + 5, blockIdx.x == 0);
        umma_commit(&slot_empty[slot_of(2 * i)]);  // Q(i) consumed
        if (has_next) {
          mbar_wait(&slot_full[slot_of(2 * i + 3)], phase_of(2 * i + 3));
          TRACE(1024 + 8 * (i & 127) + 4, blockIdx.x == 0);
          // dV(i) reads P^T(i) from the dP^T columns; dP^T(i+1) may follow it
          // at once (tcgen05.mma ops of one thread execute in issue order)
          TRACE(1024 + 8 * (i & 127) + 2, blockIdx.x == 0);
          tc_fence_after();
          issue_dp(i + 1);
        }
      }
      umma_commit(acc_done);
    }
  } else {
    // ========================================================== compute
    constexpr int NC = C::kCols;
    const int wg = warp >> 2;                 // q columns [NC wg, NC wg + NC)
    const int r = (warp & 3) * 32 + lane;     // key row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const float sl2 = a.scale_log2;
    const int kpos = k0 + r;
    const uint32_t tS = tbase + lane_off + C::kColS + wg * NC;
    const uint32_t tP = tbase + lane_off + C::kColDP + wg * NC;
    // column entries walked with counters, the next q-tile's entry loaded a
    // whole q-tile ahead (its global-load latency stays off the compute path)
    int hs = 0, eidx = n_qt - 1;
    int ent_next = n_it > 0 ? ents[eidx] : 0;
    const int* rposv = mv.col_rpos() + e0;  // row-CSR index of each column entry (stored-dS slots)
    int rpos_next = (a.ds && n_it > 0) ? rposv[eidx] : 0;
    for (int i = 0; i < n_it; ++i) {
      const int ent = ent_next;
      const int rpos = rpos_next, hcur = hs;
      if (++hs == a.group) {
        hs = 0;
        if (--eidx >= 0) {
          ent_next = ents[eidx];
          if (a.ds) rpos_next = rposv[eidx];
        }
      }
      const int qt = entry_tile(ent);
      int q0, q1, qseg;
      tile_bounds(g, qt, q0, q1, qseg);
      const bool need_mask = entry_kind(ent) == kKindPartial || (q1 - q0) < 128 || (k1 - k0) < 128;
      const float* sv = reinterpret_cast<const float*>(smem + C::kOffVec + (i & 1) * C::kVecBytes) + wg * NC;
      mbar_wait(&vec_full[i & 1], (i >> 1) & 1);
      TRACE(8 * (i & 127) + 0, blockIdx.x == 0 && threadIdx.x == 0);
      mbar_wait(s_full, i & 1);
      TRACE(8 * (i & 127) + 1, blockIdx.x == 0 && threadIdx.x == 0);
      tc_fence_after();
      // phase 1: P = exp2(S^T sl2 - lse2_q)
      float pv[NC];
      {
        uint32_t sr[NC];
        tmem_ld32(tS, sr);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p1_done);  // S^T(i) read: S^T(i+1) may be issued
        if (need_mask) {
          // visible q rows of this key form one interval (tilemap.cuh key_interval)
          int qa, qb;
          key_interval(g, kseg, kpos, qseg, qa, qb);
          if (qb > q1) qb = q1;
          if (kpos >= k1) qb = qa;
          const int cbase = q0 + wg * NC;
          p_tile<true, NC>(sr, sv, sl2, qa - cbase, qb - cbase, pv);
        } else {
          p_tile<false, NC>(sr, sv, sl2, 0, NC, pv);
        }
      }
      TRACE(8 * (i & 127) + 2, blockIdx.x == 0 && threadIdx.x == 0);
      // phase 2: dS = P (dP - D); P^T, dS^T (bf16) over the dP^T columns just
      // read, in two halves (q columns 0-15 and 16-31 of the warpgroup = the
      // even and odd k-steps of dV / dK): the even k-steps of dV(i), dK(i) run
      // while the odd half is computed
      mbar_wait(dp_full, i & 1);
      TRACE(8 * (i & 127) + 3, blockIdx.x == 0 && threadIdx.x == 0);
      tc_fence_after();
      static_assert(NC == 32, "split P^T arrival assumes 32 q columns per warpgroup");
      {
        uint32_t dr[NC], dsk[NC / 2], pk[NC / 2];
        tmem_ld32(tP, dr);
        tmem_ld_wait();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int j = 8 * hh; j < 8 * hh + 8; ++j) {
            const float2 ds = fmul2(make_float2(pv[2 * j], pv[2 * j + 1]),
                                    fadd2(make_float2(__uint_as_float(dr[2 * j]), __uint_as_float(dr[2 * j + 1])),
                                          make_float2(sv[128 + 2 * j], sv[128 + 2 * j + 1])));  // sv = -D
            dsk[j] = pack_bf16x2(ds.x, ds.y);
            pk[j] = pack_bf16x2(pv[2 * j], pv[2 * j + 1]);
          }
          tmem_st8(tP + 8 * hh, pk + 8 * hh);
          tmem_st8(tP + 16 + 8 * hh, dsk + 8 * hh);  // dS^T (bf16) beside P^T: A of dK += dS^T Q
          if (hh == 0) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pt_half[wg]);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&pt_done[wg]);  // this warpgroup's P^T(i), dS^T(i) written: its dV(i), dK(i) k-steps may issue
          mbar_arrive(&vec_empty[i & 1]);
        }
        if (a.ds) {
          // this key row's 32 q columns of dS^T(i) -> its tile slot (64 B),
          // after the arrive (off the MMA chain), streaming (evict-first) so
          // the Q / dO tiles the group's CTAs share stay in L2
          // tile layout: 16 chunks of 8 q columns, each [128 keys][8 q] (16 B
          // per key) -- the no-swizzle MN-major UMMA layout of the dQ
          // kernel's A operand, and each warp's store u is 512 contiguous bytes
          const long long slot = ((long long)b * a.n_q_heads + kvh * a.group + hcur) * a.ds_stride + rpos;
          __nv_bfloat16* dst = a.ds + slot * (kTileRows * kTileRows) + ((4 * wg) * kTileRows + r) * 8;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(dst + u * kTileRows * 8),
                         "r"(dsk[4 * u]), "r"(dsk[4 * u + 1]), "r"(dsk[4 * u + 2]), "r"(dsk[4 * u + 3])
                         : "memory");
        }
      }
      TRACE(8 * (i & 127) + 4, blockIdx.x == 0 && threadIdx.x == 0);
    }
    // ---- epilogue: dK (scaled), dV -> bf16; warpgroup wg stores columns [D/4 wg, +D/4)
    if (n_it > 0) {
      mbar_wait(acc_done, 0);
      tc_fence_after();
    }
    const bool ok = kpos < k1;
    constexpr int DC = D / C::kWGs;  // 32 (D = 128) or 16 (D = 64)
    const size_t orow = (((size_t)b * a.N + kpos) * a.kv_row_heads + kvh) * D + wg * DC;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t col = (which ? C::kColDK : C::kColDV) + wg * DC;
      const float mul = n_it > 0 ? (which ? a.scale : 1.f) : 0.f;
      __nv_bfloat16* out = (which ? a.dk : a.dv) + orow;
      uint32_t v[32];
      if (DC == 32) {
        tmem_ld32(tbase + lane_off + col, v);
      } else {
        tmem_ld16(tbase + lane_off + col, v);
      }
      tmem_ld_wait();
      if (n_it == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0u;
      }
      store_row_bf16_n<DC>(out, v, mul, ok);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::kTmemCols>(tbase);
  if (a.trace == 3 && threadIdx.x == 0 && blockIdx.x < 32768) {  // BD_TRACE=3: per-CTA timeline
    long long* e = g_cta_tl + 4 * blockIdx.x;
    e[0] = t_entry;
    e[1] = gtimer();
    e[2] = n_it;
    e[3] = smid();
  }
}

// ===================================================================== dQ
template <int D>
struct DqCfg {
  static constexpr int kTileBytes = 128 * D * 2;
  // K tiles live from S(j) to dQ(j), V tiles only until dP(j): separate rings,
  // K(j) -> slot j % kKSlots, V(j) -> slot kKSlots + j % kVSlots (ring index 2j / 2j+1).
#ifndef BD_DQ_KSLOTS
#define BD_DQ_KSLOTS 4
#endif
  // 4 K slots + 1 V slot measured 1.5% faster than 3 + 2 (K(j+2) no longer waits
  // for its load behind dQ(j-1); V(j+1) has a whole period to land)
  static constexpr int kKSlots = BD_DQ_KSLOTS, kVSlots = 5 - BD_DQ_KSLOTS;
  static constexpr int kStages = kKSlots + kVSlots;
  static constexpr int kWGs = 4;     // compute warpgroups, 32 key columns each
  static constexpr int kComputeWarps = 4 * kWGs;
  static constexpr int kTmaWarp = kComputeWarps;
  static constexpr int kMmaWarp = kComputeWarps + 1;
  static constexpr int kThreads = 32 * (kComputeWarps + 2);
  static constexpr int kColS0 = 0, kColS1 = 128, kColDP = 256, kColDQ = 384;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kOffQ = 0;
  static constexpr int kOffDO = kTileBytes;
  static constexpr int kOffRing = 2 * kTileBytes;
  static constexpr int kOffBar = kOffRing + kStages * kTileBytes;
  // q_full, kv_full[S], kv_empty[S], s_full[2], dp_full, dp_free, compute_done[2], acc_full,
  // qdo_empty, acc_empty, unit_full[2], unit_empty[2]
  static constexpr int kNumBars = 1 + 2 * kStages + 13;
  // unit ring (2 slots): the TMA warp publishes each unit's decoded
  // descriptor (128 B) and its rows' -log2 LSE and -D (2 x 512 B, bulk copy)
  static constexpr int kOffUnit = (kOffBar + kNumBars * 8 + 16 + 127) / 128 * 128;
  static constexpr int kSmemBytes = kOffUnit + 2 * 128 + 2 * 1024;
  static_assert(kSmemBytes <= 232448, "dq smem budget");
};

// ring index 2j = K(j), 2j+1 = V(j)
template <class C>
__device__ __forceinline__ int dq_ring_slot(int idx) {
  const int j = idx >> 1;
  return (idx & 1) ? C::kKSlots + j % C::kVSlots : j % C::kKSlots;
}
template <class C>
__device__ __forceinline__ uint32_t dq_ring_phase(int idx) {
  const int j = idx >> 1;
  return (uint32_t)(((idx & 1) ? j / C::kVSlots : j / C::kKSlots) & 1);
}

// ================================================================ dQ, persistent
// One CTA per SM walks the dQ work units (same unit order as the one-CTA-per-
// unit grid: (sequence, kv head)-major, LPT rank, q-head) with a static
// stride.  The TMA / MMA / compute pipelines run on across units, so the
// per-unit prologue (TMEM alloc, barrier init, Q / dO / first K, V loads, the
// first S and dP) and epilogue overlap the neighbouring units' work instead of
// costing ~5 us per unit (BD_TRACE=2 timeline: 11% of the one-CTA-per-unit
// kernel).  Q / dO of unit u+1 load as soon as the last S and dP MMAs of unit
// u are issued; the first dQ MMA of unit u+1 waits for the compute warps to
// have drained unit u's accumulator from TMEM.
struct __align__(128) DqUnit {  // one 128 B slot of the unit ring
  int b, h, qt, n_kt, q0, q1, qseg, u;
  const int* ents;
  Geom g;
  bool valid;
};

template <bool VARLEN>
__device__ __forceinline__ DqUnit dq_unit(const BwdArgs& a, int u) {
  const Geom& gm = a.g;
  DqUnit r;
  const int per_unit = gm.NT * a.group;
  const int unit = u / per_unit;
  const int rem = u - unit * per_unit;
  const int rank = rem / a.group;
  const int mi = unit / a.n_kv_heads;
  const int kvh = unit - mi * a.n_kv_heads;
  r.h = kvh * a.group + (rem - rank * a.group);
  const int* mapb = VARLEN ? a.map + (size_t)mi * a.map_stride : a.map;
  r.u = u;
  r.b = VARLEN ? map_seq(mapb) : mi;
  r.g = VARLEN ? map_geom(mapb) : gm;
  r.valid = !(VARLEN && rank >= r.g.NT);
  if (!r.valid) {
    r.n_kt = 0;
    return r;
  }
  const MapView mv{const_cast<int*>(mapb), r.g.NT, map_capacity(r.g)};
  r.qt = mv.fwd_order()[rank];
  const int e0 = mv.row_ptr()[r.qt];
  r.n_kt = mv.row_ptr()[r.qt + 1] - e0;
  r.ents = mv.row_ent() + e0;
  tile_bounds(r.g, r.qt, r.q0, r.q1, r.qseg);
  return r;
}

template <int D, bool VARLEN>
__global__ void __launch_bounds__(DqCfg<D>::kThreads, 1)
    attn_bwd_dqp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                        const BwdArgs a, int n_units) {
  using C = DqCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + C::kOffQ;
  uint8_t* sDO = smem + C::kOffDO;
  uint8_t* sRing = smem + C::kOffRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;  // [2]
  uint64_t* dp_full = s_full + 2;
  uint64_t* dp_free = dp_full + 1;
  // [2]: dS(jg) written, one barrier per S buffer -- the warps can reach tile
  // jg+1 (its dP was issued before the MMA thread waits for tile jg), never
  // jg+2 (its S is issued after that wait), so no phase passes unobserved
  uint64_t* compute_done = dp_free + 1;
  uint64_t* acc_full = compute_done + 2;
  uint64_t* qdo_empty = acc_full + 1;  // last S, dP of a unit done: Q / dO reusable
  uint64_t* acc_empty = qdo_empty + 1;  // compute warps drained dQ from TMEM
  uint64_t* unit_full = acc_empty + 1;   // [2] descriptor + LSE / D of a unit published
  uint64_t* unit_empty = unit_full + 2;  // [2] read by the MMA thread and the 16 compute warps
  uint32_t* tslot = reinterpret_cast<uint32_t*>(unit_empty + 2);
  DqUnit* udesc = reinterpret_cast<DqUnit*>(smem + C::kOffUnit);           // [2], 128 B apart
  float* uvec = reinterpret_cast<float*>(smem + C::kOffUnit + 2 * 128);    // [2][256]
  static_assert(sizeof(DqUnit) <= 128, "unit descriptor slot");

  const int warp = (int)warp_id(), lane = (int)lane_id();
  if ((smem_u32(smem) & 1023u) != 0) __trap();

  if (warp == 0) tmem_alloc<C::kTmemCols>(tslot);
  if (warp == C::kTmaWarp && lane == 0) {
    mbar_init(q_full, 1);
    for (int s2 = 0; s2 < C::kStages; ++s2) {
      mbar_init(&kv_full[s2], 1);
      mbar_init(&kv_empty[s2], 1);
    }
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(dp_full, 1);
    mbar_init(dp_free, C::kComputeWarps);
    mbar_init(&compute_done[0], C::kComputeWarps);
    mbar_init(&compute_done[1], C::kComputeWarps);
    mbar_init(acc_full, 1);
    mbar_init(qdo_empty, 1);
    mbar_init(acc_empty, C::kComputeWarps);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&unit_full[t], 1);
      mbar_init(&unit_empty[t], C::kComputeWarps + 1);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == C::kTmaWarp) {
    // ================================================================ TMA
    if (elect_one()) {
      int jg = 0, uu = 0;  // tiles and units this CTA has issued
      // publication uu of the unit ring: slot uu & 1; a descriptor with
      // valid = false ends the stream
      auto publish = [&](const DqUnit& w, int pu) {
        const int sl = pu & 1;
        mbar_wait(&unit_empty[sl], (uint32_t)(((pu >> 1) & 1) ^ 1));
        udesc[sl] = w;
        if (w.valid) {
          mbar_expect_tx(&unit_full[sl], 1024);
          const size_t v0 = (((size_t)w.b * a.n_q_heads + w.h) * a.g.NT + w.qt) * kTileRows;
          bulk_load(uvec + sl * 256, a.lse2_t + v0, 512, &unit_full[sl]);
          bulk_load(uvec + sl * 256 + 128, a.dsum_t + v0, 512, &unit_full[sl]);
        } else {
          mbar_arrive(&unit_full[sl]);
        }
      };
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const DqUnit w = dq_unit<VARLEN>(a, u);
        if (!w.valid) continue;
        publish(w, uu);
        const int kvh = w.h / a.group;
        mbar_wait(qdo_empty, (uint32_t)((uu & 1) ^ 1));
        mbar_expect_tx(q_full, 2 * C::kTileBytes);
        for (int kb = 0; kb < D / 64; ++kb) {
          tma_load_4d(sQ + kb * 16384, &tmQ, q_full, kb * 64, w.h, w.q0, w.b);
          tma_load_4d(sDO + kb * 16384, &tmDO, q_full, kb * 64, w.h, w.q0, w.b);
        }
        for (int j = 0; j < w.n_kt; ++j, ++jg) {
          const int k0 = tile_start(w.g, entry_tile(w.ents[j]));
#pragma unroll
          for (int kv = 0; kv < 2; ++kv) {
            const int stage = dq_ring_slot<C>(2 * jg + kv);
            mbar_wait(&kv_empty[stage], dq_ring_phase<C>(2 * jg + kv) ^ 1);
#ifdef BD_DQ_T_NOKV  // timing-only build: K / V loaded once per ring slot, never again (wrong results)
            if (jg >= C::kStages) {
              mbar_arrive(&kv_full[stage]);
              continue;
            }
#endif
            mbar_expect_tx(&kv_full[stage], C::kTileBytes);
            uint8_t* dst = sRing + stage * C::kTileBytes;
            for (int kb = 0; kb < D / 64; ++kb)
              tma_load_4d(dst + kb * 16384, kv ? &tmV : &tmK, &kv_full[stage], kb * 64, kvh, k0, w.b);
          }
        }
        ++uu;
      }
      {
        DqUnit end = {};
        end.valid = false;
        publish(end, uu);
      }
      if (uu > 0) mbar_wait(qdo_empty, (uint32_t)((uu - 1) & 1));  // observe the last unit's release
    }
  } else if (warp == C::kMmaWarp) {
    // ================================================================ MMA
    if (elect_one()) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_q = umma_idesc_bf16(128, D, false, true);
      const uint32_t qaddr = smem_u32(sQ), doaddr = smem_u32(sDO);
      auto slot = [&](int idx) { return dq_ring_slot<C>(idx); };
      auto ph = [&](int idx) { return dq_ring_phase<C>(idx); };
      auto ring = [&](int idx) { return smem_u32(sRing + slot(idx) * C::kTileBytes); };
      auto issue_s = [&](int jg) {
        const uint32_t kaddr = ring(2 * jg);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
#ifdef BD_DQ_T_TS  // timing-only: A from TMEM (garbage: the dQ columns), as if Q lived in TMEM
          umma_ts(tbase + ((jg & 1) ? C::kColS1 : C::kColS0), tbase + C::kColDQ + k * 8,
                  umma_desc_sw128(kaddr + off, 16, 1024), idesc_s, k > 0);
#else
          umma_ss(tbase + ((jg & 1) ? C::kColS1 : C::kColS0), umma_desc_sw128(qaddr + off, 16, 1024),
                  umma_desc_sw128(kaddr + off, 16, 1024), idesc_s, k > 0);
#endif
        }
        umma_commit(&s_full[jg & 1]);
      };
      auto issue_dp = [&](int jg) {
        const uint32_t vaddr = ring(2 * jg + 1);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
#ifdef BD_DQ_T_TS
          umma_ts(tbase + C::kColDP, tbase + C::kColDQ + 64 + k * 8, umma_desc_sw128(vaddr + off, 16, 1024), idesc_s,
                  k > 0);
#else
          umma_ss(tbase + C::kColDP, umma_desc_sw128(doaddr + off, 16, 1024),
                  umma_desc_sw128(vaddr + off, 16, 1024), idesc_s, k > 0);
#endif
        }
        umma_commit(dp_full);
        umma_commit(&kv_empty[slot(2 * jg + 1)]);  // V consumed
      };
      int jb = 0, uu = 0;  // first global tile of the unit, units done
      for (;; ) {
        const int sl = uu & 1;
        mbar_wait(&unit_full[sl], (uint32_t)((uu >> 1) & 1));
        const bool valid = udesc[sl].valid;
        const int n = udesc[sl].n_kt;
        mbar_arrive(&unit_empty[sl]);
        if (!valid) break;
        mbar_wait(q_full, (uint32_t)(uu & 1));
        mbar_wait(&kv_full[slot(2 * jb)], ph(2 * jb));
        tc_fence_after();
        issue_s(jb);
        mbar_wait(&kv_full[slot(2 * jb + 1)], ph(2 * jb + 1));
        tc_fence_after();
        issue_dp(jb);
        if (n == 1) umma_commit(qdo_empty);  // last S and dP of the unit issued
        if (n > 1) {
          mbar_wait(&kv_full[slot(2 * jb + 2)], ph(2 * jb + 2));
          tc_fence_after();
          issue_s(jb + 1);
        }
        for (int j = 0; j < n; ++j) {
          const int jg = jb + j;
          mbar_wait(dp_free, (uint32_t)(jg & 1));
          if (j + 1 < n) {
            mbar_wait(&kv_full[slot(2 * jg + 3)], ph(2 * jg + 3));
            tc_fence_after();
            issue_dp(jg + 1);
            if (j + 2 == n) umma_commit(qdo_empty);  // dP(n-1) follows S(n-1)
          }
          mbar_wait(&compute_done[jg & 1], (uint32_t)((jg >> 1) & 1));
          if (j == 0) mbar_wait(acc_empty, (uint32_t)((uu & 1) ^ 1));  // previous unit's dQ drained
          tc_fence_after();
          const uint32_t sbase = tbase + ((jg & 1) ? C::kColS1 : C::kColS0);
          const uint32_t kaddr = ring(2 * jg);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            umma_ts(tbase + C::kColDQ, sbase + 32 * (k >> 1) + 8 * (k & 1),
                    umma_desc_sw128(kaddr + k * 2048, 16384, 1024), idesc_q, (j > 0 || k > 0) ? 1u : 0u);
          umma_commit(&kv_empty[slot(2 * jg)]);  // K consumed
          if (j + 2 < n) {
            mbar_wait(&kv_full[slot(2 * jg + 4)], ph(2 * jg + 4));
            tc_fence_after();
            issue_s(jg + 2);
          }
        }
        umma_commit(acc_full);
        jb += n;
        ++uu;
      }
      if (uu > 0) mbar_wait(acc_empty, (uint32_t)((uu - 1) & 1));  // observe the last drain
    }
  } else {
    // ========================================================== compute
    const int wg = warp >> 2;
    const int r = (warp & 3) * 32 + lane;  // query row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const float sl2 = a.scale_log2;
    const int cb = wg * 32;
    int jg = 0, uu = 0;
    for (;; ) {
      const int sl = uu & 1;
      mbar_wait(&unit_full[sl], (uint32_t)((uu >> 1) & 1));
      const DqUnit w = udesc[sl];
      if (!w.valid) break;
      const long long t_unit = (a.trace == 2 && threadIdx.x == 0) ? gtimer() : 0;
      const float nlse2 = uvec[sl * 256 + r];  // -lse2 and -D (negated by bwd_pre)
      const float ndsum = uvec[sl * 256 + 128 + r];
      int ent_next = w.ents[0];
      __syncwarp();
      if (lane == 0) mbar_arrive(&unit_empty[sl]);
      const int u = w.u;
      const Geom& g = w.g;
      const int row = w.q0 + r;
      int lo0, hi0, lo1, hi1;
      row_interval(g, w.qseg, row, 0, lo0, hi0);
      row_interval(g, w.qseg, row, w.qseg ? w.qseg : 1, lo1, hi1);  // the row's own noisy copy
      for (int j = 0; j < w.n_kt; ++j, ++jg) {
        const int ent = ent_next;
        if (j + 1 < w.n_kt) ent_next = w.ents[j + 1];
        const int kt = entry_tile(ent);
        const int k0 = tile_start(g, kt), k1 = tile_end(g, kt);
        const bool need_mask = entry_kind(ent) == kKindPartial || (k1 - k0) < 128;
        const bool xt = tile_seg(g, kt) != 0;
        const int lo = (xt ? lo1 : lo0) - k0;
        const int hi = min(xt ? hi1 : hi0, k1) - k0;
        const uint32_t sbase = tbase + lane_off + ((jg & 1) ? C::kColS1 : C::kColS0);
        mbar_wait(&s_full[jg & 1], (uint32_t)((jg >> 1) & 1));
        tc_fence_after();
#ifdef BD_DQ_T_NOCOMP  // timing-only build: no TMEM traffic or math in the compute warps (wrong results)
        (void)need_mask; (void)lo; (void)hi; (void)sbase;
        mbar_wait(dp_full, (uint32_t)(jg & 1));
        tc_fence_after();
        __syncwarp();
        if (lane == 0) mbar_arrive(dp_free);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&compute_done[jg & 1]);
        continue;
#endif
        float pv[32];
        {
          uint32_t sr[32];
          tmem_ld32(sbase + cb, sr);
          tmem_ld_wait();
          if (need_mask)
            p_row<true>(sr, nlse2, sl2, lo - cb, hi - cb, pv);
          else
            p_row<false>(sr, nlse2, sl2, 0, 32, pv);
        }
        mbar_wait(dp_full, (uint32_t)(jg & 1));
        tc_fence_after();
        uint32_t pk[16];
        {
          uint32_t dr[32];
          tmem_ld32(tbase + lane_off + C::kColDP + cb, dr);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_free);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const float2 ds = fmul2(make_float2(pv[2 * jj], pv[2 * jj + 1]),
                                    fadd2(make_float2(__uint_as_float(dr[2 * jj]), __uint_as_float(dr[2 * jj + 1])),
                                          make_float2(ndsum, ndsum)));
            pk[jj] = pack_bf16x2(ds.x, ds.y);
          }
        }
        tmem_st16(sbase + cb, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&compute_done[jg & 1]);
      }
      // ---- epilogue of the unit: dQ = scale * acc -> bf16
      mbar_wait(acc_full, (uint32_t)(uu & 1));
      tc_fence_after();
      constexpr int DC = D / C::kWGs;
      uint32_t v[32];
      if (DC == 32)
        tmem_ld32(tbase + lane_off + C::kColDQ + wg * DC, v);
      else
        tmem_ld16(tbase + lane_off + C::kColDQ + wg * DC, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);  // accumulator free for the next unit
      __nv_bfloat16* out = a.dq + (((size_t)w.b * a.N + row) * a.q_row_heads + w.h) * D + wg * DC;
      store_row_bf16_n<DC>(out, v, a.scale, row < w.q1);
      if (a.trace == 2 && threadIdx.x == 0 && u < 32768) {
        long long* e = g_cta_tl + 4 * u;
        e[0] = t_unit;
        e[1] = gtimer();
        e[2] = w.n_kt;
        e[3] = smid();
      }
      ++uu;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::kTmemCols>(tbase);
}

template <typename K>
int set_smem(K kernel, int bytes) {
  return ensure_smem_attr(reinterpret_cast<const void*>(kernel), bytes, "cudaFuncSetAttribute(bwd)");
}

// ========================================================= dQ from stored dS
// dQ = scale dS K over a q-tile's row of tiles, dS^T read from the workspace
// where the dK/dV kernel stored it (BwdArgs::ds): no S / dP recompute, no
// exps -- 2 d FLOP per visible pair instead of 6 d, and the kernel streams
// each tile's 32 KB of dS^T once from HBM (the K tiles, shared by the
// group's heads and the sequence's q-tiles, come from L2).  Persistent: one
// CTA per SM walks the dQ units in the same order as attn_bwd_dqp_kernel.
// Warps 0-3: epilogue (TMEM lane quarters); warp 4: TMA; warp 5: MMA.
// TMEM: two D-column dQ accumulators (unit u in buffer u & 1), so a unit's
// drain overlaps the next unit's MMAs.
template <int D>
struct DqDsCfg {
  // dS^T tile, bf16: 16 chunks of 8 q columns, each [128 keys][8 q] (the
  // no-swizzle MN-major A layout; one 32 KB bulk copy per tile)
  static constexpr int kDsBytes = kTileRows * kTileRows * 2;
  static constexpr int kKBytes = kTileRows * D * 2;
  static constexpr int kStageBytes = kDsBytes + kKBytes;
  static constexpr int kStages = D == 128 ? 3 : 4;
  static constexpr int kTmaWarp = 4, kMmaWarp = 5;
  static constexpr int kThreads = 6 * 32;
  static constexpr uint32_t kTmemCols = 2 * D;
  static constexpr int kOffBar = kStages * kStageBytes;
  // full[S], empty[S], acc_full[2], acc_empty[2]
  static constexpr int kNumBars = 2 * kStages + 4;
  static constexpr int kSmemBytes = kOffBar + kNumBars * 8 + 16;
  static_assert(kSmemBytes <= 232448, "dq-ds smem budget");
};

template <int D>
__global__ void __launch_bounds__(DqDsCfg<D>::kThreads, 1)
    attn_bwd_dq_ds_kernel(const __grid_constant__ CUtensorMap tmK, const BwdArgs a, int n_units) {
  using C = DqDsCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* full = bars;
  uint64_t* empty = full + C::kStages;
  uint64_t* acc_full = empty + C::kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);
  const int warp = (int)warp_id(), lane = (int)lane_id();
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  if (warp == 0) tmem_alloc<C::kTmemCols>(tslot);
  if (warp == C::kTmaWarp && lane == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmK);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const MapView mv{const_cast<int*>(a.map), a.g.NT, map_capacity(a.g)};

  if (warp == C::kTmaWarp) {
    // ================================================================ TMA
    if (elect_one()) {
      int it = 0;  // tiles issued by this CTA
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const DqUnit w = dq_unit<false>(a, u);
        const int kvh = w.h / a.group;
        const long long slot0 = ((long long)w.b * a.n_q_heads + w.h) * a.ds_stride + mv.row_ptr()[w.qt];
        for (int j = 0; j < w.n_kt; ++j, ++it) {
          const int st = it % C::kStages;
          mbar_wait(&empty[st], (uint32_t)(((it / C::kStages) & 1) ^ 1));
          mbar_expect_tx(&full[st], C::kStageBytes);
          uint8_t* dst = smem + st * C::kStageBytes;
          bulk_load(dst, a.ds + (slot0 + j) * (kTileRows * kTileRows), C::kDsBytes, &full[st]);
          const int k0 = tile_start(w.g, entry_tile(w.ents[j]));
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_4d(dst + C::kDsBytes + kb * 16384, &tmK, &full[st], kb * 64, kvh, k0, w.b);
        }
      }
    }
  } else if (warp == C::kMmaWarp) {
    // ================================================================ MMA
    if (elect_one()) {
      // A = dS (M = q rows, K = keys): the stored dS^T tile is MN-major A;
      // B = K (K = keys, N = d): MN-major B
      constexpr uint32_t idesc = umma_idesc_bf16(128, D, true, true);
      int it = 0, uu = 0;  // tiles consumed, units with tiles
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const DqUnit w = dq_unit<false>(a, u);
        if (w.n_kt == 0) continue;
        const int ab = uu & 1;
        mbar_wait(&acc_empty[ab], (uint32_t)(((uu >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t acc = tbase + ab * D;
        for (int j = 0; j < w.n_kt; ++j, ++it) {
          const int st = it % C::kStages;
          mbar_wait(&full[st], (uint32_t)((it / C::kStages) & 1));
          tc_fence_after();
          const uint32_t sds = smem_u32(smem + st * C::kStageBytes), sk = sds + C::kDsBytes;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            umma_ss(acc, umma_desc_noswz(sds + k * 256, 128, 2048), umma_desc_sw128(sk + k * 2048, 16384, 1024),
                    idesc, (j > 0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[st]);
        }
        umma_commit(&acc_full[ab]);
        ++uu;
      }
    }
  } else if (warp < 4) {
    // =========================================================== epilogue
    const int r = warp * 32 + lane;  // query row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    int uu = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const DqUnit w = dq_unit<false>(a, u);
      const int row = w.q0 + r;
      const bool ok = row < w.q1;
      __nv_bfloat16* out = a.dq + (((size_t)w.b * a.N + row) * a.q_row_heads + w.h) * D;
      if (w.n_kt == 0) {
        uint32_t z[32] = {};
#pragma unroll
        for (int c = 0; c < D / 32; ++c) store_row_bf16(out + 32 * c, z, 0.f, ok);
        continue;
      }
      const int ab = uu & 1;
      mbar_wait(&acc_full[ab], (uint32_t)((uu >> 1) & 1));
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + lane_off + ab * D + 32 * c, v);
        tmem_ld_wait();
        store_row_bf16(out + 32 * c, v, a.scale, ok);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
      ++uu;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D, bool VARLEN>
int launch_bwd(const bd_problem& p, const Geom& g, const void* q, const void* k, const void* v, const void* o,
               const float* lse, const void* dout, void* dq, void* dk, void* dv, const int* map, int map_stride,
               float* vec_ws, const DsPlan& ds, cudaStream_t stream) {
  const int Hq = p.n_q_heads;
  const size_t nvec = (size_t)p.batch * Hq * g.NT * kTileRows;
  float* lse2_t = vec_ws;
  float* dsum_t = vec_ws + nvec;
  // 1. preprocess: D and log2 LSE, tile-major (pad rows zeroed)
  zero_kernel<<<296, 256, 0, stream>>>(reinterpret_cast<float4*>(vec_ws), 2 * nvec / 4);
  {
    constexpr int kRows = 256 / (D / 8);
    dim3 grid((g.N + kRows - 1) / kRows, p.batch * Hq);
    bwd_pre_kernel<D, VARLEN><<<grid, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(o),
                                                         reinterpret_cast<const __nv_bfloat16*>(dout), lse, lse2_t,
                                                         dsum_t, g.N, Hq, q_row_heads(p), g, map, map_stride);
  }
  CUtensorMap tmQ, tmK, tmV, tmDO;
  const int qrh = q_row_heads(p), kvrh = kv_row_heads(p);
  if (!make_qkv_tmap(&tmQ, q, p.batch, g.N, Hq, D, 128, qrh) ||
      !make_qkv_tmap(&tmK, k, p.batch, g.N, p.n_kv_heads, D, 128, kvrh) ||
      !make_qkv_tmap(&tmV, v, p.batch, g.N, p.n_kv_heads, D, 128, kvrh) ||
      !make_qkv_tmap(&tmDO, dout, p.batch, g.N, Hq, D, 128, qrh))
    return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  int rc = set_smem(attn_bwd_dkdv_kernel<D, VARLEN>, DkdvCfg<D>::kSmemBytes);
  if (rc) return rc;
  if ((rc = set_smem(attn_bwd_dqp_kernel<D, VARLEN>, DqCfg<D>::kSmemBytes))) return rc;
  if (!VARLEN && (rc = set_smem(attn_bwd_dq_ds_kernel<D>, DqDsCfg<D>::kSmemBytes))) return rc;
  BwdArgs a;
  a.map = map;
  a.map_stride = map_stride;
  a.lse2_t = lse2_t;
  a.dsum_t = dsum_t;
  a.dq = reinterpret_cast<__nv_bfloat16*>(dq);
  a.dk = reinterpret_cast<__nv_bfloat16*>(dk);
  a.dv = reinterpret_cast<__nv_bfloat16*>(dv);
  a.batch = p.batch;
  a.n_q_heads = Hq;
  a.n_kv_heads = p.n_kv_heads;
  a.q_row_heads = qrh;
  a.kv_row_heads = kvrh;
  a.group = Hq / p.n_kv_heads;
  a.N = g.N;
  a.g = g;
  a.scale = scale_of(p);
  a.scale_log2 = a.scale * kLog2e;
  static const int trace_on = getenv("BD_TRACE") ? atoi(getenv("BD_TRACE")) : 0;
  a.trace = trace_on;
  a.ds = nullptr;
  a.ds_stride = 0;
  int n_sm = 0;
  if ((rc = current_sm_count(&n_sm))) return rc;
  if (!VARLEN && ds.buf) {
    // stored-dS path, in chunks of ds.chunk sequences (the dS^T buffer holds
    // one chunk): dK/dV(chunk) writes every tile's dS^T, dQ(chunk) reads it
    const int Hkv = p.n_kv_heads;
    int launches = 2;  // zero, pre
    for (int s0 = 0; s0 < p.batch; s0 += ds.chunk) {
      const int nb = p.batch - s0 < ds.chunk ? p.batch - s0 : ds.chunk;
      const size_t qoff = (size_t)s0 * g.N * qrh * D, kvoff = (size_t)s0 * g.N * kvrh * D;
      const auto* qb = reinterpret_cast<const __nv_bfloat16*>(q) + qoff;
      const auto* kb = reinterpret_cast<const __nv_bfloat16*>(k) + kvoff;
      const auto* vb = reinterpret_cast<const __nv_bfloat16*>(v) + kvoff;
      const auto* dob = reinterpret_cast<const __nv_bfloat16*>(dout) + qoff;
      CUtensorMap cQ, cK, cV, cDO;
      if (!make_qkv_tmap(&cQ, qb, nb, g.N, Hq, D, 128, qrh) || !make_qkv_tmap(&cK, kb, nb, g.N, Hkv, D, 128, kvrh) ||
          !make_qkv_tmap(&cV, vb, nb, g.N, Hkv, D, 128, kvrh) ||
          !make_qkv_tmap(&cDO, dob, nb, g.N, Hq, D, 128, qrh))
        return set_error(BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
      BwdArgs c = a;
      c.batch = nb;
      c.lse2_t = lse2_t + (size_t)s0 * Hq * g.NT * kTileRows;
      c.dsum_t = dsum_t + (size_t)s0 * Hq * g.NT * kTileRows;
      c.dq = a.dq + qoff;
      c.dk = a.dk + kvoff;
      c.dv = a.dv + kvoff;
      c.ds = reinterpret_cast<__nv_bfloat16*>(ds.buf);
      c.ds_stride = ds.stride;
      const long long grid_kv = (long long)g.NT * nb * Hkv;
      attn_bwd_dkdv_kernel<D, VARLEN><<<(unsigned)grid_kv, DkdvCfg<D>::kThreads, DkdvCfg<D>::kSmemBytes, stream>>>(
          cQ, cK, cV, cDO, c);
      if ((rc = check_cuda(cudaGetLastError(), "attn_bwd_dkdv_kernel launch"))) return rc;
      const long long units = (long long)g.NT * nb * Hq;
      if (units > 0x7FFFFFFF) return set_error(BD_ERR_UNSUPPORTED, "grid too large");
      const int grid_p = (int)(units < n_sm ? units : n_sm);
      attn_bwd_dq_ds_kernel<D><<<(unsigned)grid_p, DqDsCfg<D>::kThreads, DqDsCfg<D>::kSmemBytes, stream>>>(
          cK, c, (int)units);
      if ((rc = check_cuda(cudaGetLastError(), "attn_bwd_dq_ds_kernel launch"))) return rc;
      launches += 2;
    }
    note_launches(launches);
    return BD_OK;
  }
  // 2. dK, dV
  const long long grid_kv = (long long)g.NT * p.batch * p.n_kv_heads;
  attn_bwd_dkdv_kernel<D, VARLEN><<<(unsigned)grid_kv, DkdvCfg<D>::kThreads, DkdvCfg<D>::kSmemBytes, stream>>>(
      tmQ, tmK, tmV, tmDO, a);
  if ((rc = check_cuda(cudaGetLastError(), "attn_bwd_dkdv_kernel launch"))) return rc;
  // 3. dQ
  const long long grid_q = (long long)g.NT * p.batch * Hq;
  if (grid_q > 0x7FFFFFFF) return set_error(BD_ERR_UNSUPPORTED, "grid too large");
  const int grid_p = (int)(grid_q < n_sm ? grid_q : n_sm);
  attn_bwd_dqp_kernel<D, VARLEN><<<(unsigned)grid_p, DqCfg<D>::kThreads, DqCfg<D>::kSmemBytes, stream>>>(
      tmQ, tmK, tmV, tmDO, a, (int)grid_q);
  note_launches(4);  // zero, pre, dkdv, dq
  return check_cuda(cudaGetLastError(), "attn_bwd_dqp_kernel launch");
}

}  // namespace

size_t ds_plan_bytes(const bd_problem& p, const Geom& g, long long* stride, int* chunk) {
  *stride = 0;
  *chunk = 0;
  // read per call (the workspace query and the launch of one call agree as
  // long as the environment does not change in between).  BD_BWD_DS unset:
  // on only when the whole batch fits one chunk of the budget (default
  // 8 GiB) -- where it pays (SDAR-1.7B bwd -12%); 1: on,
  // chunked, budget default 24 GiB; 0: off.
  const char* env = getenv("BD_BWD_DS");
  const int mode = env ? (atoi(env) != 0 ? 1 : 0) : 2;  // 2 = auto
  const char* benv = getenv("BD_BWD_DS_BUDGET_MB");
  const long long budget = (benv ? atoll(benv) : (mode == 1 ? 24576LL : 8192LL)) << 20;
  if (mode == 0 || is_varlen(p) || p.batch <= 0) return 0;
  const long long E = map_entries_bound(g);
  const long long per_seq = (long long)p.n_q_heads * E * kTileRows * kTileRows * 2;
  if (E <= 0 || per_seq > budget) return 0;
  if (mode == 2 && per_seq * p.batch > budget) return 0;
  const long long c = budget / per_seq;
  *chunk = (int)(c < p.batch ? c : p.batch);
  *stride = E;
  return (size_t)(*chunk) * (size_t)per_seq;
}

size_t bwd_vec_floats(const bd_problem& p, const Geom& g) {
  return 2 * (size_t)p.batch * p.n_q_heads * g.NT * kTileRows;
}

int run_attn_bwd(const bd_problem& p, const Geom& g, const void* q, const void* k, const void* v, const void* o,
                 const float* lse, const void* dout, void* dq, void* dk, void* dv, const int* map, int map_stride,
                 float* vec_ws, const DsPlan& ds, cudaStream_t stream) {
  const bool vl = map_stride != 0;
#define BD_BWD_CASE(D_)                                                                                      \
  return vl ? launch_bwd<D_, true>(p, g, q, k, v, o, lse, dout, dq, dk, dv, map, map_stride, vec_ws, ds, stream) \
            : launch_bwd<D_, false>(p, g, q, k, v, o, lse, dout, dq, dk, dv, map, map_stride, vec_ws, ds, stream)
  if (p.head_dim == 128) BD_BWD_CASE(128);
  if (p.head_dim == 64) BD_BWD_CASE(64);
#undef BD_BWD_CASE
  return set_error(BD_ERR_UNSUPPORTED, "head_dim %d not in {64, 128}", p.head_dim);
}

}  // namespace bd

extern "C" int bd_debug_cta_timeline(int64_t* host_out, int n) {
  if (!host_out || n <= 0 || n > 4 * 32768) return BD_ERR_INVALID_ARG;
  return bd::check_cuda(cudaMemcpyFromSymbol(host_out, bd::g_cta_tl, n * sizeof(long long)), "timeline copy");
}
extern "C" int bd_debug_trace(int64_t* host_out, int n) {
  if (!host_out || n <= 0 || n > 8192) return BD_ERR_INVALID_ARG;
  return bd::check_cuda(cudaMemcpyFromSymbol(host_out, bd::g_trace, n * sizeof(long long)), "trace copy");
}
