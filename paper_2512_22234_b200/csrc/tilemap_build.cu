// Tile-map builder: device kernel (writes the map into the caller's
// workspace on the call's stream -- no host round trip, no allocation) and
// the identical host path behind bd_tilemap_dump / bd_tilemap_stats.
#include "tilemap.cuh"
#include "abi_common.h"
#include "problem.h"

#include <algorithm>
#include <vector>

namespace bd {

// ------------------------------------------------------------------ host
void build_map_host(const Geom& g, std::vector<int>& w) {
  const int cap = map_capacity(g);
  w.assign(static_cast<size_t>(map_words(g)), 0);
  MapView mv{w.data(), g.NT, cap};
  w[0] = kMapMagic;
  w[1] = g.L;
  w[2] = g.xb;
  w[3] = g.B;
  w[4] = g.NT;
  w[5] = g.T0;
  w[8] = g.S;
  int n = 0, maxrow = 0;
  std::vector<int> rowlen(g.NT), collen(g.NT, 0);
  for (int t = 0; t < g.NT; ++t) {
    mv.row_ptr()[t] = n;
    const int qs = tile_seg(g, t);
    for (int kk = 0; kk < (qs ? 2 : 1); ++kk) {
      const int ks = kk ? qs : 0;  // x0, then the row's own copy
      int a, b;
      candidate_range(g, t, ks, a, b);
      for (int kt = a; kt < b; ++kt) {
        const int kind = classify_pair(g, t, kt);
        if (kind) {
          mv.row_ent()[n++] = entry_make(kt, kind);
          collen[kt]++;
        }
      }
    }
    rowlen[t] = n - mv.row_ptr()[t];
    maxrow = std::max(maxrow, rowlen[t]);
  }
  mv.row_ptr()[g.NT] = n;
  w[6] = n;
  w[7] = maxrow;
  int c = 0;
  for (int kt = 0; kt < g.NT; ++kt) {
    mv.col_ptr()[kt] = c;
    c += collen[kt];
  }
  mv.col_ptr()[g.NT] = c;
  std::vector<int> fill(g.NT, 0);
  for (int t = 0; t < g.NT; ++t)
    for (int e = mv.row_ptr()[t]; e < mv.row_ptr()[t + 1]; ++e) {
      const int kt = entry_tile(mv.row_ent()[e]);
      mv.col_rpos()[mv.col_ptr()[kt] + fill[kt]] = e;
      mv.col_ent()[mv.col_ptr()[kt] + fill[kt]++] = entry_make(t, entry_kind(mv.row_ent()[e]));
    }
  std::vector<int> ord(g.NT);
  for (int i = 0; i < g.NT; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return rowlen[a] > rowlen[b]; });
  for (int i = 0; i < g.NT; ++i) mv.fwd_order()[i] = ord[i];
  for (int i = 0; i < g.NT; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return collen[a] > collen[b]; });
  for (int i = 0; i < g.NT; ++i) mv.bwd_order()[i] = ord[i];
}

// ---------------------------------------------------------------- device
namespace {

constexpr int kBuildThreads = 1024;

// Exclusive scan of cnt[0..n) into out[0..n], out[n] = total.  All threads.
__device__ void block_exclusive_scan(const int* cnt, int* out, int n, int* scratch) {
  const int tid = threadIdx.x;
  const int per = (n + kBuildThreads - 1) / kBuildThreads;
  const int a = tid * per, b = min(n, a + per);
  int s = 0;
  for (int i = a; i < b; ++i) s += cnt[i];
  scratch[tid] = s;
  __syncthreads();
  // Hillis-Steele over the 1024 partials
  for (int off = 1; off < kBuildThreads; off <<= 1) {
    const int v = tid >= off ? scratch[tid - off] : 0;
    __syncthreads();
    scratch[tid] += v;
    __syncthreads();
  }
  int run = scratch[tid] - s;  // exclusive prefix of this chunk
  for (int i = a; i < b; ++i) {
    out[i] = run;
    run += cnt[i];
  }
  if (tid == kBuildThreads - 1) out[n] = scratch[tid];
  __syncthreads();
}

// Warp-cooperative classification of (qt, kt) from the per-row intervals of
// q-tile qt held in shared memory (lo/hi for key segment ks); same result as
// classify_pair.
__device__ int classify_pair_warp(const Geom& g, int qt, int kt, const int* s_lo, const int* s_hi) {
  const int nrow = tile_end(g, qt) - tile_start(g, qt);
  const int k0 = tile_start(g, kt), k1 = tile_end(g, kt);
  bool any = false, all = true;
  for (int r = (int)(threadIdx.x & 31); r < nrow; r += 32) {
    const int a = max(s_lo[r], k0), b = min(s_hi[r], k1);
    if (b > a) any = true;
    if (!(a == k0 && b == k1)) all = false;
  }
  any = __any_sync(0xffffffffu, any);
  all = __all_sync(0xffffffffu, all);
  return any ? (all ? kKindFull : kKindPartial) : 0;
}

#ifndef BD_MAP_TRACE
#define BD_MAP_TRACE 0
#endif
#if BD_MAP_TRACE
__device__ long long g_map_trace[16];
#define MAP_STAMP(i) \
  do {               \
    __syncthreads(); \
    if (threadIdx.x == 0 && blockIdx.x == 0) g_map_trace[i] = clock64(); \
  } while (0)
#else
#define MAP_STAMP(i) \
  do {               \
  } while (0)
#endif

// One warp per q-tile (strided).  Shared memory: rowlen[NT], collen[NT],
// colfill[NT], scan scratch[1024], and per warp 4 x 128 ints of row intervals.
// stage != 0 (the map fits): pass 1 also keeps every row's entries in shared
// memory (fixed stride cap / NT per q-tile), so the fill pass copies them
// instead of classifying every candidate a second time, and pass 3 reads
// entries and column pointers from shared memory (BD_MAP_TRACE: the two
// classification passes were ~85% of the builder's time).
__device__ void build_map_body(const Geom& g, int* __restrict__ ws, int seq, int stage) {
  extern __shared__ int sh[];
  const int NT = g.NT;
  int* rowlen = sh;                 // NT
  int* collen = sh + NT;            // NT
  int* colfill = sh + 2 * NT;       // NT
  int* scratch = sh + 3 * NT;       // kBuildThreads
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = kBuildThreads / 32;
  int* wiv = sh + 3 * NT + kBuildThreads + warp * 512;  // this warp's row intervals
  const int cap = map_capacity(g);
  const int stride = cap / NT;  // per-q-tile entry bound (T0 + own-copy tiles)
  int* s_cp = sh + 3 * NT + kBuildThreads + (kBuildThreads / 32) * 512;  // stage: col_ptr[NT + 1]
  int* s_ent = s_cp + NT + 1;                                              // stage: [NT][stride]
  MapView mv{ws, NT, cap};
  MAP_STAMP(0);
  for (int i = tid; i < NT; i += kBuildThreads) {
    collen[i] = 0;
    colfill[i] = 0;
  }
  __syncthreads();
  // passes 1 and 2: classify candidate k-tiles of each q-tile; count, then fill
  for (int pass = 0; pass < 2; ++pass) {
    if (pass && stage) {
      // fill from the entries kept by pass 1
      for (int t = warp; t < NT; t += nwarps) {
        const int r0 = mv.row_ptr()[t], n = rowlen[t];
        for (int i = lane; i < n; i += 32) {
          const int e = s_ent[t * stride + i];
          mv.row_ent()[r0 + i] = e;
          atomicAdd(&collen[entry_tile(e)], 1);
        }
      }
      __syncthreads();
      MAP_STAMP(3);
      MAP_STAMP(4);
      break;
    }
    for (int t = warp; t < NT; t += nwarps) {
      const int q0 = tile_start(g, t), nrow = tile_end(g, t) - q0, qs = tile_seg(g, t);
      for (int r = lane; r < nrow; r += 32) {
        row_interval(g, qs, q0 + r, 0, wiv[r], wiv[128 + r]);
        if (qs) row_interval(g, qs, q0 + r, qs, wiv[256 + r], wiv[384 + r]);
      }
      __syncwarp();
      int n = pass ? mv.row_ptr()[t] : 0;
      if (!pass) {
        // count (and, staged, keep) the row's entries: lane i classifies
        // candidate base + i over all rows of the tile (broadcast reads of the
        // row intervals), a ballot keeps the entries in increasing k-tile order
        for (int kk = 0; kk < (qs ? 2 : 1); ++kk) {
          const int ks = kk ? qs : 0;  // x0, then the row's own copy
          int a, b;
          candidate_range(g, t, ks, a, b);
          const int* s_lo = wiv + 256 * kk;
          const int* s_hi = s_lo + 128;
          for (int base = a; base < b; base += 32) {
            const int kt = base + lane;
            int kind = 0;
            if (kt < b) {
              const int k0 = tile_start(g, kt), k1 = tile_end(g, kt);
              bool any = false, all = true;
#pragma unroll 8
              for (int r = 0; r < nrow; ++r) {
                const int lo = max(s_lo[r], k0), hi = min(s_hi[r], k1);
                any |= hi > lo;
                all &= (lo == k0 && hi == k1);
              }
              kind = any ? (all ? kKindFull : kKindPartial) : 0;
            }
            const unsigned m = __ballot_sync(0xffffffffu, kind != 0);
            if (stage && kind) s_ent[t * stride + n + __popc(m & ((1u << lane) - 1u))] = entry_make(kt, kind);
            n += __popc(m);
          }
        }
        if (lane == 0) rowlen[t] = n;
        __syncwarp();
        continue;
      }
      for (int kk = 0; kk < (qs ? 2 : 1); ++kk) {
        const int ks = kk ? qs : 0;  // x0, then the row's own copy
        int a, b;
        candidate_range(g, t, ks, a, b);
        for (int kt = a; kt < b; ++kt) {
          const int kind = classify_pair_warp(g, t, kt, wiv + 256 * kk, wiv + 256 * kk + 128);
          if (kind) {
            if (lane == 0) {
              mv.row_ent()[n] = entry_make(kt, kind);
              atomicAdd(&collen[kt], 1);
            }
            ++n;
          }
        }
      }
      __syncwarp();
    }
    __syncthreads();
    MAP_STAMP(1 + 2 * pass);
    if (!pass) block_exclusive_scan(rowlen, mv.row_ptr(), NT, scratch);
    MAP_STAMP(2 + 2 * pass);
  }
  block_exclusive_scan(collen, mv.col_ptr(), NT, scratch);
  MAP_STAMP(5);
  if (stage) {
    for (int i = tid; i <= NT; i += kBuildThreads) s_cp[i] = mv.col_ptr()[i];
    __syncthreads();
  }
  // pass 3: column entries in increasing q-tile order -- warp 0 walks the rows
  // in order, lanes take a row's entries (each k-tile appears once per row)
  if (warp == 0) {
    for (int t = 0; t < NT; ++t) {
      if (stage) {
        const int n = rowlen[t];
        for (int i = lane; i < n; i += 32) {
          const int ent = s_ent[t * stride + i];
          const int kt = entry_tile(ent);
          mv.col_rpos()[s_cp[kt] + colfill[kt]] = mv.row_ptr()[t] + i;
          mv.col_ent()[s_cp[kt] + colfill[kt]++] = entry_make(t, entry_kind(ent));
        }
      } else {
        const int e0 = mv.row_ptr()[t], e1 = mv.row_ptr()[t + 1];
        for (int e = e0 + lane; e < e1; e += 32) {
          const int ent = mv.row_ent()[e];
          const int kt = entry_tile(ent);
          mv.col_rpos()[mv.col_ptr()[kt] + colfill[kt]] = e;
          mv.col_ent()[mv.col_ptr()[kt] + colfill[kt]++] = entry_make(t, entry_kind(ent));
        }
      }
      __syncwarp();
    }
  }
  MAP_STAMP(6);
  // pass 4: longest-first orders (stable: ties by index)
  for (int t = tid; t < NT; t += kBuildThreads) {
    const int lt = rowlen[t], ct = collen[t];
    int rr = 0, rc = 0;
    for (int u = 0; u < NT; ++u) {
      const int lu = rowlen[u], cu = collen[u];
      rr += (lu > lt) || (lu == lt && u < t);
      rc += (cu > ct) || (cu == ct && u < t);
    }
    mv.fwd_order()[rr] = t;
    mv.bwd_order()[rc] = t;
  }
  __syncthreads();
  MAP_STAMP(7);
  if (tid == 0) {
    int maxrow = 0;
    for (int t = 0; t < NT; ++t) maxrow = max(maxrow, rowlen[t]);
    ws[0] = kMapMagic;
    ws[1] = g.L;
    ws[2] = g.xb;
    ws[3] = g.B;
    ws[4] = g.NT;
    ws[5] = g.T0;
    ws[6] = mv.row_ptr()[NT];
    ws[7] = maxrow;
    ws[8] = g.S;
    ws[9] = seq;
  }
}

__global__ void __launch_bounds__(kBuildThreads, 1) build_map_kernel(Geom g, int* __restrict__ ws, int stage) {
  build_map_body(g, ws, 0, stage);
}

// Varlen: CTA i builds sequence i's map at ws + i * stride.
__global__ void __launch_bounds__(kBuildThreads, 1)
    build_map_varlen_kernel(const __grid_constant__ SeqLens lens, int* __restrict__ ws, long long stride, int stage) {
  build_map_body(seq_geom(lens, blockIdx.x), ws + blockIdx.x * stride, lens.seq[blockIdx.x], stage);
}

// Dynamic shared memory of the builder; the staged layout if it fits in 227 KB
// (varlen: sized for the longest sequence, whose map bounds every other one).
size_t build_smem(const Geom& g, int& stage) {
  const size_t base = (3 * (size_t)g.NT + kBuildThreads + (kBuildThreads / 32) * 512) * sizeof(int);
  const size_t staged = base + ((size_t)g.NT + 1 + (size_t)map_capacity(g)) * sizeof(int);
  stage = staged <= 227 * 1024 ? 1 : 0;
  return stage ? staged : base;
}

}  // namespace

int build_map_device(const Geom& g, int* ws, cudaStream_t stream) {
  int stage = 0;
  const size_t smem = build_smem(g, stage);
  if (g.NT > kMaxTiles) return set_error(BD_ERR_UNSUPPORTED, "too many tiles (%d > %d)", g.NT, kMaxTiles);
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(build_map_kernel), 227 * 1024,
                                "cudaFuncSetAttribute(build_map_kernel)"))
    return rc;
  build_map_kernel<<<1, kBuildThreads, smem, stream>>>(g, ws, stage);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "build_map_kernel launch");
}

int build_map_device_varlen(const Geom& gmax, const SeqLens& lens, int* ws, long long stride, cudaStream_t stream) {
  int stage = 0;
  const size_t smem = build_smem(gmax, stage);
  if (gmax.NT > kMaxTiles) return set_error(BD_ERR_UNSUPPORTED, "too many tiles (%d > %d)", gmax.NT, kMaxTiles);
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(build_map_varlen_kernel), 227 * 1024,
                                "cudaFuncSetAttribute(build_map_varlen_kernel)"))
    return rc;
  build_map_varlen_kernel<<<lens.n, kBuildThreads, smem, stream>>>(lens, ws, stride, stage);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "build_map_varlen_kernel launch");
}

}  // namespace bd

// ---------------------------------------------------------------- C ABI
extern "C" int bd_tilemap_dump(const bd_problem* prob, int32_t* host_out, size_t cap, int64_t* n_tiles) {
  using namespace bd;
  int rc = validate_problem(prob);
  if (rc) return rc;
  if (!host_out && cap) return set_error(BD_ERR_INVALID_ARG, "host_out is null");
  const Geom g = geom_of(*prob);
  std::vector<int> w;
  build_map_host(g, w);
  MapView mv{w.data(), g.NT, map_capacity(g)};
  const int n = mv.row_ptr()[g.NT];
  if (n_tiles) *n_tiles = n;
  if (cap < (size_t)n * 5) return set_error(BD_ERR_WORKSPACE, "capacity %zu < %d", cap, n * 5);
  size_t o = 0;
  for (int t = 0; t < g.NT; ++t)
    for (int e = mv.row_ptr()[t]; e < mv.row_ptr()[t + 1]; ++e) {
      const int kt = entry_tile(mv.row_ent()[e]);
      host_out[o++] = tile_seg(g, t);
      host_out[o++] = tile_idx(g, t);
      host_out[o++] = tile_seg(g, kt);
      host_out[o++] = tile_idx(g, kt);
      host_out[o++] = entry_kind(mv.row_ent()[e]);
    }
  return BD_OK;
}

extern "C" int bd_tilemap_stats(const bd_problem* prob, int64_t* out) {
  using namespace bd;
  int rc = validate_problem(prob);
  if (rc) return rc;
  if (!out) return set_error(BD_ERR_INVALID_ARG, "out is null");
  const Geom g = geom_of(*prob);
  std::vector<int> w;
  build_map_host(g, w);
  MapView mv{w.data(), g.NT, map_capacity(g)};
  int64_t full = 0, part = 0;
  for (int e = 0; e < mv.row_ptr()[g.NT]; ++e) (entry_kind(mv.row_ent()[e]) == kKindFull ? full : part)++;
  out[0] = g.NT;
  out[1] = full + part;
  out[2] = full;
  out[3] = part;
  return BD_OK;
}

extern "C" int64_t bd_tilemap_entries_bound(const bd_problem* prob) {
  using namespace bd;
  if (validate_problem(prob)) return -1;
  return map_entries_bound(geom_of(*prob));
}

// Copies the host-built workspace image of the map (tests compare it with the
// device-built one).  Not part of the public header's contract beyond tests.
extern "C" int bd_tilemap_host_image(const bd_problem* prob, int32_t* host_out, size_t cap_words,
                                     int64_t* n_words) {
  using namespace bd;
  int rc = validate_problem(prob);
  if (rc) return rc;
  const Geom g = geom_of(*prob);
  std::vector<int> w;
  build_map_host(g, w);
  if (n_words) *n_words = (int64_t)w.size();
  if (!host_out || cap_words < w.size()) return set_error(BD_ERR_WORKSPACE, "capacity too small");
  std::copy(w.begin(), w.end(), host_out);
  return BD_OK;
}

// Consistency of the two interval views used by the kernels (host, tests):
// key k is in row r's interval (row_interval) iff row r is in key k's
// interval (key_interval), for every packed (row, key).  Returns the number of
// mismatches in *mismatches.
extern "C" int bd_tilemap_selfcheck(const bd_problem* prob, int64_t* mismatches) {
  using namespace bd;
  int rc = validate_problem(prob);
  if (rc) return rc;
  if (!mismatches) return set_error(BD_ERR_INVALID_ARG, "mismatches is null");
  const Geom g = geom_of(*prob);
  if ((int64_t)g.N * g.N > (int64_t)1 << 26) return set_error(BD_ERR_UNSUPPORTED, "problem too large for selfcheck");
  int64_t bad = 0;
  for (int r = 0; r < g.N; ++r) {
    const int qs = seg_of_row(g, r);
    for (int k = 0; k < g.N; ++k) {
      const int ks = seg_of_row(g, k);
      int lo, hi, qa, qb;
      row_interval(g, qs, r, ks, lo, hi);
      key_interval(g, ks, k, qs, qa, qb);
      const bool a = k >= lo && k < hi;
      const bool b = r >= qa && r < qb;
      bad += (a != b);
    }
  }
  *mismatches = bad;
  return BD_OK;
}

// Element-level mask the kernels evaluate (host, tests): for rows
// [row0, row0 + n_rows) of sequence `seq`, every packed key of that sequence,
// bit 0 = key inside the row's interval (row_interval: forward and dQ
// kernels), bit 1 = row inside the key's interval (key_interval: dK/dV
// kernel).  Tests compare both bits with the oracle's dense mask.
extern "C" int bd_mask_dump(const bd_problem* prob, int32_t seq, int64_t row0, int64_t n_rows, uint8_t* host_out,
                            size_t cap, int64_t* n_keys) {
  using namespace bd;
  int rc = validate_problem(prob);
  if (rc) return rc;
  if (seq < 0 || seq >= prob->batch) return set_error(BD_ERR_INVALID_ARG, "sequence %d out of range", seq);
  Geom g = geom_of(*prob);
  if (is_varlen(*prob)) {
    const int P = prob->seq_prompt_len[seq], R = prob->seq_response_len[seq];
    g = make_geom(P + R, prob->repeat_prompt ? 0 : P, prob->block_size, prob->n_copies);
  }
  if (n_keys) *n_keys = g.N;
  if (row0 < 0 || n_rows < 0 || row0 + n_rows > g.N) return set_error(BD_ERR_INVALID_ARG, "row range outside [0, %d)", g.N);
  if (cap < (size_t)n_rows * g.N) return set_error(BD_ERR_WORKSPACE, "capacity %zu < %lld", cap, (long long)n_rows * g.N);
  if (!host_out && n_rows) return set_error(BD_ERR_INVALID_ARG, "host_out is null");
  for (int64_t i = 0; i < n_rows; ++i) {
    const int r = (int)(row0 + i);
    const int qs = seg_of_row(g, r);
    int lo[64], hi[64];
    const int nseg = 1 + g.S;
    if (nseg > 64) return set_error(BD_ERR_UNSUPPORTED, "too many copies for the dump");
    for (int s = 0; s < nseg; ++s) row_interval(g, qs, r, s, lo[s], hi[s]);
    uint8_t* o = host_out + i * g.N;
    for (int k = 0; k < g.N; ++k) {
      const int ks = seg_of_row(g, k);
      int qa, qb;
      key_interval(g, ks, k, qs, qa, qb);
      o[k] = (uint8_t)((k >= lo[ks] && k < hi[ks]) | ((r >= qa && r < qb) << 1));
    }
  }
  return BD_OK;
}

#if BD_MAP_TRACE
extern "C" int bd_debug_map_trace(int64_t* host_out, int n) {
  if (!host_out || n <= 0 || n > 16) return BD_ERR_INVALID_ARG;
  return bd::check_cuda(cudaMemcpyFromSymbol(host_out, bd::g_map_trace, n * sizeof(long long)), "map trace copy");
}
#endif
