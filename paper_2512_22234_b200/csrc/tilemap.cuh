// Block-diffusion mask -> 128x128 tile map (block-sparse schedule).
//
// The mask rule (Eq. 2; Fig. 4b) makes every
// query row's visible keys, per key segment, ONE contiguous packed interval:
//   x0 row at clean position p, bq = p / B:
//       x0 keys [0, min((bq+1)B, L))                (block-causal)
//   xt row at clean position p:
//       x0 keys [0, bq B)                            (clean blocks < bq)
//       xt keys clean positions [max(bq B, xb), min((bq+1)B, L))   (own block)
// Both ends are non-decreasing in p.  The builder below classifies every
// (q-tile, k-tile) pair from these intervals (FULL / PARTIAL / EMPTY), and
// the kernels evaluate the same intervals per row on PARTIAL tiles.  EMPTY
// tiles are never listed, hence never loaded.
//
// One __host__ __device__ implementation serves the device builder kernel
// (bd_attn_fwd/bwd build the map into the caller's workspace every call) and
// the host path (bd_tilemap_dump / bd_tilemap_stats).
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace bd {

constexpr int kTileRows = 128;
constexpr int kKindFull = 1;
constexpr int kKindPartial = 2;

struct Geom {
  int L, xb, N, B, T0, T1, NT;
  int S;   // noisy copies (trace replay, reading c19); 1 = DiRL single copy
  int Lx;  // L - xb: length of one noisy copy
};

__host__ __device__ inline Geom make_geom(int L, int xb, int B, int S = 1) {
  Geom g;
  g.L = L;
  g.xb = xb;
  g.S = S < 1 ? 1 : S;
  g.Lx = L - xb;
  g.N = L + g.S * g.Lx;
  g.B = B;
  g.T0 = (L + kTileRows - 1) / kTileRows;
  g.T1 = (g.Lx + kTileRows - 1) / kTileRows;
  g.NT = g.T0 + g.S * g.T1;
  return g;
}

// Segments: 0 = x0 (packed [0, L)), s = 1..S noisy copy s (packed
// [L + (s-1) Lx, L + s Lx)).  Each segment is tiled from its own start.
__host__ __device__ inline int seg_base(const Geom& g, int s) { return s ? g.L + (s - 1) * g.Lx : 0; }
__host__ __device__ inline int seg_end(const Geom& g, int s) { return s ? g.L + s * g.Lx : g.L; }
// (S == 1, the hot path, avoids the integer divisions: the kernels evaluate
// these per tile in their inner loops.)
__host__ __device__ inline int seg_of_row(const Geom& g, int n) {
  return n < g.L ? 0 : (g.S == 1 ? 1 : 1 + (n - g.L) / g.Lx);
}
__host__ __device__ inline int seg_first_tile(const Geom& g, int s) { return s ? g.T0 + (s - 1) * g.T1 : 0; }
__host__ __device__ inline int tile_seg(const Geom& g, int t) {
  return t < g.T0 ? 0 : (g.S == 1 ? 1 : 1 + (t - g.T0) / g.T1);
}
__host__ __device__ inline int tile_idx(const Geom& g, int t) {
  return t < g.T0 ? t : (g.S == 1 ? t - g.T0 : (t - g.T0) % g.T1);
}
// [start, end) and segment of tile t with at most one division
__host__ __device__ inline void tile_bounds(const Geom& g, int t, int& start, int& end, int& seg) {
  if (t < g.T0) {
    seg = 0;
    start = t * kTileRows;
    end = start + kTileRows < g.L ? start + kTileRows : g.L;
    return;
  }
  const int j = t - g.T0;
  const int s = g.S == 1 ? 0 : j / g.T1;
  const int base = g.L + s * g.Lx;
  seg = s + 1;
  start = base + (j - s * g.T1) * kTileRows;
  end = start + kTileRows < base + g.Lx ? start + kTileRows : base + g.Lx;
}
__host__ __device__ inline int tile_start(const Geom& g, int t) {
  int a, b, s;
  tile_bounds(g, t, a, b, s);
  return a;
}
__host__ __device__ inline int tile_end(const Geom& g, int t) {
  int a, b, s;
  tile_bounds(g, t, a, b, s);
  return b;
}
// q-tile holding packed row n
__host__ __device__ inline int tile_of_row(const Geom& g, int n) {
  if (n < g.L) return n / kTileRows;
  const int j = n - g.L, s = g.S == 1 ? 0 : j / g.Lx;
  return g.T0 + s * g.T1 + (j - s * g.Lx) / kTileRows;
}

// Visible packed-column interval [lo, hi) of packed row `row` (a row of
// segment `qseg`) within key segment `kseg`.  Empty intervals have lo >= hi.
// A noisy row sees no other copy (reading c19), so for kseg >= 1 only
// kseg == qseg is non-empty.
__host__ __device__ inline void row_interval(const Geom& g, int qseg, int row, int kseg, int& lo, int& hi) {
  const int p = qseg ? g.xb + (row - seg_base(g, qseg)) : row;  // clean position
  const int bq = p / g.B;
  const int b0 = bq * g.B, b1 = b0 + g.B;
  if (kseg == 0) {
    lo = 0;
    hi = qseg ? b0 : (b1 < g.L ? b1 : g.L);
  } else if (qseg != kseg) {
    lo = hi = seg_base(g, kseg);  // x0 never sees xt; copies never see each other
  } else {
    const int a = b0 > g.xb ? b0 : g.xb;
    const int c = b1 < g.L ? b1 : g.L;
    lo = seg_base(g, kseg) + a - g.xb;
    hi = seg_base(g, kseg) + c - g.xb;
  }
}

// The transpose view used by the backward's key-row threads: the packed query
// rows of segment `qseg` that see key `key` (a packed row of segment kseg)
// also form one interval [qa, qb) (row intervals are monotone in the row):
//   x0 key, x0 rows:        blk(q) >= blk(k)      -> [blk(k) B, L)
//   x0 key, copy-s rows:    blk(q) >= blk(k) + 1  -> clean positions >= (blk(k)+1) B
//   copy-s key, copy-s rows: blk(q) == blk(k)     -> its own block (clipped to xb)
//   xt key, x0 rows / another copy's rows: never
__host__ __device__ inline void key_interval(const Geom& g, int kseg, int key, int qseg, int& qa, int& qb) {
  const int pk = kseg ? g.xb + (key - seg_base(g, kseg)) : key;
  const int bk = pk / g.B;
  if (qseg == 0) {
    if (kseg) {
      qa = qb = 0;
    } else {
      qa = bk * g.B;
      qb = g.L;
    }
  } else if (kseg && kseg != qseg) {
    qa = qb = seg_base(g, qseg);
  } else {
    int a, b;  // clean positions
    if (kseg == 0) {
      a = (bk + 1) * g.B;
      b = g.L;
    } else {
      a = bk * g.B;
      b = (bk + 1) * g.B < g.L ? (bk + 1) * g.B : g.L;
    }
    if (a < g.xb) a = g.xb;
    qa = seg_base(g, qseg) + a - g.xb;
    qb = seg_base(g, qseg) + b - g.xb;
    if (qb < qa) qb = qa;
  }
}

// Kind of tile pair (qt, kt): 0 = EMPTY, kKindFull, kKindPartial -- decided
// over the tile's valid rows and columns, row by row.
__host__ __device__ inline int classify_pair(const Geom& g, int qt, int kt) {
  const int q0 = tile_start(g, qt), q1 = tile_end(g, qt), qs = tile_seg(g, qt);
  const int k0 = tile_start(g, kt), k1 = tile_end(g, kt), ks = tile_seg(g, kt);
  bool any = false, all = true;
  for (int r = q0; r < q1; ++r) {
    int lo, hi;
    row_interval(g, qs, r, ks, lo, hi);
    const int a = lo > k0 ? lo : k0;
    const int b = hi < k1 ? hi : k1;
    if (b > a) any = true;
    if (!(a == k0 && b == k1)) all = false;
  }
  return any ? (all ? kKindFull : kKindPartial) : 0;
}

// Candidate k-tiles of q-tile qt: the union of its rows' intervals is
// [0, hi0) in x0 and [lo1, hi1) in its own copy (intervals are monotone and
// the xt ones of consecutive blocks are adjacent), so only tiles overlapping
// those ranges are classified.
__host__ __device__ inline void candidate_range(const Geom& g, int qt, int kseg, int& t_lo, int& t_hi) {
  const int q0 = tile_start(g, qt), q1 = tile_end(g, qt), qs = tile_seg(g, qt);
  int lo_a, hi_a, lo_b, hi_b;
  row_interval(g, qs, q0, kseg, lo_a, hi_a);
  row_interval(g, qs, q1 - 1, kseg, lo_b, hi_b);
  const int lo = lo_a, hi = hi_b;
  const int base = seg_first_tile(g, kseg);
  const int seg0 = seg_base(g, kseg);
  if (hi <= lo) {
    t_lo = t_hi = base;
    return;
  }
  t_lo = base + (lo - seg0) / kTileRows;
  t_hi = base + (hi - seg0 + kTileRows - 1) / kTileRows;
}

// Entries are int32: k-tile index | kind << 28.
__host__ __device__ inline int entry_make(int tile, int kind) { return tile | (kind << 28); }
__host__ __device__ inline int entry_tile(int e) { return e & 0x0FFFFFFF; }
__host__ __device__ inline int entry_kind(int e) { return (e >> 28) & 0xF; }

// Workspace image of the map (int32 words):
//   [0]            magic
//   [1..8]         L, xb, B, NT, T0, n_entries, max_row_len, S
//   row_ptr[NT+1]  entries of q-tile t are row_ent[row_ptr[t] .. row_ptr[t+1])
//   row_ent[cap]   k-tiles in increasing order
//   col_ptr[NT+1]  column CSR (q-tiles visiting k-tile t), for the backward
//   col_ent[cap]   q-tile | kind << 28, q-tiles in increasing order
//   fwd_order[NT]  q-tiles by decreasing row length (longest first, LPT)
//   bwd_order[NT]  k-tiles by decreasing column length
//   col_rpos[cap]  for column entry c (of q-tile t, k-tile kt): the index e of
//                  kt in the ROW CSR (row_ent[e]) -- where the dK/dV kernel
//                  stores that tile's dS^T so the dQ kernel reads its row's
//                  tiles contiguously
constexpr int kMapMagic = 0x42444D31;  // "BDM1"
constexpr int kMapHeader = 16;  // [8] = S (noisy copies); [9] = sequence (varlen); [10..15] reserved

struct MapView {
  int* base;
  int NT, cap;
  __host__ __device__ int* row_ptr() const { return base + kMapHeader; }
  __host__ __device__ int* row_ent() const { return row_ptr() + NT + 1; }
  __host__ __device__ int* col_ptr() const { return row_ent() + cap; }
  __host__ __device__ int* col_ent() const { return col_ptr() + NT + 1; }
  __host__ __device__ int* fwd_order() const { return col_ent() + cap; }
  __host__ __device__ int* bwd_order() const { return fwd_order() + NT; }
  __host__ __device__ int* col_rpos() const { return bwd_order() + NT; }
};

// Upper bound on entries: a q-tile lists at most T0 x0 tiles and xt_max tiles
// of its own copy.  Its rows' own-copy intervals union to [blockstart(p0),
// blockend(p0 + 127)), at most 126 + 2B keys at any offset -- blocks need not
// be tile-aligned (B not dividing 128, or xb % B != 0 in response-only mode) --
// so at most ceil((126 + 2B) / 128) + 1 tiles.  The device builder also uses
// capacity / NT as the per-q-tile stride of its staged entries.
__host__ __device__ inline int map_capacity(const Geom& g) {
  const int xt_max = (2 * g.B + 126 + kTileRows - 1) / kTileRows + 1;
  return g.NT * (g.T0 + (xt_max < g.T1 ? xt_max : g.T1));
}
__host__ __device__ inline long long map_words(const Geom& g) {
  return (long long)kMapHeader + 2LL * (g.NT + 1) + 3LL * map_capacity(g) + 2LL * g.NT;
}

// Number of listed (q-tile, k-tile) pairs, from the candidate ranges alone
// (O(NT), host side): every candidate tile is non-empty -- a row's x0
// interval starts at key 0 and the own-copy intervals of a tile's rows are
// whole adjacent blocks, so the union over the tile's rows is one interval
// per segment and each tile overlapping it holds a key some row sees -- so
// this equals the builder's n_entries; it is used as an upper bound (the
// per-(sequence, head) stride of the stored dS^T tiles) either way.
__host__ __device__ inline long long map_entries_bound(const Geom& g) {
  long long n = 0;
  for (int t = 0; t < g.NT; ++t) {
    const int qs = tile_seg(g, t);
    for (int kk = 0; kk < (qs ? 2 : 1); ++kk) {
      int a, b;
      candidate_range(g, t, kk ? qs : 0, a, b);
      n += b - a;
    }
  }
  return n;
}

// Geometry of the sequence whose map starts at `base` (varlen batches keep
// one map per sequence; the kernels read their sequence's geometry from it).
__host__ __device__ inline Geom map_geom(const int* base) { return make_geom(base[1], base[2], base[3], base[8]); }
__host__ __device__ inline int map_seq(const int* base) { return base[9]; }

// Per-sequence lengths of a varlen batch, passed by
// value to the map builder (kernel parameter: no host->device copy, no sync).
// Entry i describes sequence seq[i]; the host lists the sequences longest
// first, and map i is built for entry i, so the (sequence, kv head)-major
// grid of the attention kernels starts the long sequences first (LPT across
// the batch) while keeping each sequence's CTAs together (L2 reuse).
constexpr int kMaxVarlenSeqs = 1024;
struct SeqLens {
  int n, repeat_prompt, B, S;
  int seq[kMaxVarlenSeqs];
  int P[kMaxVarlenSeqs];
  int R[kMaxVarlenSeqs];
};
__host__ __device__ inline Geom seq_geom(const SeqLens& s, int i) {
  const int L = s.P[i] + s.R[i];
  return make_geom(L, s.repeat_prompt ? 0 : s.P[i], s.B, s.S);
}

}  // namespace bd
