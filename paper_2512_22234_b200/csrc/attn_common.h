// Shared host helpers for the attention kernels.
#pragma once
#include <cuda_runtime.h>

#include "tma_host.h"
#include "tilemap.cuh"
#include "bd_attn.h"

namespace bd {

// 4-D TMA map over a [b, N, H, D] bf16 tensor whose token rows hold
// row_heads >= H heads in memory (head sharding; 0 = H): dims (D, H, N, b),
// box (64, 1, 128, 1), 128-byte swizzle.  Rows past N are zero-filled.
inline bool make_qkv_tmap(CUtensorMap* m, const void* base, int batch, int N, int H, int D, int box_rows = 128,
                          int row_heads = 0) {
  const uint64_t RH = row_heads > 0 ? (uint64_t)row_heads : (uint64_t)H;
  const uint64_t dims[4] = {(uint64_t)D, (uint64_t)H, (uint64_t)N, (uint64_t)batch};
  const uint64_t strides[3] = {(uint64_t)D * 2, RH * D * 2, (uint64_t)N * RH * D * 2};
  const uint32_t box[4] = {64, 1, (uint32_t)box_rows, 1};
  return make_tmap_bf16(m, base, 4, dims, strides, box);
}

int build_map_device(const Geom& g, int* ws, cudaStream_t stream);
int build_map_device_varlen(const Geom& gmax, const SeqLens& lens, int* ws, long long stride, cudaStream_t stream);
// map_stride: words between consecutive sequences' maps (0 = one shared map)
int run_attn_fwd(const bd_problem& p, const Geom& g, const void* q, const void* k, const void* v, void* o,
                 float* lse, const int* map, int map_stride, cudaStream_t stream);
// Stored-dS backward (uniform batches): the dK/dV kernel writes every
// visible tile's dS^T (bf16, 32 KB) into `buf`, `stride` tiles per (sequence,
// q-head) (map_entries_bound), and the dQ kernel reads it back -- in chunks of
// `chunk` sequences, `buf` holding one chunk.  buf == nullptr: the dQ kernel
// recomputes S and dP (varlen batches, or when disabled / over budget).
struct DsPlan {
  void* buf = nullptr;
  long long stride = 0;
  int chunk = 0;
};
// The plan's sizes for a problem (host, deterministic): bytes of the dS^T
// buffer (0 = path off).  BD_BWD_DS unset: on when the whole batch fits one
// chunk of BD_BWD_DS_BUDGET_MB (default 8,192); BD_BWD_DS=1: on, chunked
// (floor(budget / per sequence) sequences per chunk, default budget 24,576;
// off if one sequence exceeds it); BD_BWD_DS=0: off.  The environment is
// read per call: keep it fixed between the workspace query and the call.
size_t ds_plan_bytes(const bd_problem& p, const Geom& g, long long* stride, int* chunk);
int run_attn_bwd(const bd_problem& p, const Geom& g, const void* q, const void* k, const void* v, const void* o,
                 const float* lse, const void* dout, void* dq, void* dk, void* dv, const int* map, int map_stride,
                 float* vec_ws, const DsPlan& ds, cudaStream_t stream);
size_t bwd_vec_floats(const bd_problem& p, const Geom& g);

}  // namespace bd
