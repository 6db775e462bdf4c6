// C ABI of the attention path: validation, workspace carving, launches.
#include "abi_common.h"
#include "problem.h"
#include "attn_common.h"

namespace bd {
namespace {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
  size_t map_off, dsum_off, ds_off, ds_bytes, total;
  int map_stride;  // words between per-sequence maps (varlen), 0 = one map
  long long ds_stride;
  int ds_chunk;
};

WsLayout ws_layout(const bd_problem& p, int backward) {
  const Geom g = geom_of(p);
  WsLayout w{};
  w.map_off = 0;
  const size_t one = (size_t)map_words(g);
  w.map_stride = is_varlen(p) ? (int)((one + 63) & ~size_t(63)) : 0;
  size_t off = align256((is_varlen(p) ? (size_t)w.map_stride * p.batch : one) * sizeof(int));
  if (backward) {
    w.dsum_off = off;  // tile-major log2-LSE and D vectors (dQ accumulates in TMEM)
    off = align256(off + bwd_vec_floats(p, g) * sizeof(float));
    w.ds_bytes = ds_plan_bytes(p, g, &w.ds_stride, &w.ds_chunk);  // stored dS^T tiles (one chunk)
    w.ds_off = off;
    off = align256(off + w.ds_bytes);
  }
  w.total = off;
  return w;
}

int build_maps(const bd_problem& p, const Geom& g, const WsLayout& wl, int* map, cudaStream_t stream) {
  if (!is_varlen(p)) return build_map_device(g, map, stream);
  const SeqLens lens = seq_lens_of(p);
  return build_map_device_varlen(g, lens, map, wl.map_stride, stream);
}

int check_ptrs(std::initializer_list<const void*> ps) {
  for (const void* x : ps) {
    if (!x) return set_error(BD_ERR_INVALID_ARG, "null tensor pointer");
    if (!aligned16(x)) return set_error(BD_ERR_ALIGNMENT, "tensor pointer not 16-byte aligned");
  }
  return BD_OK;
}

int check_head_dim(const bd_problem& p) {
  if (p.head_dim != 64 && p.head_dim != 128)
    return set_error(BD_ERR_UNSUPPORTED, "head_dim %d not in {64, 128}", p.head_dim);
  return BD_OK;
}

}  // namespace
}  // namespace bd

extern "C" int64_t bd_packed_len(const bd_problem* prob) {
  if (bd::validate_problem(prob)) return -1;
  return bd::geom_of(*prob).N;
}

extern "C" size_t bd_attn_workspace_bytes(const bd_problem* prob, int backward) {
  if (bd::validate_problem(prob)) return 0;
  return bd::ws_layout(*prob, backward).total;
}

extern "C" int bd_attn_fwd(const bd_problem* prob, const void* q, const void* k, const void* v, void* o, float* lse,
                           void* ws, size_t ws_bytes, void* stream_) {
  using namespace bd;
  int rc = validate_problem(prob);
  if (rc) return rc;
  if ((rc = check_head_dim(*prob))) return rc;
  if ((rc = check_ptrs({q, k, v, o, lse, ws}))) return rc;
  const WsLayout wl = ws_layout(*prob, 0);
  if (ws_bytes < wl.total) return set_error(BD_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, wl.total);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const Geom g = geom_of(*prob);
  int* map = reinterpret_cast<int*>(static_cast<char*>(ws) + wl.map_off);
  if ((rc = build_maps(*prob, g, wl, map, stream))) return rc;
  return run_attn_fwd(*prob, g, q, k, v, o, lse, map, wl.map_stride, stream);
}

extern "C" int bd_attn_bwd(const bd_problem* prob, const void* q, const void* k, const void* v, const void* o,
                           const float* lse, const void* dout, void* dq, void* dk, void* dv, void* ws,
                           size_t ws_bytes, void* stream_) {
  using namespace bd;
  int rc = validate_problem(prob);
  if (rc) return rc;
  if ((rc = check_head_dim(*prob))) return rc;
  if ((rc = check_ptrs({q, k, v, o, lse, dout, dq, dk, dv, ws}))) return rc;
  const WsLayout wl = ws_layout(*prob, 1);
  if (ws_bytes < wl.total) return set_error(BD_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, wl.total);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const Geom g = geom_of(*prob);
  char* w = static_cast<char*>(ws);
  int* map = reinterpret_cast<int*>(w + wl.map_off);
  if ((rc = build_maps(*prob, g, wl, map, stream))) return rc;
  DsPlan ds;
  if (wl.ds_bytes) {
    ds.buf = w + wl.ds_off;
    ds.stride = wl.ds_stride;
    ds.chunk = wl.ds_chunk;
  }
  return run_attn_bwd(*prob, g, q, k, v, o, lse, dout, dq, dk, dv, map, wl.map_stride,
                      reinterpret_cast<float*>(w + wl.dsum_off), ds, stream);
}
