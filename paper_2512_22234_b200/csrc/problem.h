// Validation of bd_problem and derived geometry (host).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "abi_common.h"
#include "tilemap.cuh"

namespace bd {

constexpr int kMaxTiles = 8192;  // NT bound of the device map builder (L <= ~512K)

inline int validate_problem(const bd_problem* p) {
  if (!p) return set_error(BD_ERR_INVALID_ARG, "problem is null");
  if (p->batch <= 0 || p->block_size <= 0 || p->n_q_heads <= 0 || p->n_kv_heads <= 0 || p->head_dim <= 0)
    return set_error(BD_ERR_INVALID_ARG, "non-positive dimension");
  if (p->prompt_len < 0 || p->response_len < 0)
    return set_error(BD_ERR_INVALID_ARG, "negative length");
  const int64_t L = (int64_t)p->prompt_len + p->response_len;
  if (L <= 0) return set_error(BD_ERR_INVALID_ARG, "empty sequence");
  if (p->n_q_heads % p->n_kv_heads) return set_error(BD_ERR_INVALID_ARG, "n_q_heads %% n_kv_heads != 0");
  if (L % p->block_size) return set_error(BD_ERR_LAYOUT, "L = %lld not a multiple of block_size %d", (long long)L,
                                          p->block_size);
  if (p->repeat_prompt != 0 && p->repeat_prompt != 1) return set_error(BD_ERR_INVALID_ARG, "repeat_prompt not 0/1");
  if (p->n_copies < 0) return set_error(BD_ERR_INVALID_ARG, "n_copies < 0");
  const int64_t S = p->n_copies > 1 ? p->n_copies : 1;
  const int64_t Lx = L - (p->repeat_prompt ? 0 : p->prompt_len);
  if (L + S * Lx > (int64_t)1 << 30) return set_error(BD_ERR_UNSUPPORTED, "sequence too long");
  const int64_t NT = (L + kTileRows - 1) / kTileRows + S * ((Lx + kTileRows - 1) / kTileRows);
  if (NT > kMaxTiles) return set_error(BD_ERR_UNSUPPORTED, "sequence too long for the tile map (%lld tiles)",
                                       (long long)NT);
  if (p->q_row_heads < 0 || p->kv_row_heads < 0 || (p->q_row_heads && p->q_row_heads < p->n_q_heads) ||
      (p->kv_row_heads && p->kv_row_heads < p->n_kv_heads))
    return set_error(BD_ERR_INVALID_ARG, "row heads (%d, %d) below (n_q_heads, n_kv_heads) = (%d, %d)", p->q_row_heads,
                     p->kv_row_heads, p->n_q_heads, p->n_kv_heads);
  if ((p->seq_prompt_len == nullptr) != (p->seq_response_len == nullptr))
    return set_error(BD_ERR_INVALID_ARG, "seq_prompt_len and seq_response_len must both be set or both null");
  if (p->seq_prompt_len) {
    if (p->batch > kMaxVarlenSeqs)
      return set_error(BD_ERR_UNSUPPORTED, "varlen batch %d > %d sequences", p->batch, kMaxVarlenSeqs);
    for (int i = 0; i < p->batch; ++i) {
      const int Pi = p->seq_prompt_len[i], Ri = p->seq_response_len[i];
      if (Pi < 0 || Ri < 0 || Pi > p->prompt_len || Ri > p->response_len)
        return set_error(BD_ERR_INVALID_ARG, "sequence %d: lengths (%d, %d) outside [0, (%d, %d)]", i, Pi, Ri,
                         p->prompt_len, p->response_len);
      if (Pi + Ri <= 0) return set_error(BD_ERR_INVALID_ARG, "sequence %d is empty", i);
      if ((Pi + Ri) % p->block_size)
        return set_error(BD_ERR_LAYOUT, "sequence %d: L = %d not a multiple of block_size %d", i, Pi + Ri,
                         p->block_size);
    }
  }
  return BD_OK;
}

inline Geom geom_of(const bd_problem& p) {
  const int L = p.prompt_len + p.response_len;
  return make_geom(L, p.repeat_prompt ? 0 : p.prompt_len, p.block_size, p.n_copies);
}

inline bool is_varlen(const bd_problem& p) { return p.seq_prompt_len != nullptr; }

inline SeqLens seq_lens_of(const bd_problem& p) {
  SeqLens s;
  s.n = p.batch;
  s.repeat_prompt = p.repeat_prompt;
  s.B = p.block_size;
  s.S = p.n_copies > 1 ? p.n_copies : 1;
  for (int i = 0; i < p.batch; ++i) s.seq[i] = i;
  // longest first (stable), see tilemap.cuh SeqLens
  std::stable_sort(s.seq, s.seq + p.batch, [&](int a, int b) {
    return p.seq_prompt_len[a] + p.seq_response_len[a] > p.seq_prompt_len[b] + p.seq_response_len[b];
  });
  for (int i = 0; i < p.batch; ++i) {
    s.P[i] = p.seq_prompt_len[s.seq[i]];
    s.R[i] = p.seq_response_len[s.seq[i]];
  }
  return s;
}

// Heads per token row in memory (head sharding; 0 = dense).
inline int q_row_heads(const bd_problem& p) { return p.q_row_heads ? p.q_row_heads : p.n_q_heads; }
inline int kv_row_heads(const bd_problem& p) { return p.kv_row_heads ? p.kv_row_heads : p.n_kv_heads; }

inline float scale_of(const bd_problem& p) {
  return p.softmax_scale > 0.f ? p.softmax_scale : 1.0f / std::sqrt((float)p.head_dim);
}

}  // namespace bd
