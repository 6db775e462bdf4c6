/* bd_attn.h -- C ABI of the B200 (sm_100a) block-diffusion training hot path
 * of DiRL / DiPO (arXiv 2512.22234).
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 *
 * The hot path:
 *   bd_attn_fwd   -- masked attention over the packed [x0 | xt] sequence with
 *                    the block-diffusion mask (Eq. 2, Fig. 4,
 *                    P:261 "repeats both parts blockwise"), fp32 LSE out.
 *   bd_attn_bwd   -- dQ / dK / dV of the same op, reusing the tile map.
 *   bd_logprob    -- per-token log-softmax gather (numerators of Eqs. 6-8,
 *                    P:150-156; CE of Eq. 3), optionally fused with its
 *                    gradient.
 *   bd_dipo_*     -- DiPO advantage / token-level reduction at the
 *                    stop-gradient behaviour policy (P:92, P:172-174,
 *                    P:179-225); the only cross-GPU step is a NCCL all-reduce
 *                    of its scalar partials, done by the caller.
 *
 * General conventions
 *  - Every pointer argument is a DEVICE pointer unless marked "host".  The
 *    library allocates nothing: the caller owns every buffer, including the
 *    workspace.  Work is enqueued asynchronously on `stream` (a cudaStream_t;
 *    NULL = legacy default stream).
 *  - Return value: BD_OK (0) or one of the BD_ERR_* codes below; no
 *    exception ever crosses the ABI.  bd_error_string() names a code,
 *    bd_last_error() returns a thread-local message for the last failure.
 *  - Tensors are dense row-major (C order) with the stated shapes.
 *  - Device pointers passed to TMA-loaded tensors must be 16-byte aligned.
 */
#ifndef BD_ATTN_H_
#define BD_ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BD_OK = 0,
  BD_ERR_INVALID_ARG = 1, /* null pointer, non-positive dimension, Hq % Hkv != 0 */
  BD_ERR_LAYOUT = 2,      /* L % block_size != 0 ("length not multiple of B -> layout error") */
  BD_ERR_UNSUPPORTED = 3, /* head_dim not in {64, 128}, sizes beyond int32 tile indexing */
  BD_ERR_ALIGNMENT = 4,   /* device pointer not 16-byte aligned */
  BD_ERR_WORKSPACE = 5,   /* workspace null or smaller than bd_attn_workspace_bytes() */
  BD_ERR_CUDA = 6         /* a CUDA runtime/driver call failed (see bd_last_error) */
};

/* One block-diffusion attention problem.  Fields follow the paper's statement
 * of the problem: prompt ("input") length P, response ("output") length R,
 * block size B ("each block contains B tokens", "input length
 * 1024 and output length 8192"), GQA heads and head_dim.
 *
 * Packed sequence (reading c1): per sequence the token axis holds
 * Ntot = L + (L - xb) rows, L = P + R:
 *     rows [0, L)       x0: clean copy of clean positions 0..L-1
 *     rows [L, Ntot)    xt: noisy copy of clean positions xb..L-1
 * with xb = 0 if repeat_prompt (DiRL, Fig. 4b; the default) and
 * xb = P otherwise (TraceRL, Fig. 4a).  Noisy rows keep their clean
 * position ids (RoPE is the caller's).
 *
 * Visibility (blk(p) = p / B):  x0->x0 blk(k) <= blk(q);  xt->x0 blk(k) <
 * blk(q);  xt->xt blk(k) == blk(q);  x0->xt never.                         */
typedef struct bd_problem {
  int32_t batch;
  int32_t prompt_len;    /* P >= 0                                     */
  int32_t response_len;  /* R >= 0, L = P + R > 0, L % block_size == 0 */
  int32_t block_size;    /* B >= 1                                     */
  int32_t n_q_heads;     /* Hq                                         */
  int32_t n_kv_heads;    /* Hkv, Hq % Hkv == 0; kv(h) = h / (Hq/Hkv)   */
  int32_t head_dim;      /* d in {64, 128}                             */
  int32_t repeat_prompt; /* 1 = DiRL (default), 0 = response-only       */
  float softmax_scale;   /* <= 0 -> 1/sqrt(head_dim)            */
  int32_t n_copies;      /* S noisy copies, 0 or 1 = single copy; S > 1 =
                          * trace replay (Eq. 6):
                          * packed [x0 | xt(1) | ... | xt(S)], copy s = every
                          * block's state before decoding step s; copy s of
                          * block k sees x0 blocks < k and itself only
                          * (reading c19)                      */
  /* Varlen batch (RL responses vary in length, P:331,
   * P:382): optional HOST arrays of `batch` per-sequence prompt / response
   * lengths (both NULL = every sequence has prompt_len / response_len).
   * Sequence i then has L_i = P_i + R_i (L_i % block_size == 0, 0 <= P_i <=
   * prompt_len, 0 <= R_i <= response_len) and packed length
   * N_i = L_i + S (L_i - xb_i) <= Ntot; tensors keep the padded [b, Ntot, H, d]
   * layout and rows n >= N_i of sequence i are neither read for any output
   * nor written (q/k/v/o/lse/dO there may hold anything; O/LSE/dQ/dK/dV there
   * are left untouched).  The arrays are read during the call only (copied
   * into a kernel parameter, no host->device transfer); batch <= 1024.     */
  const int32_t* seq_prompt_len;
  const int32_t* seq_response_len;
  /* Head sharding ((sequence, kv-head-group) units when there
   * are fewer sequences than GPUs; north star "sequences and heads are
   * partitioned"): the number of heads per token row IN MEMORY of the
   * q / o / dout / dq tensors (q_row_heads) and of the k / v / dk / dv tensors
   * (kv_row_heads); 0 = dense (n_q_heads / n_kv_heads).  A rank that owns kv
   * heads [g0, g0 + n_kv_heads) of a model with Hkv_total kv heads passes
   * k + g0 d, v + g0 d, ... and q + g0 (Hq/Hkv) d, ... with kv_row_heads =
   * Hkv_total, q_row_heads = Hq_total: no copies.  Must be >= n_q_heads /
   * n_kv_heads.  LSE stays a dense [b, n_q_heads, Ntot] buffer of the local
   * heads.                                                                */
  int32_t q_row_heads;
  int32_t kv_row_heads;
} bd_problem;

/* Packed length Ntot of one sequence, or -1 if the problem is invalid. */
int64_t bd_packed_len(const bd_problem* prob);

/* Workspace bytes needed by bd_attn_fwd (backward = 0) or bd_attn_bwd
 * (backward = 1).  The forward workspace holds the tile map; the backward
 * one additionally holds D = rowsum(dO * O) and the log2-scaled LSE, fp32,
 * tile-major [b, Hq, n_tiles, 128], and -- for uniform (non-varlen) batches
 * -- the stored-dS buffer: bf16 dS^T of every visible 128x128 tile of one
 * chunk of sequences, Hq * bd_tilemap_entries_bound(prob) * 32 KB per
 * sequence.  Env BD_BWD_DS unset: the buffer is used when the whole batch
 * fits BD_BWD_DS_BUDGET_MB (default 8,192 MiB; e.g. SDAR-1.7B at batch 16:
 * 3.6 GB; SDAR-8B: no buffer); BD_BWD_DS=1: always, in chunks of as many
 * sequences as fit the budget (default 24,576 MiB; SDAR-8B: 4 sequences,
 * 22.3 GB); BD_BWD_DS=0: never.  Without the buffer dQ recomputes S and dP.
 * The environment is read per call: keep it fixed between this query and
 * the call.  Returns 0 for an invalid problem. */
size_t bd_attn_workspace_bytes(const bd_problem* prob, int backward);

/* Forward.
 *   q    bf16 [b, Ntot, Hq,  d]      k, v  bf16 [b, Ntot, Hkv, d]
 *   o    bf16 [b, Ntot, Hq,  d]      (written)
 *        (row strides q_row_heads d / kv_row_heads d elements when set)
 *   lse  fp32 [b, Hq, Ntot]          natural-log log-sum-exp of the scaled,
 *                                    masked scores of each row (written)
 *   ws   device workspace of >= bd_attn_workspace_bytes(prob, 0) bytes.
 * O_i = sum_j softmax_j(scale q_i.k_j | M_ij) v_j.  Tiles of 128x128
 * that the mask leaves empty are never loaded ("accepts fine-grained
 * masks"; S:97 block skip).  Deterministic. */
int bd_attn_fwd(const bd_problem* prob, const void* q, const void* k, const void* v, void* o, float* lse,
                void* ws, size_t ws_bytes, void* stream);

/* Backward of bd_attn_fwd for upstream gradient dout (bf16, like q), given the
 * forward's o and lse.  Writes dq (bf16 like q) and dk, dv (bf16 like k); dk
 * and dv sum over the Hq/Hkv query heads of each kv head.  ws must be
 * >= bd_attn_workspace_bytes(prob, 1) bytes.  Kernels: preprocess, dK/dV
 * over the column tile map, dQ over the row tile map (recomputing S and dP).
 * With the stored-dS buffer (see bd_attn_workspace_bytes), per
 * chunk of sequences the dK/dV kernel also stores each tile's dS^T = P (dP -
 * D), bf16 (the value its dK MMA consumes), and dQ = scale dS K reads it back
 * instead of recomputing.  No atomics: the result is deterministic. */
int bd_attn_bwd(const bd_problem* prob, const void* q, const void* k, const void* v, const void* o,
                const float* lse, const void* dout, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes,
                void* stream);

/* Per-token log-probabilities over a vocabulary.
 *   logits   bf16 [n_rows, vocab] with row stride `row_stride` elements
 *   targets  int32 [n_rows]
 *   logp     fp32 [n_rows]  logp_n = z[n, t_n] - LSE_n        (written)
 *   lse      fp32 [n_rows]  LSE_n = ln sum_v exp z[n, v]      (written; may be NULL)
 *   dlogp    fp32 [n_rows]  upstream gradient w_n, or NULL for forward only
 *   dlogits  bf16 [n_rows, vocab] (row stride dlogits_stride) receiving
 *            w_n (1[v = t_n] - softmax(z_n)_v); may alias logits (in place,
 *            then dlogits_stride must equal row_stride); ignored if dlogp is NULL.
 * A target outside [0, vocab) yields logp = NaN for that row (the DiPO step
 * treats a non-finite value as "abort"). */
int bd_logprob(int64_t n_rows, int32_t vocab, const void* logits, int64_t row_stride, const int32_t* targets,
               float* logp, float* lse, const float* dlogp, void* dlogits, int64_t dlogits_stride, void* stream);

/* Gradient of bd_logprob from a known LSE (one read of the logits, one
 * write of the gradient), for when dlogp depends on logp (clipped ratios):
 *   dlogits[n, v] = dlogp_n (1[v = t_n] - exp(z[n, v] - lse_n)).
 * Arguments as in bd_logprob; lse is the fp32 [n_rows] output of bd_logprob;
 * dlogits may alias logits (in place, equal strides). */
int bd_logprob_bwd(int64_t n_rows, int32_t vocab, const void* logits, int64_t row_stride, const int32_t* targets,
                   const float* lse, const float* dlogp, void* dlogits, int64_t dlogits_stride, void* stream);

/* ---- LM head fused with the log-softmax gather ----
 * The policy probabilities of Eqs. 6-8 are the softmax of the
 * logits z = h W^T of the (bias-free, [ext] Qwen3/SDAR) LM head.  These calls
 * compute log-probs and their gradients straight from the hidden states: the
 * forward never materialises z [n, V]; the backward materialises only a chunk
 * of dz = w (1[v = t] - softmax(z)) (bf16, chunk_rows x V, in the workspace).
 *   h        bf16 [n_rows, hidden]     final hidden states of the scored rows
 *   w        bf16 [vocab, hidden]      LM-head weight (nn.Linear layout)
 *   targets  int32 [n_rows]            token ids (reading c9: rows are the caller's choice)
 * hidden and vocab must be multiples of 8 (16-byte rows; Qwen3: 4096 / 2048
 * and 151,936), else BD_ERR_UNSUPPORTED; pointers 16-byte aligned.
 * tcgen05 CTA-pair GEMMs (256 x 256 tiles), fp32 accumulation and fp32
 * softmax; deterministic. */

/* Workspace bytes: forward (backward = 0) holds per-chunk softmax partials;
 * backward holds one dz chunk of min(chunk_rows, n_rows) rows (chunk_rows
 * <= 0 means all rows).  0 for invalid sizes. */
size_t bd_lmhead_workspace_bytes(int64_t n_rows, int32_t hidden, int32_t vocab, int backward, int64_t chunk_rows);

/* Forward: logp[n] = z[n, t_n] - LSE_n, LSE_n = ln sum_v exp z[n, v], z = h W^T.
 *   logp  fp32 [n_rows] (written; NaN for a target outside [0, vocab))
 *   lse   fp32 [n_rows] (written; may be NULL -- the backward needs it) */
int bd_lmhead_logprob(int64_t n_rows, int32_t hidden, int32_t vocab, const void* h, const void* w,
                      const int32_t* targets, float* logp, float* lse, void* ws, size_t ws_bytes, void* stream);

/* Backward for upstream gradient dlogp (fp32 [n_rows]) given the forward's lse:
 *   dz = dlogp_n (1[v = t_n] - exp(z[n, v] - lse_n))      (recomputed, per chunk)
 *   dh bf16 [n_rows, hidden] = dz W                       (written)
 *   dw fp32 [vocab, hidden]  = dz^T h                     (written; summed over all rows)
 * Rows are processed in chunks of chunk_rows (<= 0: all at once); ws must hold
 * bd_lmhead_workspace_bytes(n_rows, hidden, vocab, 1, chunk_rows) bytes. */
int bd_lmhead_logprob_bwd(int64_t n_rows, int32_t hidden, int32_t vocab, const void* h, const void* w,
                          const int32_t* targets, const float* lse, const float* dlogp, void* dh, float* dw,
                          int64_t chunk_rows, void* ws, size_t ws_bytes, void* stream);

/* ---- Blockwise KV-cache decoding for the rollout ----
 * Blockwise dLLMs denoise the active block k conditioned on the clean history,
 * p(b^k_0 | b^k_t, b^{<k}) (Eq. 2), which admits a KV cache;
 * SPEC's inference mask: the active block sees every earlier block
 * and itself bidirectionally.
 *
 * Attention of the active block's B query rows to the first kv_len[b] cached
 * keys of each sequence (the caller has written the active block's own K/V at
 * [kv_len - B, kv_len)); no mask inside that range.
 *   q        bf16 [b, B, Hq, d]          k_cache, v_cache  bf16 [b, cap, Hkv, d]
 *   kv_len   int32 [b] (device), B <= kv_len <= cap; cache rows >= kv_len may
 *            hold anything (never read into the result)
 *   o        bf16 [b, B, Hq, d] (written)     lse  fp32 [b, Hq, B] natural log (written)
 * d must be 128 and B <= 32 (else BD_ERR_UNSUPPORTED); GQA kv(h) = h / (Hq/Hkv);
 * softmax_scale <= 0 -> 1/sqrt(d).  Split-KV tcgen05 kernel + combine;
 * deterministic.  ws: bd_decode_workspace_bytes(...) bytes (0 = invalid args). */
size_t bd_decode_workspace_bytes(int32_t batch, int32_t block, int32_t n_q_heads, int32_t n_kv_heads,
                                 int32_t head_dim, int32_t cap);
int bd_decode_attn(int32_t batch, int32_t block, int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                   int32_t cap, float softmax_scale, const void* q, const void* k_cache, const void* v_cache,
                   const int32_t* kv_len, void* o, float* lse, void* ws, size_t ws_bytes, void* stream);

/* Dynamic decoding step ("decoding tokens whose top-1 probability
 * exceeds 0.9 directly"; reading c20).
 *   logits  bf16 [b, B, vocab]    masked  uint8 [b, B] (1 = still [MASK])
 *   token   int32 [b, B]  argmax_v (lowest index among ties)        (written)
 *   conf    fp32 [b, B]   softmax probability of that token (fp32)   (written)
 *   commit  uint8 [b, B]  1 for every masked position with conf > threshold;
 *           if a sequence has masked positions but none qualifies, its most
 *           confident one (lowest position among ties); 0 elsewhere   (written)
 * threshold >= 1 gives static one-token-per-step decoding. */
int bd_decode_select(int32_t batch, int32_t block, int32_t vocab, const void* logits, const uint8_t* masked,
                     float threshold, int32_t* token, float* conf, uint8_t* commit, void* stream);

/* DiPO, step 1: per-group partial statistics of the local trajectories.
 *   rewards        fp32 [n_traj]       r_i
 *   group_of_traj  int32 [n_traj]      global group id in [0, n_groups); other ids are ignored
 *   traj_len       int32 [n_traj]      |tau_i| in tokens (reading c10)
 *   group_stats    fp64 [n_groups, 3]  += (sum r, count, sum |tau|)   (accumulated;
 *                                      zero it first; all-reduce(SUM) it across
 *                                      ranks when a group straddles ranks)
 * Deterministic: each group's sums run in trajectory order (no atomics). */
int bd_dipo_group_stats(int32_t n_traj, const float* rewards, const int32_t* group_of_traj,
                        const int32_t* traj_len, int32_t n_groups, double* group_stats, void* stream);

/* DiPO, step 2: token-level objective of Eq. 8 with the
 * stop-gradient behaviour policy of Eq. 7.
 *   logp, logp_old fp32 [n_tokens]    rho_k = exp(logp_k - logp_old_k); both NULL means
 *                                      the online setting of Eq. 7 (pi_old = sg(pi_theta)):
 *                                      rho == 1, so the weights are known before the
 *                                      log-probs (enables the fused bd_logprob pass)
 *   traj_of_token  int32 [n_tokens]    local trajectory index in [0, n_traj)
 *   rewards, group_of_traj             as in step 1 (n_traj local trajectories)
 *   group_stats    fp64 [n_groups, 3]  globally reduced output of step 1
 *   n_groups_global                    number of non-empty groups overall (the 1/n_groups
 *                                      normaliser; reading c11)
 *   eps                                clip range of C_eps
 *   dlogp          fp32 [n_tokens]     dloss/dlogp_k (written)
 *   partials       fp64 [3]            += (loss partial, tokens, clipped tokens)
 * A_i = r_i - mean_g r;  loss = -(1/n_groups) sum_g (1/N_g) sum C_eps(rho, A).
 * A token whose trajectory or group id is out of range, or whose group is
 * empty, gets dlogp = NaN and makes the loss partial NaN ("abort").
 * Deterministic: the partials are summed by one CTA in a fixed order. */
int bd_dipo_token_loss(int64_t n_tokens, const float* logp, const float* logp_old, const int32_t* traj_of_token,
                       int32_t n_traj, const float* rewards, const int32_t* group_of_traj, const double* group_stats,
                       int32_t n_groups, int32_t n_groups_global, float eps, float* dlogp, double* partials,
                       void* stream);

/* Tile map (host path, for tests).  Writes the ordered list of non-empty
 * 128x128 tiles as 5-tuples (q_seg, q_tile, k_seg, k_tile, kind) of int32
 * into host_out (capacity `cap` int32 elements), kind 1 = FULL, 2 = PARTIAL;
 * segment 0 = x0, 1 = xt; tiles in packed order.  *n_tiles (host) receives
 * the number of tuples.  Returns BD_ERR_WORKSPACE if cap is too small. */
int bd_tilemap_dump(const bd_problem* prob, int32_t* host_out, size_t cap, int64_t* n_tiles);

/* Tile-map statistics (host): counts of q-tiles, non-empty, FULL and PARTIAL
 * tiles per (sequence, head); out = int64[4]. */
int bd_tilemap_stats(const bd_problem* prob, int64_t* out);

/* Number of non-empty tiles per (sequence, head) computed from the candidate
 * ranges alone (O(NT); tilemap.cuh map_entries_bound): the per-(sequence,
 * q-head) stride of the stored dS^T tiles in the backward workspace.  Equals
 * bd_tilemap_stats' out[1] (tests check it); -1 on an invalid problem. */
int64_t bd_tilemap_entries_bound(const bd_problem* prob);

/* Diagnostic (host): checks that the per-row visible-key intervals used by the
 * forward/dQ kernels and the per-key visible-row intervals used by the dK/dV
 * kernel describe the same mask for every (row, key); *mismatches (host)
 * receives the count (0 expected).  Small problems only (Ntot^2 <= 2^26). */
int bd_tilemap_selfcheck(const bd_problem* prob, int64_t* mismatches);

/* Element mask (host, tests): the per-element visibility the kernels
 * evaluate on PARTIAL and ragged tiles, for rows [row0, row0 + n_rows) of
 * sequence `seq` (a varlen batch: that sequence's own lengths) and all of its
 * *n_keys packed keys: host_out[i * n_keys + k] bit 0 = key k inside row
 * row0 + i's visible interval (forward / dQ kernels), bit 1 = that row inside
 * key k's visible-row interval (dK/dV kernel).  Must equal the dense mask of
 * the rule ("bitmatrix and predicate agree everywhere").
 * Returns BD_ERR_WORKSPACE if cap < n_rows * n_keys (n_keys is set). */
int bd_mask_dump(const bd_problem* prob, int32_t seq, int64_t row0, int64_t n_rows, uint8_t* host_out, size_t cap,
                 int64_t* n_keys);

const char* bd_error_string(int code);
const char* bd_last_error(void);

/* Number of CUDA kernels this library has enqueued since it was loaded
 * (process-wide counter; bench.py reports launches per timed region). */
int64_t bd_launch_count(void);

/* Hardware self-test of the UMMA / TMEM / TMA conventions (diagnostic).
 * a, b, v bf16 [128][128]; c = a.b^T, o_* = bf16(c).v via TMEM-A, smem-A
 * (K-major) and smem-A (MN-major); all fp32 [128][128]. */
int bd_selftest_mma(const void* a, const void* b, const void* v, float* c, float* o_ts, float* o_ss, float* o_mn,
                    void* stream);

/* Self-test of the CTA-pair GEMM engine behind bd_lmhead_*: out fp32 [M][N] =
 * sum_k A[m, k] B[n, k]; a is bf16 [M][K] (a_mn = 0) or [K][M] (a_mn = 1), b
 * likewise; M, N, K multiples of 8. */
int bd_selftest_gemm(int32_t M, int32_t N, int32_t K, const void* a, int a_mn, const void* b, int b_mn, float* out,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BD_ATTN_H_ */
