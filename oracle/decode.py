"""Blockwise KV-cache decoding (rollout) primitives, fp64
(SURVEY §8(f) NEXT #4).

Blockwise dLLMs factorise p(x) = prod_k p(b^k | b^{<k}) (Eq. 1) and
denoise the active block in parallel conditioned on the clean history,
p(b^k_0 | b^k_t, b^{<k}) (Eq. 2), which is what lets a KV cache be
used.  SPEC's inference mask: a token of the active block
sees every token of the earlier blocks and every token of its own block.

* ``decode_attention``: the active block's B query rows (per head) attend to
  all ``kv_len`` cached keys of their sequence -- the clean blocks < k
  followed by the active block's own (noisy) keys, which the caller has
  written at [kv_len - B, kv_len).  No mask inside that range.
    q       [b, B, Hq, d]       k, v  [b, cap, Hkv, d]      kv_len [b]
    O_i     = sum_j softmax_j(scale q_i.k_j) v_j   over j < kv_len
    LSE_i   = ln sum_j exp(scale q_i.k_j)          -> [b, Hq, B]
  GQA: kv(h) = h // (Hq / Hkv) (reading c7).

* ``select_tokens``: dynamic decoding ("a threshold of 0.9, decoding
  tokens whose top-1 probability exceeds 0.9 directly").  For each still
  masked position: token = argmax_v z (lowest index among ties), conf =
  softmax(z)[token] = 1 / sum_v exp(z_v - max z).  Commit every masked
  position with conf > threshold; if none of a sequence's masked positions
  qualifies, commit the single most confident one (lowest position among
  ties) so every denoising step makes progress (reading c20; with
  threshold >= 1 this is static one-token-per-step decoding).

ORACLE: test infrastructure only (see oracle/__init__.py).
"""

import math

import numpy as np

from .attention import _f64


def decode_attention(q, k, v, kv_len, scale=None):
    """Return (O [b, B, Hq, d], LSE [b, Hq, B]) fp64."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    b, B, Hq, d = q.shape
    _, cap, Hkv, _ = k.shape
    if Hq % Hkv:
        raise ValueError("Hq % Hkv != 0")
    kv_len = [int(x) for x in np.asarray(kv_len).reshape(-1)]
    if len(kv_len) != b:
        raise ValueError("kv_len must have one entry per sequence")
    scale = 1.0 / math.sqrt(d) if scale is None or scale <= 0 else scale
    G = Hq // Hkv
    O = np.zeros((b, B, Hq, d))
    LSE = np.zeros((b, Hq, B))
    for s in range(b):
        n = kv_len[s]
        if not (B <= n <= cap):
            raise ValueError("need B <= kv_len <= cap (the active block's keys are in the cache)")
        for h in range(Hq):
            g = h // G
            S = scale * q[s, :, h, :] @ k[s, :n, g, :].T      # [B, n]
            m = S.max(axis=1, keepdims=True)
            e = np.exp(S - m)
            l = e.sum(axis=1, keepdims=True)
            O[s, :, h, :] = (e / l) @ v[s, :n, g, :]
            LSE[s, h, :] = (m + np.log(l))[:, 0]
    return O, LSE


def select_tokens(z, masked, threshold):
    """z [b, B, V] logits, masked [b, B] bool -> (token [b, B] int64, conf [b, B] fp64,
    commit [b, B] bool).  token/conf are defined for every position; commit only
    for masked ones."""
    z = _f64(z)
    masked = np.asarray(masked, dtype=bool)
    b, B, V = z.shape
    token = np.zeros((b, B), dtype=np.int64)
    conf = np.zeros((b, B))
    commit = np.zeros((b, B), dtype=bool)
    for s in range(b):
        for i in range(B):
            row = z[s, i]
            t = int(np.argmax(row))          # first maximal index
            token[s, i] = t
            conf[s, i] = 1.0 / np.exp(row - row[t]).sum()
        cand = [i for i in range(B) if masked[s, i]]
        if not cand:
            continue
        hit = [i for i in cand if conf[s, i] > threshold]
        if not hit:
            best = max(conf[s, i] for i in cand)
            hit = [min(i for i in cand if conf[s, i] == best)]
        commit[s, hit] = True
    return token, conf, commit
