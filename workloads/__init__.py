"""Seeded synthetic workloads shared by the tests, smoke() and bench.py.

This module holds shapes and random-number recipes ONLY -- none of the
method's arithmetic -- so that both the CUDA path and the fp64 oracle can be
fed the same inputs without sharing code (DESIGN.md §3 "input recipe").

Shapes are BASELINE.json's configs (SDAR / Qwen3-shaped heads; the paper's
RL workload is "batch size 4, input length 1024 and output length 8192",
P:294).  Value distributions:

* q, k, v, dO ~ N(0, 1), rounded to bf16 (mimics post-QK-norm activations);
  ``stress`` multiplies q by 8 for peaky softmax / frequent rescaling;
  ``structured_do`` zeroes dO on x0 rows and noisy-prompt rows (only the
  repeated response carries loss).
* logits ~ N(0, 3^2) (optionally the target logit + 20), targets uniform.
* rewards ~ Bernoulli(0.5) per trajectory.
"""

from dataclasses import dataclass, replace
import math

import torch

VOCAB_QWEN3 = 151_936  # [ext] Qwen3 / SDAR vocabulary (reading c18)


@dataclass(frozen=True)
class AttnConfig:
    name: str
    batch: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    prompt_len: int
    response_len: int
    block_size: int
    repeat_prompt: int = 1
    seed: int = 0
    n_copies: int = 1  # S noisy copies: trace replay (reading c19)
    resp_lens: tuple = None  # varlen: per-sequence response lengths (<= response_len)

    @property
    def L(self):
        return self.prompt_len + self.response_len

    @property
    def xb(self):
        return 0 if self.repeat_prompt else self.prompt_len

    @property
    def ntot(self):
        return self.L + self.n_copies * (self.L - self.xb)

    def with_(self, **kw):
        return replace(self, **kw)


CONFIGS = {
    "tiny": AttnConfig("tiny", 1, 2, 2, 64, 32, 64, 4, seed=0),
    "sdar_1_7b": AttnConfig("sdar_1_7b", 16, 16, 8, 128, 512, 2048, 4, seed=1),
    "sdar_8b": AttnConfig("sdar_8b", 16, 32, 8, 128, 1024, 8192, 4, seed=2),
    "sweep_b4": AttnConfig("sweep_b4", 16, 32, 8, 128, 1024, 4096, 4, seed=3),
    "sweep_b8": AttnConfig("sweep_b8", 16, 32, 8, 128, 1024, 4096, 8, seed=3),
    "sweep_b16": AttnConfig("sweep_b16", 16, 32, 8, 128, 1024, 4096, 16, seed=3),
    "sweep_b32": AttnConfig("sweep_b32", 16, 32, 8, 128, 1024, 4096, 32, seed=3),
    # 8xB200 RL step: 128 prompts x group 8 = 1024 sequences, micro-batch 16
    "rl8_micro": AttnConfig("rl8_micro", 16, 32, 8, 128, 1024, 8192, 4, seed=4),
    # trace replay: SDAR-8B shape, B = 4 decoded one token
    # per step -> S = 4 noisy copies [x0 | xt(1) | .. | xt(4)], Ntot = 5 L
    "trace_s4": AttnConfig("trace_s4", 16, 32, 8, 128, 1024, 8192, 4, seed=5, n_copies=4),
    # varlen: SDAR-8B heads, one group of 16 rollouts with
    # response lengths ~ U[512, 8192] (multiples of B, seeded): mean ~4.3k, inside
    # the paper's 707-5,434 per-benchmark averages under the 8k cap
    "sdar_8b_varlen": AttnConfig("sdar_8b_varlen", 16, 32, 8, 128, 1024, 8192, 4, seed=6,
                                 resp_lens=tuple(int(x) for x in (
                                     (torch.randint(128, 2049, (16,), generator=torch.Generator().manual_seed(6))
                                      * 4).tolist()))),
}

# logprob rows per config: N = b * R response rows
LOGPROB_ROWS = {"tiny": 64, "sdar_1_7b": 16 * 2048, "sdar_8b": 16 * 8192}


def _gen(seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def attn_inputs(cfg: AttnConfig, device="cpu", seed=None, stress=False, dtype=torch.bfloat16,
                with_do=True, structured_do=False):
    """q, k, v, do tensors in the ABI layout [b, Ntot, H, d] (bf16)."""
    seed = cfg.seed if seed is None else seed
    g = _gen(seed, device)
    N = cfg.ntot
    shape_q = (cfg.batch, N, cfg.n_q_heads, cfg.head_dim)
    shape_k = (cfg.batch, N, cfg.n_kv_heads, cfg.head_dim)
    q = torch.randn(shape_q, generator=g, device=device, dtype=torch.float32)
    if stress:
        q = q * 8.0
    q = q.to(dtype)
    k = torch.randn(shape_k, generator=g, device=device, dtype=torch.float32).to(dtype)
    v = torch.randn(shape_k, generator=g, device=device, dtype=torch.float32).to(dtype)
    do = None
    if with_do:
        do = torch.randn(shape_q, generator=g, device=device, dtype=torch.float32)
        if structured_do:
            # zero on x0 rows and on noisy-prompt rows (loss only on the
            # repeated response)
            keep = torch.zeros(N, device=device, dtype=torch.float32)
            Lx = cfg.L - cfg.xb
            for c in range(cfg.n_copies):
                keep[cfg.L + c * Lx + (cfg.prompt_len - cfg.xb):cfg.L + (c + 1) * Lx] = 1.0
            do = do * keep[None, :, None, None]
        do = do.to(dtype)
    return q, k, v, do


def logits_inputs(n_rows, vocab, device="cpu", seed=0, peaked=False, dtype=torch.bfloat16):
    """z ~ N(0, 3^2) [n_rows, vocab] and uniform targets [n_rows] int32."""
    g = _gen(seed, device)
    z = torch.randn((n_rows, vocab), generator=g, device=device, dtype=torch.float32) * 3.0
    t = torch.randint(0, vocab, (n_rows,), generator=g, device=device, dtype=torch.int64)
    if peaked and n_rows:
        z[torch.arange(n_rows, device=device), t] += 20.0
    return z.to(dtype), t.to(torch.int32)


# LM head + logprob: rows = b * R response rows,
# hidden = [ext] Qwen3 hidden size (4,096 for 8B, 2,048 for 1.7B), V = 151,936.
LMHEAD_SHAPES = {"tiny": (64, 256, 1000), "sdar_1_7b": (16 * 2048, 2048, VOCAB_QWEN3),
                 "sdar_8b": (16 * 8192, 4096, VOCAB_QWEN3)}


def lmhead_inputs(n_rows, hidden, vocab, device="cpu", seed=0, dtype=torch.bfloat16):
    """h ~ N(0, 1) [n_rows, hidden] (post-final-norm hidden states), W ~ N(0, (3/sqrt(hidden))^2)
    [vocab, hidden] (so logits ~ N(0, 3^2) like logits_inputs), uniform targets int32 [n_rows]
    and upstream weights w ~ N(0, 1) fp32 [n_rows]."""
    g = _gen(seed, device)
    h = torch.randn((n_rows, hidden), generator=g, device=device, dtype=torch.float32).to(dtype)
    W = (torch.randn((vocab, hidden), generator=g, device=device, dtype=torch.float32)
         * (3.0 / math.sqrt(hidden))).to(dtype)
    t = torch.randint(0, vocab, (n_rows,), generator=g, device=device, dtype=torch.int64).to(torch.int32)
    w = torch.randn((n_rows,), generator=g, device=device, dtype=torch.float32)
    return h, W, t, w


# Blockwise KV-cache decode: per GPU the 8xB200 RL step's
# 128 rollouts (128 prompts x G 8 / 8 GPUs), SDAR-8B heads, B = 4, cache capacity
# P + R = 9,216; mid-rollout cache lengths kv_len ~ U over block multiples in
# [P + B, P + R] (the active block's keys are the last B).
DECODE_SHAPES = {"tiny": dict(batch=3, block=4, n_q_heads=4, n_kv_heads=2, head_dim=128, cap=300),
                 "sdar_8b": dict(batch=128, block=4, n_q_heads=32, n_kv_heads=8, head_dim=128, cap=9216)}


def decode_inputs(batch, block, n_q_heads, n_kv_heads, head_dim, cap, device="cpu", seed=0, min_len=None,
                  dtype=torch.bfloat16):
    """q [b, B, Hq, d], k/v caches [b, cap, Hkv, d] ~ N(0, 1) bf16 and kv_len int32 [b]
    (multiples of B in [max(B, min_len), cap])."""
    g = _gen(seed, device)
    q = torch.randn((batch, block, n_q_heads, head_dim), generator=g, device=device).to(dtype)
    k = torch.randn((batch, cap, n_kv_heads, head_dim), generator=g, device=device).to(dtype)
    v = torch.randn((batch, cap, n_kv_heads, head_dim), generator=g, device=device).to(dtype)
    lo = max(1, (min_len or block) // block)
    kv_len = (torch.randint(lo, cap // block + 1, (batch,), generator=_gen(seed + 1, "cpu")) * block).to(torch.int32)
    return q, k, v, kv_len.to(device)


def rl_batch(n_groups, group_size, resp_lens, seed=0):
    """Rewards ~ Bernoulli(0.5), trajectory/group ids and per-token traj ids.

    resp_lens: int (fixed length) or list per trajectory."""
    g = torch.Generator().manual_seed(int(seed))
    n_traj = n_groups * group_size
    rewards = torch.bernoulli(torch.full((n_traj,), 0.5), generator=g).double()
    group_of_traj = torch.arange(n_groups).repeat_interleave(group_size)
    if isinstance(resp_lens, int):
        lens = [resp_lens] * n_traj
    else:
        lens = list(resp_lens)
    traj_of_token = torch.cat([torch.full((n,), i, dtype=torch.int64) for i, n in enumerate(lens)])
    return rewards, group_of_traj, traj_of_token


def useful_pairs(cfg: AttnConfig) -> int:
    """Closed-form count of visible pairs per (sequence, head) in DiRL mode,
    L (L + B) (derived), (1 + S) L (L + B) / 2 with S noisy
    copies (reading c19); for response-only mode counted by the caller from
    the oracle."""
    assert cfg.repeat_prompt == 1
    return (1 + cfg.n_copies) * cfg.L * (cfg.L + cfg.block_size) // 2


def total_pairs(cfg: AttnConfig) -> int:
    """Visible pairs per head summed over the batch (varlen: per sequence)."""
    if cfg.resp_lens is None:
        return cfg.batch * useful_pairs(cfg)
    return sum(useful_pairs(cfg.with_(response_len=r, resp_lens=None)) for r in cfg.resp_lens)


def total_tokens(cfg: AttnConfig) -> int:
    """Original (clean) tokens of the batch, sum of L_i."""
    if cfg.resp_lens is None:
        return cfg.batch * cfg.L
    return sum(cfg.prompt_len + r for r in cfg.resp_lens)


def useful_flops(cfg: AttnConfig, pairs=None):
    """(fwd, bwd) useful FLOPs: fwd = 4 d Hq b pairs, bwd = 2.5 x fwd
    (flash convention)."""
    if pairs is None:
        fwd = 4 * cfg.head_dim * cfg.n_q_heads * total_pairs(cfg)
    else:
        fwd = 4 * cfg.head_dim * cfg.n_q_heads * cfg.batch * pairs
    return fwd, 2.5 * fwd


def _ceil_div(a, b):
    return -(-a // b)


__all__ = ["AttnConfig", "CONFIGS", "attn_inputs", "logits_inputs", "lmhead_inputs", "LMHEAD_SHAPES", "decode_inputs", "DECODE_SHAPES", "rl_batch", "useful_pairs", "total_pairs",
           "total_tokens",
           "useful_flops", "VOCAB_QWEN3", "LOGPROB_ROWS", "math"]
