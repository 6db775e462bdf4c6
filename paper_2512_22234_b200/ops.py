"""Thin Python binding of include/bd_attn.h.

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of libbdattn.so.  PyTorch supplies device memory, streams and
process groups.  There is no CPU fallback -- a missing library or a non-CUDA
tensor raises.
"""

from dataclasses import dataclass, replace
import ctypes
import math

import torch

from . import _lib
from ._lib import BdProblem, check

TILE = 128


@dataclass(frozen=True)
class Problem:
    """bd_problem (include/bd_attn.h): prompt/response lengths and block size
    as in the paper, GQA heads and head_dim."""
    batch: int
    prompt_len: int
    response_len: int
    block_size: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    repeat_prompt: int = 1
    softmax_scale: float = 0.0
    n_copies: int = 1  # S noisy copies (trace replay, reading c19)
    # varlen batch: per-sequence prompt / response lengths (tuples of `batch`
    # ints, both None = uniform); prompt_len / response_len are the maxima
    seq_prompt_lens: tuple = None
    seq_response_lens: tuple = None

    @property
    def L(self):
        return self.prompt_len + self.response_len

    @property
    def xb(self):
        return 0 if self.repeat_prompt else self.prompt_len

    @property
    def ntot(self):
        return self.L + max(self.n_copies, 1) * (self.L - self.xb)

    @property
    def scale(self):
        return self.softmax_scale if self.softmax_scale > 0 else 1.0 / math.sqrt(self.head_dim)

    def c(self):
        st = BdProblem(self.batch, self.prompt_len, self.response_len, self.block_size, self.n_q_heads,
                       self.n_kv_heads, self.head_dim, self.repeat_prompt, float(self.softmax_scale),
                       self.n_copies)
        if self.seq_prompt_lens is not None or self.seq_response_lens is not None:
            arrs = []
            for name, vals in (("seq_prompt_len", self.seq_prompt_lens), ("seq_response_len", self.seq_response_lens)):
                if vals is None:
                    continue
                arr = (ctypes.c_int32 * len(vals))(*[int(x) for x in vals])
                arrs.append(arr)
                setattr(st, name, ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32)))
            st._keep = arrs  # the arrays must outlive the call
        return st

    def seq_packed_len(self, i):
        """Packed length N_i of sequence i of a varlen batch."""
        if self.seq_prompt_lens is None:
            return self.ntot
        P, R = self.seq_prompt_lens[i], self.seq_response_lens[i]
        L = P + R
        return L + max(self.n_copies, 1) * (L - (0 if self.repeat_prompt else P))

    def with_(self, **kw):
        return replace(self, **kw)

    @staticmethod
    def from_cfg(cfg, **kw):
        rl = getattr(cfg, "resp_lens", None)
        p = Problem(cfg.batch, cfg.prompt_len, cfg.response_len, cfg.block_size, cfg.n_q_heads,
                    cfg.n_kv_heads, cfg.head_dim, cfg.repeat_prompt, n_copies=getattr(cfg, "n_copies", 1),
                    seq_prompt_lens=None if rl is None else (cfg.prompt_len,) * cfg.batch,
                    seq_response_lens=None if rl is None else tuple(rl))
        return p.with_(**kw) if kw else p


def _stream_ptr(t):
    return torch.cuda.current_stream(t.device).cuda_stream


def _need_cuda(*ts):
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise _lib.BdError("bd ops take CUDA tensors only (no CPU fallback)")
        if not t.is_contiguous():
            raise _lib.BdError("bd ops take contiguous tensors")


_ws_cache = {}


def workspace(nbytes, device):
    """Per-device workspace buffer, grown on demand (caller-owned memory)."""
    key = torch.device(device).index
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def packed_len(prob: Problem) -> int:
    p = prob.c()
    n = _lib.lib().bd_packed_len(ctypes.byref(p))
    if n < 0:
        raise _lib.BdError(_lib.lib().bd_last_error().decode())
    return n


def workspace_bytes(prob: Problem, backward: bool) -> int:
    p = prob.c()
    return _lib.lib().bd_attn_workspace_bytes(ctypes.byref(p), int(backward))


def attn_fwd(prob: Problem, q, k, v, o=None, lse=None):
    """bd_attn_fwd: returns (o bf16 like q, lse fp32 [b, Hq, Ntot])."""
    _need_cuda(q, k, v)
    if o is None:
        o = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((prob.batch, prob.n_q_heads, prob.ntot), dtype=torch.float32, device=q.device)
    p = prob.c()
    nbytes = _lib.lib().bd_attn_workspace_bytes(ctypes.byref(p), 0)
    ws = workspace(nbytes, q.device)
    check(_lib.lib().bd_attn_fwd(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                 lse.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(q)), "bd_attn_fwd")
    return o, lse


def attn_bwd(prob: Problem, q, k, v, o, lse, do, dq=None, dk=None, dv=None):
    """bd_attn_bwd: returns (dq, dk, dv) bf16."""
    _need_cuda(q, k, v, o, lse, do)
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    p = prob.c()
    nbytes = _lib.lib().bd_attn_workspace_bytes(ctypes.byref(p), 1)
    ws = workspace(nbytes, q.device)
    check(_lib.lib().bd_attn_bwd(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                 lse.data_ptr(), do.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                 ws.data_ptr(), ws.numel(), _stream_ptr(q)), "bd_attn_bwd")
    return dq, dk, dv


class BlockDiffusionAttention(torch.autograd.Function):
    """autograd wrapper: forward = bd_attn_fwd, backward = bd_attn_bwd."""

    @staticmethod
    def forward(ctx, q, k, v, prob):
        o, lse = attn_fwd(prob, q, k, v)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.prob = prob
        return o, lse

    @staticmethod
    def backward(ctx, do, dlse):
        q, k, v, o, lse = ctx.saved_tensors
        dq, dk, dv = attn_bwd(ctx.prob, q, k, v, o, lse, do.contiguous())
        return dq, dk, dv, None


def block_diffusion_attention(q, k, v, prob: Problem):
    return BlockDiffusionAttention.apply(q, k, v, prob)[0]


def logprob(logits, targets, dlogp=None, dlogits=None, lse=None):
    """bd_logprob over bf16 logits [N, V] (row stride may exceed V).

    Returns logp (and writes dlogits when dlogp is given; dlogits may be
    `logits` itself for an in-place gradient)."""
    _need_cuda(targets, dlogp)
    if not logits.is_cuda or logits.stride(1) != 1:
        raise _lib.BdError("logits must be a CUDA tensor with unit inner stride")
    n, V = logits.shape
    logp = torch.empty(n, dtype=torch.float32, device=logits.device)
    lse_t = torch.empty(n, dtype=torch.float32, device=logits.device) if lse is None else lse
    dl_ptr = dlogp.data_ptr() if dlogp is not None else None
    if dlogp is not None and dlogits is None:
        dlogits = torch.empty_like(logits)
    dz_ptr = dlogits.data_ptr() if dlogits is not None else None
    dz_stride = dlogits.stride(0) if dlogits is not None else 0
    check(_lib.lib().bd_logprob(n, V, logits.data_ptr(), logits.stride(0), targets.data_ptr(), logp.data_ptr(),
                                lse_t.data_ptr(), dl_ptr, dz_ptr, dz_stride, _stream_ptr(logits)), "bd_logprob")
    return (logp, lse_t, dlogits) if dlogp is not None else (logp, lse_t)


def tilemap_dump(prob: Problem):
    """Host path of the tile-map builder: list of (q_seg, q_tile, k_seg, k_tile, kind)."""
    p = prob.c()
    n = ctypes.c_int64(0)
    L = _lib.lib()
    rc = L.bd_tilemap_dump(ctypes.byref(p), None, 0, ctypes.byref(n))
    if rc not in (0, 5):
        check(rc, "bd_tilemap_dump")
    buf = (ctypes.c_int32 * (5 * n.value))()
    check(L.bd_tilemap_dump(ctypes.byref(p), buf, 5 * n.value, ctypes.byref(n)), "bd_tilemap_dump")
    flat = list(buf)
    return [tuple(flat[i:i + 5]) for i in range(0, len(flat), 5)]


def tilemap_stats(prob: Problem):
    p = prob.c()
    out = (ctypes.c_int64 * 4)()
    check(_lib.lib().bd_tilemap_stats(ctypes.byref(p), out), "bd_tilemap_stats")
    return {"tiles": out[0], "nonempty": out[1], "full": out[2], "partial": out[3]}


def tilemap_host_image(prob: Problem):
    p = prob.c()
    L = _lib.lib()
    fn = L.bd_tilemap_host_image
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(BdProblem), ctypes.POINTER(ctypes.c_int32), ctypes.c_size_t,
                   ctypes.POINTER(ctypes.c_int64)]
    n = ctypes.c_int64(0)
    fn(ctypes.byref(p), None, 0, ctypes.byref(n))
    buf = (ctypes.c_int32 * n.value)()
    check(fn(ctypes.byref(p), buf, n.value, ctypes.byref(n)), "bd_tilemap_host_image")
    return list(buf)


def logprob_bwd(logits, targets, lse, dlogp, dlogits=None):
    """bd_logprob_bwd: dlogits = dlogp (onehot - softmax) from a known LSE (may be in place)."""
    _need_cuda(targets, lse, dlogp)
    if not logits.is_cuda or logits.stride(1) != 1:
        raise _lib.BdError("logits must be a CUDA tensor with unit inner stride")
    n, V = logits.shape
    if dlogits is None:
        dlogits = torch.empty_like(logits)
    check(_lib.lib().bd_logprob_bwd(n, V, logits.data_ptr(), logits.stride(0), targets.data_ptr(), lse.data_ptr(),
                                    dlogp.data_ptr(), dlogits.data_ptr(), dlogits.stride(0), _stream_ptr(logits)),
          "bd_logprob_bwd")
    return dlogits


def lmhead_logprob(h, w, targets):
    """bd_lmhead_logprob: (logp, lse) fp32 [n] of softmax(h w^T) at targets, logits never materialised."""
    _need_cuda(h, w, targets)
    n, C = h.shape
    V = w.shape[0]
    logp = torch.empty(n, dtype=torch.float32, device=h.device)
    lse = torch.empty(n, dtype=torch.float32, device=h.device)
    L = _lib.lib()
    ws = workspace(L.bd_lmhead_workspace_bytes(n, C, V, 0, 0), h.device)
    check(L.bd_lmhead_logprob(n, C, V, h.data_ptr(), w.data_ptr(), targets.data_ptr(), logp.data_ptr(),
                              lse.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(h)), "bd_lmhead_logprob")
    return logp, lse


def lmhead_logprob_bwd(h, w, targets, lse, dlogp, chunk_rows=16384, dh=None, dw=None):
    """bd_lmhead_logprob_bwd: (dh bf16 like h, dw fp32 [V, C]) for upstream dL/dlogp."""
    _need_cuda(h, w, targets, lse, dlogp)
    n, C = h.shape
    V = w.shape[0]
    dh = torch.empty_like(h) if dh is None else dh
    dw = torch.empty((V, C), dtype=torch.float32, device=h.device) if dw is None else dw
    L = _lib.lib()
    ws = workspace(L.bd_lmhead_workspace_bytes(n, C, V, 1, chunk_rows), h.device)
    check(L.bd_lmhead_logprob_bwd(n, C, V, h.data_ptr(), w.data_ptr(), targets.data_ptr(), lse.data_ptr(),
                                  dlogp.data_ptr(), dh.data_ptr(), dw.data_ptr(), chunk_rows, ws.data_ptr(),
                                  ws.numel(), _stream_ptr(h)), "bd_lmhead_logprob_bwd")
    return dh, dw


def decode_attn(q, k_cache, v_cache, kv_len, softmax_scale=0.0, o=None, lse=None):
    """bd_decode_attn: active-block attention over the KV cache -> (o bf16 like q, lse fp32 [b, Hq, B])."""
    _need_cuda(q, k_cache, v_cache, kv_len)
    b, B, Hq, d = q.shape
    _, cap, Hkv, _ = k_cache.shape
    o = torch.empty_like(q) if o is None else o
    lse = torch.empty((b, Hq, B), dtype=torch.float32, device=q.device) if lse is None else lse
    L = _lib.lib()
    nbytes = L.bd_decode_workspace_bytes(b, B, Hq, Hkv, d, cap)
    ws = workspace(max(nbytes, 256), q.device)
    check(L.bd_decode_attn(b, B, Hq, Hkv, d, cap, float(softmax_scale), q.data_ptr(), k_cache.data_ptr(),
                           v_cache.data_ptr(), kv_len.data_ptr(), o.data_ptr(), lse.data_ptr(), ws.data_ptr(),
                           ws.numel(), _stream_ptr(q)), "bd_decode_attn")
    return o, lse


def decode_select(logits, masked, threshold=0.9):
    """bd_decode_select over bf16 logits [b, B, V] and uint8 masked [b, B] -> (token, conf, commit)."""
    _need_cuda(logits, masked)
    b, B, V = logits.shape
    token = torch.empty((b, B), dtype=torch.int32, device=logits.device)
    conf = torch.empty((b, B), dtype=torch.float32, device=logits.device)
    commit = torch.empty((b, B), dtype=torch.uint8, device=logits.device)
    check(_lib.lib().bd_decode_select(b, B, V, logits.data_ptr(), masked.data_ptr(), float(threshold),
                                      token.data_ptr(), conf.data_ptr(), commit.data_ptr(), _stream_ptr(logits)),
          "bd_decode_select")
    return token, conf, commit


def selftest_gemm(a, b, a_mn=False, b_mn=False):
    """bd_selftest_gemm: fp32 A B^T of the CTA-pair GEMM engine (operands K- or MN-major)."""
    _need_cuda(a, b)
    M = a.shape[1] if a_mn else a.shape[0]
    K = a.shape[0] if a_mn else a.shape[1]
    N = b.shape[1] if b_mn else b.shape[0]
    out = torch.empty((M, N), dtype=torch.float32, device=a.device)
    check(_lib.lib().bd_selftest_gemm(M, N, K, a.data_ptr(), int(a_mn), b.data_ptr(), int(b_mn), out.data_ptr(),
                                      _stream_ptr(a)), "bd_selftest_gemm")
    return out


def launch_count() -> int:
    """Kernels enqueued by libbdattn.so so far (process-wide)."""
    return int(_lib.lib().bd_launch_count())


def dipo_group_stats(rewards, group_of_traj, traj_len, n_groups, out=None):
    """bd_dipo_group_stats: fp64 [n_groups, 3] += (sum r, count, sum |tau|)."""
    _need_cuda(rewards, group_of_traj, traj_len)
    if out is None:
        out = torch.zeros((n_groups, 3), dtype=torch.float64, device=rewards.device)
    check(_lib.lib().bd_dipo_group_stats(rewards.numel(), rewards.data_ptr(), group_of_traj.data_ptr(),
                                         traj_len.data_ptr(), n_groups, out.data_ptr(), _stream_ptr(rewards)),
          "bd_dipo_group_stats")
    return out


def dipo_token_loss(logp, logp_old, traj_of_token, rewards, group_of_traj, group_stats, n_groups_global,
                    eps=0.2, partials=None):
    """bd_dipo_token_loss: returns (dlogp fp32 [n], partials fp64 [3] += (loss, tokens, clipped))."""
    _need_cuda(logp, logp_old, traj_of_token, rewards, group_of_traj, group_stats)
    if (logp is None) != (logp_old is None):
        raise _lib.BdError("logp and logp_old must both be given or both be None (rho == 1)")
    dlogp = torch.empty(traj_of_token.numel(), dtype=torch.float32, device=traj_of_token.device)
    if partials is None:
        partials = torch.zeros(3, dtype=torch.float64, device=traj_of_token.device)
    lp = logp.data_ptr() if logp is not None else None
    lo = logp_old.data_ptr() if logp_old is not None else None
    check(_lib.lib().bd_dipo_token_loss(traj_of_token.numel(), lp, lo, traj_of_token.data_ptr(),
                                        rewards.data_ptr(), group_of_traj.data_ptr(), group_stats.data_ptr(),
                                        int(n_groups_global), float(eps), dlogp.data_ptr(), partials.data_ptr(),
                                        _stream_ptr(traj_of_token)), "bd_dipo_token_loss")
    return dlogp, partials
