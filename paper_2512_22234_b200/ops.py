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
    # head sharding: heads per token row in memory of q/o/dO/dQ and k/v/dK/dV
    # (0 = dense); see head_shard()
    q_row_heads: int = 0
    kv_row_heads: int = 0

    @property
    def q_rows(self):
        return self.q_row_heads or self.n_q_heads

    @property
    def kv_rows(self):
        return self.kv_row_heads or self.n_kv_heads

    def head_shard(self, kv0, n_kv):
        """Problem of kv heads [kv0, kv0 + n_kv) (and their query heads) of this
        problem, run in place on head slices of the full-width tensors
        (SURVEY 8(e) (sequence, kv-head-group) units): slice q/o/dO/dQ with
        head_slice_q() and k/v/dK/dV with head_slice_kv()."""
        if not (0 <= kv0 and n_kv > 0 and kv0 + n_kv <= self.n_kv_heads):
            raise _lib.BdError(f"kv head range [{kv0}, {kv0 + n_kv}) outside [0, {self.n_kv_heads})")
        g = self.n_q_heads // self.n_kv_heads
        return replace(self, n_q_heads=n_kv * g, n_kv_heads=n_kv, q_row_heads=self.q_rows, kv_row_heads=self.kv_rows,
                       _shard=(kv0 * g, kv0))

    _shard: tuple = (0, 0)

    def head_slice_q(self, t):
        h0 = self._shard[0]
        return t[:, :, h0:h0 + self.n_q_heads]

    def head_slice_kv(self, t):
        h0 = self._shard[1]
        return t[:, :, h0:h0 + self.n_kv_heads]

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
        st.q_row_heads = int(self.q_row_heads)
        st.kv_row_heads = int(self.kv_row_heads)
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


def _err(msg):
    raise _lib.BdError(msg)


def _same_device(*ts):
    devs = {t.device for t in ts if t is not None}
    if len(devs) > 1:
        _err(f"tensors on different devices: {sorted(str(d) for d in devs)}")


def _check(name, t, dtype, shape=None, contiguous=True):
    """Validate one ABI argument before its pointer crosses the boundary: the
    library reads raw pointers, so a wrong dtype / shape / device would read
    or write out of bounds or silently misinterpret the data."""
    if t is None:
        _err(f"{name} is None")
    if not t.is_cuda:
        _err(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        _err(f"{name} must be {dtype}, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        _err(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if contiguous and not t.is_contiguous():
        _err(f"{name} must be contiguous")
    if t.data_ptr() % 16:
        _err(f"{name} must be 16-byte aligned")


def _check_rows(name, t, b, N, H, RH, d):
    """[b, N, H, d] bf16 whose token rows hold RH >= H heads in memory (a head
    slice of a [b, N, RH, d] tensor when RH > H, head sharding)."""
    _check(name, t, torch.bfloat16, (b, N, H, d), contiguous=False)
    want = (N * RH * d, RH * d, d, 1)
    got = t.stride()
    if any(g != w for g, w, n in zip(got, want, t.shape) if n > 1):
        _err(f"{name} strides {got} do not match the [b, N, {RH}, d] row layout {want}")


def workspace(nbytes, device):
    """Workspace of one call, allocated on the current stream of `device`.

    The caching allocator makes this cheap and stream-ordered: the block is
    reused only by work queued later on the same stream, so concurrent calls on
    different streams never share a tile map, and CUDA-graph capture takes it
    from the graph's private pool (no buffer a graph captured is ever freed
    under it).  Callers may pass their own buffer (``ws=``) instead."""
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _ws(ws, nbytes, device):
    if ws is None:
        return workspace(nbytes, device)
    _check("ws", ws, torch.uint8)
    if ws.numel() < nbytes:
        _err(f"workspace holds {ws.numel()} bytes, {nbytes} needed")
    if ws.device != torch.device(device):
        _err("workspace on another device")
    return ws


def packed_len(prob: Problem) -> int:
    p = prob.c()
    n = _lib.lib().bd_packed_len(ctypes.byref(p))
    if n < 0:
        raise _lib.BdError(_lib.lib().bd_last_error().decode())
    return n


def workspace_bytes(prob: Problem, backward: bool) -> int:
    p = prob.c()
    return _lib.lib().bd_attn_workspace_bytes(ctypes.byref(p), int(backward))


def _check_attn_inputs(prob: Problem, q, k, v):
    N, d = prob.ntot, prob.head_dim
    _check_rows("q", q, prob.batch, N, prob.n_q_heads, prob.q_rows, d)
    _check_rows("k", k, prob.batch, N, prob.n_kv_heads, prob.kv_rows, d)
    _check_rows("v", v, prob.batch, N, prob.n_kv_heads, prob.kv_rows, d)


def attn_fwd(prob: Problem, q, k, v, o=None, lse=None, ws=None):
    """bd_attn_fwd: returns (o bf16 like q, lse fp32 [b, Hq, Ntot]).

    With head sharding (prob.q_row_heads / kv_row_heads set) q, k, v (and o)
    are head slices of full-width tensors; a missing o is allocated full width
    and returned as the matching slice."""
    _check_attn_inputs(prob, q, k, v)
    if o is None:
        o = torch.empty((prob.batch, prob.ntot, prob.q_rows, prob.head_dim), dtype=q.dtype,
                        device=q.device)[:, :, :prob.n_q_heads]
    if lse is None:
        lse = torch.empty((prob.batch, prob.n_q_heads, prob.ntot), dtype=torch.float32, device=q.device)
    _check_rows("o", o, prob.batch, prob.ntot, prob.n_q_heads, prob.q_rows, prob.head_dim)
    _check("lse", lse, torch.float32, (prob.batch, prob.n_q_heads, prob.ntot))
    _same_device(q, k, v, o, lse)
    p = prob.c()
    L = _lib.lib()
    with torch.cuda.device(q.device):
        nbytes = L.bd_attn_workspace_bytes(ctypes.byref(p), 0)
        w = _ws(ws, nbytes, q.device)
        check(L.bd_attn_fwd(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                            lse.data_ptr(), w.data_ptr(), w.numel(), _stream_ptr(q)), "bd_attn_fwd")
    return o, lse


def attn_bwd(prob: Problem, q, k, v, o, lse, do, dq=None, dk=None, dv=None, ws=None):
    """bd_attn_bwd: returns (dq, dk, dv) bf16 (laid out like q, k, v)."""
    _check_attn_inputs(prob, q, k, v)
    b, N, d = prob.batch, prob.ntot, prob.head_dim
    _check_rows("o", o, b, N, prob.n_q_heads, prob.q_rows, d)
    _check_rows("do", do, b, N, prob.n_q_heads, prob.q_rows, d)
    _check("lse", lse, torch.float32, (b, prob.n_q_heads, N))

    def like(t, H, RH):
        return torch.empty((b, N, RH, d), dtype=t.dtype, device=t.device)[:, :, :H]
    dq = like(q, prob.n_q_heads, prob.q_rows) if dq is None else dq
    dk = like(k, prob.n_kv_heads, prob.kv_rows) if dk is None else dk
    dv = like(v, prob.n_kv_heads, prob.kv_rows) if dv is None else dv
    _check_rows("dq", dq, b, N, prob.n_q_heads, prob.q_rows, d)
    _check_rows("dk", dk, b, N, prob.n_kv_heads, prob.kv_rows, d)
    _check_rows("dv", dv, b, N, prob.n_kv_heads, prob.kv_rows, d)
    _same_device(q, k, v, o, lse, do, dq, dk, dv)
    p = prob.c()
    L = _lib.lib()
    with torch.cuda.device(q.device):
        nbytes = L.bd_attn_workspace_bytes(ctypes.byref(p), 1)
        w = _ws(ws, nbytes, q.device)
        check(L.bd_attn_bwd(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                            lse.data_ptr(), do.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                            w.data_ptr(), w.numel(), _stream_ptr(q)), "bd_attn_bwd")
    return dq, dk, dv


class BlockDiffusionAttention(torch.autograd.Function):
    """autograd wrapper: forward = bd_attn_fwd, backward = bd_attn_bwd.

    The LSE output is not differentiable (marked so): a loss that depends on
    it gets no gradient through it rather than a silently wrong one."""

    @staticmethod
    def forward(ctx, q, k, v, prob):
        o, lse = attn_fwd(prob, q, k, v)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.prob = prob
        ctx.mark_non_differentiable(lse)
        return o, lse

    @staticmethod
    def backward(ctx, do, dlse):
        q, k, v, o, lse = ctx.saved_tensors
        prob = ctx.prob
        if do is None:
            do = torch.zeros_like(o)
        elif prob.q_rows == prob.n_q_heads:
            do = do.contiguous()
        else:
            full = torch.zeros((prob.batch, prob.ntot, prob.q_rows, prob.head_dim), dtype=do.dtype,
                               device=do.device)
            full[:, :, :prob.n_q_heads] = do
            do = full[:, :, :prob.n_q_heads]
        dq, dk, dv = attn_bwd(prob, q, k, v, o, lse, do)
        return dq, dk, dv, None


def block_diffusion_attention(q, k, v, prob: Problem):
    return BlockDiffusionAttention.apply(q, k, v, prob)[0]


def _check_logits(logits, name="logits"):
    if logits is None or not logits.is_cuda:
        _err(f"{name} must be a CUDA tensor (no CPU fallback)")
    if logits.dtype != torch.bfloat16:
        _err(f"{name} must be bf16, got {logits.dtype}")
    if logits.dim() != 2 or logits.stride(1) != 1:
        _err(f"{name} must be 2-D [N, V] with unit inner stride")


def logprob(logits, targets, dlogp=None, dlogits=None, lse=None):
    """bd_logprob over bf16 logits [N, V] (row stride may exceed V).

    Returns (logp, lse) or, when dlogp is given, (logp, lse, dlogits) with
    dlogits = dlogp (onehot - softmax) written (dlogits may be `logits` itself
    for an in-place gradient)."""
    _check_logits(logits)
    n, V = logits.shape
    _check("targets", targets, torch.int32, (n,))
    if dlogp is not None:
        _check("dlogp", dlogp, torch.float32, (n,))
    logp = torch.empty(n, dtype=torch.float32, device=logits.device)
    lse_t = torch.empty(n, dtype=torch.float32, device=logits.device) if lse is None else lse
    _check("lse", lse_t, torch.float32, (n,))
    if dlogp is not None and dlogits is None:
        dlogits = torch.empty_like(logits)
    if dlogits is not None:
        _check_logits(dlogits, "dlogits")
        if tuple(dlogits.shape) != (n, V):
            _err(f"dlogits has shape {tuple(dlogits.shape)}, expected {(n, V)}")
    _same_device(logits, targets, dlogp, dlogits, lse_t)
    dl_ptr = dlogp.data_ptr() if dlogp is not None else None
    dz_ptr = dlogits.data_ptr() if dlogits is not None else None
    dz_stride = dlogits.stride(0) if dlogits is not None else 0
    with torch.cuda.device(logits.device):
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


def tilemap_entries_bound(prob: Problem) -> int:
    p = prob.c()
    n = _lib.lib().bd_tilemap_entries_bound(ctypes.byref(p))
    if n < 0:
        _err("invalid problem")
    return int(n)


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


def mask_dump(prob: Problem, seq=0, row0=0, n_rows=None):
    """bd_mask_dump (host): uint8 [n_rows, N_seq] numpy array, bit 0 = the row
    view of the kernels' element mask (forward / dQ), bit 1 = the key view (dK/dV)."""
    import numpy as np
    p = prob.c()
    L = _lib.lib()
    nk = ctypes.c_int64(0)
    rc = L.bd_mask_dump(ctypes.byref(p), int(seq), 0, 0, None, 0, ctypes.byref(nk))
    check(rc, "bd_mask_dump")
    if n_rows is None:
        n_rows = nk.value - row0
    out = np.zeros((n_rows, nk.value), dtype=np.uint8)
    check(L.bd_mask_dump(ctypes.byref(p), int(seq), int(row0), int(n_rows), out.ctypes.data, out.size,
                         ctypes.byref(nk)), "bd_mask_dump")
    return out


def logprob_bwd(logits, targets, lse, dlogp, dlogits=None):
    """bd_logprob_bwd: dlogits = dlogp (onehot - softmax) from a known LSE (may be in place)."""
    _check_logits(logits)
    n, V = logits.shape
    _check("targets", targets, torch.int32, (n,))
    _check("lse", lse, torch.float32, (n,))
    _check("dlogp", dlogp, torch.float32, (n,))
    if dlogits is None:
        dlogits = torch.empty_like(logits)
    _check_logits(dlogits, "dlogits")
    if tuple(dlogits.shape) != (n, V):
        _err(f"dlogits has shape {tuple(dlogits.shape)}, expected {(n, V)}")
    _same_device(logits, targets, lse, dlogp, dlogits)
    with torch.cuda.device(logits.device):
        check(_lib.lib().bd_logprob_bwd(n, V, logits.data_ptr(), logits.stride(0), targets.data_ptr(),
                                        lse.data_ptr(), dlogp.data_ptr(), dlogits.data_ptr(), dlogits.stride(0),
                                        _stream_ptr(logits)), "bd_logprob_bwd")
    return dlogits


def lmhead_logprob(h, w, targets, ws=None):
    """bd_lmhead_logprob: (logp, lse) fp32 [n] of softmax(h w^T) at targets, logits never materialised."""
    if h is None or w is None or h.dim() != 2 or w.dim() != 2:
        _err("h [n, C] and w [V, C] must be 2-D")
    n, C = h.shape
    V = w.shape[0]
    _check("h", h, torch.bfloat16, (n, C))
    _check("w", w, torch.bfloat16, (V, C))
    _check("targets", targets, torch.int32, (n,))
    _same_device(h, w, targets)
    logp = torch.empty(n, dtype=torch.float32, device=h.device)
    lse = torch.empty(n, dtype=torch.float32, device=h.device)
    L = _lib.lib()
    with torch.cuda.device(h.device):
        wb = _ws(ws, L.bd_lmhead_workspace_bytes(n, C, V, 0, 0), h.device)
        check(L.bd_lmhead_logprob(n, C, V, h.data_ptr(), w.data_ptr(), targets.data_ptr(), logp.data_ptr(),
                                  lse.data_ptr(), wb.data_ptr(), wb.numel(), _stream_ptr(h)), "bd_lmhead_logprob")
    return logp, lse


def lmhead_logprob_bwd(h, w, targets, lse, dlogp, chunk_rows=16384, dh=None, dw=None, ws=None):
    """bd_lmhead_logprob_bwd: (dh bf16 like h, dw fp32 [V, C]) for upstream dL/dlogp."""
    if h is None or w is None or h.dim() != 2 or w.dim() != 2:
        _err("h [n, C] and w [V, C] must be 2-D")
    n, C = h.shape
    V = w.shape[0]
    _check("h", h, torch.bfloat16, (n, C))
    _check("w", w, torch.bfloat16, (V, C))
    _check("targets", targets, torch.int32, (n,))
    _check("lse", lse, torch.float32, (n,))
    _check("dlogp", dlogp, torch.float32, (n,))
    dh = torch.empty_like(h) if dh is None else dh
    dw = torch.empty((V, C), dtype=torch.float32, device=h.device) if dw is None else dw
    _check("dh", dh, torch.bfloat16, (n, C))
    _check("dw", dw, torch.float32, (V, C))
    _same_device(h, w, targets, lse, dlogp, dh, dw)
    L = _lib.lib()
    with torch.cuda.device(h.device):
        wb = _ws(ws, L.bd_lmhead_workspace_bytes(n, C, V, 1, chunk_rows), h.device)
        check(L.bd_lmhead_logprob_bwd(n, C, V, h.data_ptr(), w.data_ptr(), targets.data_ptr(), lse.data_ptr(),
                                      dlogp.data_ptr(), dh.data_ptr(), dw.data_ptr(), chunk_rows, wb.data_ptr(),
                                      wb.numel(), _stream_ptr(h)), "bd_lmhead_logprob_bwd")
    return dh, dw


def decode_attn(q, k_cache, v_cache, kv_len, softmax_scale=0.0, o=None, lse=None, ws=None):
    """bd_decode_attn: active-block attention over the KV cache -> (o bf16 like q, lse fp32 [b, Hq, B])."""
    if q is None or q.dim() != 4 or k_cache is None or k_cache.dim() != 4:
        _err("q [b, B, Hq, d] and k_cache / v_cache [b, cap, Hkv, d] must be 4-D")
    b, B, Hq, d = q.shape
    _, cap, Hkv, _ = k_cache.shape
    _check("q", q, torch.bfloat16)
    _check("k_cache", k_cache, torch.bfloat16, (b, cap, Hkv, d))
    _check("v_cache", v_cache, torch.bfloat16, (b, cap, Hkv, d))
    _check("kv_len", kv_len, torch.int32, (b,))
    o = torch.empty_like(q) if o is None else o
    lse = torch.empty((b, Hq, B), dtype=torch.float32, device=q.device) if lse is None else lse
    _check("o", o, torch.bfloat16, (b, B, Hq, d))
    _check("lse", lse, torch.float32, (b, Hq, B))
    _same_device(q, k_cache, v_cache, kv_len, o, lse)
    L = _lib.lib()
    with torch.cuda.device(q.device):
        nbytes = L.bd_decode_workspace_bytes(b, B, Hq, Hkv, d, cap)
        wb = _ws(ws, max(nbytes, 256), q.device)
        check(L.bd_decode_attn(b, B, Hq, Hkv, d, cap, float(softmax_scale), q.data_ptr(), k_cache.data_ptr(),
                               v_cache.data_ptr(), kv_len.data_ptr(), o.data_ptr(), lse.data_ptr(), wb.data_ptr(),
                               wb.numel(), _stream_ptr(q)), "bd_decode_attn")
    return o, lse


def decode_select(logits, masked, threshold=0.9):
    """bd_decode_select over bf16 logits [b, B, V] and uint8 masked [b, B] -> (token, conf, commit)."""
    if logits is None or logits.dim() != 3:
        _err("logits must be [b, B, V]")
    b, B, V = logits.shape
    _check("logits", logits, torch.bfloat16)
    _check("masked", masked, torch.uint8, (b, B))
    _same_device(logits, masked)
    token = torch.empty((b, B), dtype=torch.int32, device=logits.device)
    conf = torch.empty((b, B), dtype=torch.float32, device=logits.device)
    commit = torch.empty((b, B), dtype=torch.uint8, device=logits.device)
    with torch.cuda.device(logits.device):
        check(_lib.lib().bd_decode_select(b, B, V, logits.data_ptr(), masked.data_ptr(), float(threshold),
                                          token.data_ptr(), conf.data_ptr(), commit.data_ptr(), _stream_ptr(logits)),
              "bd_decode_select")
    return token, conf, commit


def selftest_gemm(a, b, a_mn=False, b_mn=False):
    """bd_selftest_gemm: fp32 A B^T of the CTA-pair GEMM engine (operands K- or MN-major)."""
    _check("a", a, torch.bfloat16)
    _check("b", b, torch.bfloat16)
    M = a.shape[1] if a_mn else a.shape[0]
    K = a.shape[0] if a_mn else a.shape[1]
    N = b.shape[1] if b_mn else b.shape[0]
    out = torch.empty((M, N), dtype=torch.float32, device=a.device)
    with torch.cuda.device(a.device):
        check(_lib.lib().bd_selftest_gemm(M, N, K, a.data_ptr(), int(a_mn), b.data_ptr(), int(b_mn), out.data_ptr(),
                                          _stream_ptr(a)), "bd_selftest_gemm")
    return out


def launch_count() -> int:
    """Kernels enqueued by libbdattn.so so far (process-wide)."""
    return int(_lib.lib().bd_launch_count())


def dipo_group_stats(rewards, group_of_traj, traj_len, n_groups, out=None):
    """bd_dipo_group_stats: fp64 [n_groups, 3] += (sum r, count, sum |tau|)."""
    n = rewards.numel() if rewards is not None else 0
    _check("rewards", rewards, torch.float32, (n,))
    _check("group_of_traj", group_of_traj, torch.int32, (n,))
    _check("traj_len", traj_len, torch.int32, (n,))
    if out is None:
        out = torch.zeros((n_groups, 3), dtype=torch.float64, device=rewards.device)
    _check("group_stats", out, torch.float64, (n_groups, 3))
    _same_device(rewards, group_of_traj, traj_len, out)
    with torch.cuda.device(rewards.device):
        check(_lib.lib().bd_dipo_group_stats(n, rewards.data_ptr(), group_of_traj.data_ptr(), traj_len.data_ptr(),
                                             n_groups, out.data_ptr(), _stream_ptr(rewards)), "bd_dipo_group_stats")
    return out


def dipo_token_loss(logp, logp_old, traj_of_token, rewards, group_of_traj, group_stats, n_groups_global,
                    eps=0.2, partials=None):
    """bd_dipo_token_loss: returns (dlogp fp32 [n], partials fp64 [3] += (loss, tokens, clipped))."""
    if (logp is None) != (logp_old is None):
        _err("logp and logp_old must both be given or both be None (rho == 1)")
    n = traj_of_token.numel() if traj_of_token is not None else 0
    _check("traj_of_token", traj_of_token, torch.int32, (n,))
    n_traj = rewards.numel() if rewards is not None else 0
    _check("rewards", rewards, torch.float32, (n_traj,))
    _check("group_of_traj", group_of_traj, torch.int32, (n_traj,))
    if group_stats is None or group_stats.dim() != 2:
        _err("group_stats must be fp64 [n_groups, 3]")
    _check("group_stats", group_stats, torch.float64, (group_stats.shape[0], 3))
    if logp is not None:
        _check("logp", logp, torch.float32, (n,))
        _check("logp_old", logp_old, torch.float32, (n,))
    dlogp = torch.empty(n, dtype=torch.float32, device=traj_of_token.device)
    if partials is None:
        partials = torch.zeros(3, dtype=torch.float64, device=traj_of_token.device)
    _check("partials", partials, torch.float64, (3,))
    _same_device(logp, logp_old, traj_of_token, rewards, group_of_traj, group_stats, partials)
    lp = logp.data_ptr() if logp is not None else None
    lo = logp_old.data_ptr() if logp_old is not None else None
    with torch.cuda.device(traj_of_token.device):
        check(_lib.lib().bd_dipo_token_loss(n, lp, lo, traj_of_token.data_ptr(), n_traj, rewards.data_ptr(),
                                            group_of_traj.data_ptr(), group_stats.data_ptr(), group_stats.shape[0],
                                            int(n_groups_global), float(eps), dlogp.data_ptr(), partials.data_ptr(),
                                            _stream_ptr(traj_of_token)), "bd_dipo_token_loss")
    return dlogp, partials
