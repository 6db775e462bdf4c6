"""Naive masked softmax attention and its analytic gradient, fp64.

Definition (S:51-55 ``masked_attention``: "softmax(qk^T/sqrt(d) + bias) v where
bias = -inf at masked-out pairs"; the mask is ``oracle.mask`` built from the
paper's rule):

    S_ij   = scale * q_i . k_j          for M_ij, -inf otherwise
    m_i    = max_j S_ij,  l_i = sum_j exp(S_ij - m_i)
    P_ij   = exp(S_ij - m_i) / l_i
    O_i    = sum_j P_ij v_j
    LSE_i  = m_i + ln l_i                (natural log, reading c6)

Backward, given dO (chain rule through the softmax Jacobian, "analytic
gradient matches central finite differences"):

    dP_ij  = dO_i . v_j
    dS_ij  = P_ij (dP_ij - sum_l P_il dP_il)
    dQ_i   = scale * sum_j dS_ij k_j
    dK_j   = scale * sum_{h in group} sum_i dS_ij q_i
    dV_j   = sum_{h in group} sum_i P_ij dO_i

GQA mapping kv(h) = h // (Hq/Hkv) (reading c7).  Layouts match the ABI:
q/o [b, Ntot, Hq, d], k/v [b, Ntot, Hkv, d], lse [b, Hq, Ntot].

Inputs may be any float dtype; they are upcast to fp64 exactly (reading c8:
the reference is always fp64 on the upcast bf16 inputs).  Rows are processed
in chunks only to bound memory -- each chunk is the same dense formula.

ORACLE: test infrastructure only (see oracle/__init__.py).
"""

import numpy as np

from .problem import Problem
from .mask import mask_rows, assert_rows_nonempty

_CHUNK_ELEMS = 1 << 23


def _f64(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float64)


def _chunks(n_rows: int, n_cols: int):
    step = max(1, _CHUNK_ELEMS // max(1, n_cols))
    for r0 in range(0, n_rows, step):
        yield r0, min(n_rows, r0 + step)


def forward_rows(prob: Problem, q, k, v, b: int, h: int, rows):
    """O and LSE for query rows ``rows`` of sequence b, q-head h.

    Returns (O [len(rows), d] fp64, LSE [len(rows)] fp64)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    g = prob.kv_head_of(h)
    rows = np.asarray(rows, dtype=np.int64)
    kg = k[b, :, g, :]
    vg = v[b, :, g, :]
    outs, lses = [], []
    for r0, r1 in _chunks(len(rows), prob.ntot):
        rr = rows[r0:r1]
        m = mask_rows(prob, rr)
        assert_rows_nonempty(m)
        s = prob.scale * (q[b, rr, h, :] @ kg.T)
        s = np.where(m, s, -np.inf)
        mx = s.max(axis=1, keepdims=True)
        e = np.exp(s - mx)
        l = e.sum(axis=1, keepdims=True)
        p = e / l
        outs.append(p @ vg)
        lses.append((mx + np.log(l))[:, 0])
    return np.concatenate(outs, 0), np.concatenate(lses, 0)


def forward(prob: Problem, q, k, v):
    """Full forward: O [b, Ntot, Hq, d], LSE [b, Hq, Ntot] (fp64)."""
    prob.validate()
    q, k, v = _f64(q), _f64(k), _f64(v)
    b_, N, Hq, d = q.shape
    o = np.empty((b_, N, Hq, d))
    lse = np.empty((b_, Hq, N))
    rows = np.arange(N)
    for b in range(b_):
        for h in range(Hq):
            o[b, :, h, :], lse[b, h, :] = forward_rows(prob, q, k, v, b, h, rows)
    return o, lse


def backward_slice(prob: Problem, q, k, v, do, b: int, g: int):
    """Gradients of one independent (sequence b, kv-head g) slice.

    Returns (dq [Ntot, group, d], dk [Ntot, d], dv [Ntot, d], o [Ntot, group, d],
    lse [group, Ntot]) -- dq/o for the q-heads h = g*group .. g*group+group-1."""
    q, k, v, do = _f64(q), _f64(k), _f64(v), _f64(do)
    N, d, G = prob.ntot, prob.head_dim, prob.group
    kg = k[b, :, g, :]
    vg = v[b, :, g, :]
    dq = np.zeros((N, G, d))
    o = np.zeros((N, G, d))
    lse = np.zeros((G, N))
    dk = np.zeros((N, d))
    dv = np.zeros((N, d))
    for hh in range(G):
        h = g * G + hh
        for r0, r1 in _chunks(N, N):
            rr = np.arange(r0, r1)
            m = mask_rows(prob, rr)
            assert_rows_nonempty(m)
            s = prob.scale * (q[b, rr, h, :] @ kg.T)
            s = np.where(m, s, -np.inf)
            mx = s.max(axis=1, keepdims=True)
            e = np.exp(s - mx)
            l = e.sum(axis=1, keepdims=True)
            p = e / l
            o[rr, hh, :] = p @ vg
            lse[hh, rr] = (mx + np.log(l))[:, 0]
            dO = do[b, rr, h, :]
            dp = dO @ vg.T
            ds = p * (dp - (p * dp).sum(axis=1, keepdims=True))
            dq[rr, hh, :] = prob.scale * (ds @ kg)
            dk += prob.scale * (ds.T @ q[b, rr, h, :])
            dv += p.T @ dO
    return dq, dk, dv, o, lse


def backward_rows(prob: Problem, q, k, v, do, b: int, h: int, rows):
    """The same dense backward restricted to query rows ``rows`` of (b, h):
    returns (dq[rows] [n, d], dk_part [Ntot, d], dv_part [Ntot, d]) where the
    parts are those rows' contributions to dK / dV.  Used for bounded CPU
    baselines and sampled parity at full size."""
    q, k, v, do = _f64(q), _f64(k), _f64(v), _f64(do)
    g = prob.kv_head_of(h)
    rows = np.asarray(rows, dtype=np.int64)
    kg, vg = k[b, :, g, :], v[b, :, g, :]
    N, d = prob.ntot, prob.head_dim
    dq = np.zeros((len(rows), d))
    dk = np.zeros((N, d))
    dv = np.zeros((N, d))
    for r0, r1 in _chunks(len(rows), N):
        rr = rows[r0:r1]
        m = mask_rows(prob, rr)
        assert_rows_nonempty(m)
        s = prob.scale * (q[b, rr, h, :] @ kg.T)
        s = np.where(m, s, -np.inf)
        mx = s.max(axis=1, keepdims=True)
        e = np.exp(s - mx)
        p = e / e.sum(axis=1, keepdims=True)
        dO = do[b, rr, h, :]
        dp = dO @ vg.T
        ds = p * (dp - (p * dp).sum(axis=1, keepdims=True))
        dq[r0:r1] = prob.scale * (ds @ kg)
        dk += prob.scale * (ds.T @ q[b, rr, h, :])
        dv += p.T @ dO
    return dq, dk, dv


def backward(prob: Problem, q, k, v, do):
    """Full backward: dq like q, dk/dv like k (fp64)."""
    prob.validate()
    q = _f64(q)
    b_, N, Hq, d = q.shape
    Hkv = prob.n_kv_heads
    dq = np.zeros((b_, N, Hq, d))
    dk = np.zeros((b_, N, Hkv, d))
    dv = np.zeros((b_, N, Hkv, d))
    G = prob.group
    for b in range(b_):
        for g in range(Hkv):
            sdq, sdk, sdv, _, _ = backward_slice(prob, q, k, v, do, b, g)
            dq[b, :, g * G:(g + 1) * G, :] = sdq
            dk[b, :, g, :] = sdk
            dv[b, :, g, :] = sdv
    return dq, dk, dv
