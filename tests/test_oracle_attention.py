"""Pins for oracle/attention.py (CPU only, fp64)."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import Problem, attention, mask


def _rand(shape, seed, scale=1.0):
    g = np.random.default_rng(seed)
    return g.standard_normal(shape) * scale


def _inputs(prob, seed=0, qscale=1.0):
    N = prob.ntot
    q = _rand((prob.batch, N, prob.n_q_heads, prob.head_dim), seed, qscale)
    k = _rand((prob.batch, N, prob.n_kv_heads, prob.head_dim), seed + 1)
    v = _rand((prob.batch, N, prob.n_kv_heads, prob.head_dim), seed + 2)
    do = _rand((prob.batch, N, prob.n_q_heads, prob.head_dim), seed + 3)
    return q, k, v, do


def _sdpa(q, k, v, attn_mask=None, is_causal=False, scale=None):
    """torch float64 SDPA on [N, d] matrices (library routine)."""
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x))[None, None]
    m = None if attn_mask is None else torch.from_numpy(attn_mask)[None, None]
    out = F.scaled_dot_product_attention(t(q), t(k), t(v), attn_mask=m, is_causal=is_causal,
                                         scale=scale)
    return out[0, 0].numpy()


def test_block1_empty_xt_is_causal():
    """North star pin: block_size=1 with an empty xt reduces to causal
    attention (response-only mode, R=0)."""
    prob = Problem(1, 24, 0, 1, 2, 1, 16, repeat_prompt=0)
    assert prob.ntot == 24
    q, k, v, _ = _inputs(prob)
    o, _ = attention.forward(prob, q, k, v)
    for h in range(2):
        ref = _sdpa(q[0, :, h], k[0, :, 0], v[0, :, 0], is_causal=True)
        np.testing.assert_allclose(o[0, :, h], ref, rtol=1e-12, atol=1e-12)


def test_single_block_no_prompt_is_bidirectional():
    """K=1, no prompt: x0 rows = non-causal SDPA over x0, xt rows = non-causal
    SDPA over xt."""
    B = 8
    prob = Problem(1, 0, B, B, 1, 1, 16)
    q, k, v, _ = _inputs(prob, 3)
    o, _ = attention.forward(prob, q, k, v)
    np.testing.assert_allclose(o[0, :B, 0], _sdpa(q[0, :B, 0], k[0, :B, 0], v[0, :B, 0]), atol=1e-12)
    np.testing.assert_allclose(o[0, B:, 0], _sdpa(q[0, B:, 0], k[0, B:, 0], v[0, B:, 0]), atol=1e-12)


@pytest.mark.parametrize("P,R,B,rp", [(4, 12, 4, 1), (8, 16, 4, 0), (0, 24, 8, 1), (6, 18, 3, 1)])
def test_slice_and_recompute(P, R, B, rp):
    """S:59 / S:234: each noisy block k equals dense unmasked attention over
    exactly x0[0:kB] U xt[block k]; each clean block k over x0[0:(k+1)B]."""
    prob = Problem(1, P, R, B, 2, 2, 16, repeat_prompt=rp)
    q, k, v, _ = _inputs(prob, 7)
    o, lse = attention.forward(prob, q, k, v)
    L, xb = prob.L, prob.xb
    for h in range(2):
        for kb in range(L // B):
            rows0 = np.arange(kb * B, (kb + 1) * B)
            keys0 = np.arange(0, (kb + 1) * B)
            ref = _sdpa(q[0, rows0, h], k[0, keys0, h], v[0, keys0, h])
            np.testing.assert_allclose(o[0, rows0, h], ref, atol=1e-12)
            pos = np.arange(kb * B, (kb + 1) * B)
            pos = pos[pos >= xb]
            if pos.size == 0:
                continue
            rows1 = L + pos - xb
            keys1 = np.concatenate([np.arange(0, kb * B), rows1])
            ref = _sdpa(q[0, rows1, h], k[0, keys1, h], v[0, keys1, h])
            np.testing.assert_allclose(o[0, rows1, h], ref, atol=1e-12)
            # LSE over the same visible keys, by direct logsumexp
            s = prob.scale * q[0, rows1, h] @ k[0, keys1, h].T
            ref_lse = np.log(np.exp(s - s.max(1, keepdims=True)).sum(1)) + s.max(1)
            np.testing.assert_allclose(lse[0, h, rows1], ref_lse, atol=1e-12)


def test_general_vs_torch_sdpa_with_bool_mask():
    prob = Problem(2, 5, 15, 5, 4, 2, 8)
    q, k, v, _ = _inputs(prob, 11, qscale=3.0)
    o, _ = attention.forward(prob, q, k, v)
    m = mask.mask_dense(prob)
    for b in range(2):
        for h in range(4):
            ref = _sdpa(q[b, :, h], k[b, :, h // 2], v[b, :, h // 2], attn_mask=m)
            np.testing.assert_allclose(o[b, :, h], ref, atol=1e-12)


def test_softmax_invariants():
    """rows sum to 1 (v = 1 -> O = 1); invariance to adding one vector
    c to every key (adds q.c to a whole row)."""
    prob = Problem(1, 4, 12, 4, 2, 1, 8)
    q, k, v, _ = _inputs(prob, 5)
    ones = np.ones_like(v)
    o1, _ = attention.forward(prob, q, k, ones)
    np.testing.assert_allclose(o1, 1.0, atol=1e-13)
    c = _rand((8,), 99)
    o_a, lse_a = attention.forward(prob, q, k, v)
    o_b, lse_b = attention.forward(prob, q, k + c, v)
    np.testing.assert_allclose(o_a, o_b, atol=1e-12)
    shift = prob.scale * np.einsum("bnhd,d->bhn", q, c)
    np.testing.assert_allclose(lse_b - lse_a, shift, atol=1e-12)


def test_x0_independent_of_xt():
    """clean rows see only clean keys -> x0 outputs bitwise-unchanged
    when xt inputs are perturbed."""
    prob = Problem(1, 8, 16, 4, 2, 2, 8)
    q, k, v, _ = _inputs(prob, 2)
    o_a, lse_a = attention.forward(prob, q, k, v)
    q2, k2, v2 = q.copy(), k.copy(), v.copy()
    L = prob.L
    for x in (q2, k2, v2):
        x[:, L:] += 1.0
    o_b, lse_b = attention.forward(prob, q2, k2, v2)
    assert np.array_equal(o_a[:, :L], o_b[:, :L])
    assert np.array_equal(lse_a[:, :, :L], lse_b[:, :, :L])


def test_gqa_equals_repeated_mha():
    prob = Problem(1, 4, 8, 2, 4, 2, 8)
    q, k, v, do = _inputs(prob, 21)
    o, lse = attention.forward(prob, q, k, v)
    mha = Problem(1, 4, 8, 2, 4, 4, 8)
    kr, vr = np.repeat(k, 2, axis=2), np.repeat(v, 2, axis=2)
    o2, lse2 = attention.forward(mha, q, kr, vr)
    np.testing.assert_allclose(o, o2, atol=1e-13)
    dq, dk, dv = attention.backward(prob, q, k, v, do)
    dq2, dk2, dv2 = attention.backward(mha, q, kr, vr, do)
    np.testing.assert_allclose(dq, dq2, atol=1e-12)
    np.testing.assert_allclose(dk, dk2.reshape(1, prob.ntot, 2, 2, 8).sum(3), atol=1e-12)
    np.testing.assert_allclose(dv, dv2.reshape(1, prob.ntot, 2, 2, 8).sum(3), atol=1e-12)


# ---------------------------------------------------------------- backward


def test_backward_finite_differences():
    """S:89 / S:620 analytic gradient vs central finite differences; fp64,
    h = 1e-6, relative error < 1e-6."""
    prob = Problem(1, 2, 6, 2, 2, 1, 4)
    q, k, v, _ = _inputs(prob, 31)
    W = _rand(q.shape, 77)  # loss = sum(O * W)  ->  dO = W
    dq, dk, dv = attention.backward(prob, q, k, v, W)

    def loss(qq, kk, vv):
        o, _ = attention.forward(prob, qq, kk, vv)
        return float((o * W).sum())

    h = 1e-6
    for name, x, g in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
        num = np.zeros_like(x)
        it = np.nditer(x, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            xp, xm = x.copy(), x.copy()
            xp[idx] += h
            xm[idx] -= h
            args = {"q": (q, k, v), "k": (q, k, v), "v": (q, k, v)}[name]
            ap = list(args)
            am = list(args)
            pos = "qkv".index(name)
            ap[pos], am[pos] = xp, xm
            num[idx] = (loss(*ap) - loss(*am)) / (2 * h)
        rel = np.linalg.norm(num - g) / np.linalg.norm(g)
        assert rel < 1e-6, (name, rel)


def test_backward_vs_torch_autograd():
    """Gradients vs torch float64 autograd through SDPA with the bool mask."""
    prob = Problem(1, 4, 12, 4, 4, 2, 8)
    q, k, v, do = _inputs(prob, 41, qscale=2.0)
    dq, dk, dv = attention.backward(prob, q, k, v, do)
    m = torch.from_numpy(mask.mask_dense(prob))
    tq = torch.from_numpy(q).permute(0, 2, 1, 3).requires_grad_()
    tk = torch.from_numpy(k).permute(0, 2, 1, 3).requires_grad_()
    tv = torch.from_numpy(v).permute(0, 2, 1, 3).requires_grad_()
    o = F.scaled_dot_product_attention(tq, tk.repeat_interleave(2, 1), tv.repeat_interleave(2, 1),
                                       attn_mask=m)
    o.backward(torch.from_numpy(do).permute(0, 2, 1, 3))
    np.testing.assert_allclose(dq, tq.grad.permute(0, 2, 1, 3).numpy(), atol=1e-11)
    np.testing.assert_allclose(dk, tk.grad.permute(0, 2, 1, 3).numpy(), atol=1e-11)
    np.testing.assert_allclose(dv, tv.grad.permute(0, 2, 1, 3).numpy(), atol=1e-11)


def test_backward_invariants():
    """sum_j dK_j = 0 per head (since sum_j dS_ij = 0); dQ of x0 rows never
    depends on xt inputs."""
    prob = Problem(1, 4, 12, 4, 2, 2, 8)
    q, k, v, do = _inputs(prob, 51)
    dq, dk, dv = attention.backward(prob, q, k, v, do)
    np.testing.assert_allclose(dk.sum(axis=1), 0.0, atol=1e-12)
    L = prob.L
    q2, k2, v2 = q.copy(), k.copy(), v.copy()
    for x in (q2, k2, v2):
        x[:, L:] -= 0.5
    dq2, _, _ = attention.backward(prob, q2, k2, v2, do)
    assert np.array_equal(dq[:, :L], dq2[:, :L])


def test_backward_slice_matches_full():
    prob = Problem(2, 4, 8, 4, 4, 2, 8)
    q, k, v, do = _inputs(prob, 61)
    dq, dk, dv = attention.backward(prob, q, k, v, do)
    o, lse = attention.forward(prob, q, k, v)
    sdq, sdk, sdv, so, slse = attention.backward_slice(prob, q, k, v, do, 1, 1)
    np.testing.assert_allclose(sdq, dq[1, :, 2:4], atol=0)
    np.testing.assert_allclose(sdk, dk[1, :, 1], atol=0)
    np.testing.assert_allclose(so, o[1, :, 2:4], atol=1e-14)
    np.testing.assert_allclose(slse, lse[1, 2:4], atol=1e-14)


def test_backward_rows_sum_to_full():
    """backward_rows over a partition of the rows adds up to backward_slice."""
    prob = Problem(1, 4, 12, 4, 2, 1, 8)
    q, k, v, do = _inputs(prob, 71)
    dq, dk, dv, _, _ = attention.backward_slice(prob, q, k, v, do, 0, 0)
    acc_k = np.zeros_like(dk)
    acc_v = np.zeros_like(dv)
    for h in range(2):
        for rows in (np.arange(0, 13), np.arange(13, prob.ntot)):
            dqr, dkp, dvp = attention.backward_rows(prob, q, k, v, do, 0, h, rows)
            np.testing.assert_allclose(dqr, dq[rows, h], atol=1e-13)
            acc_k += dkp
            acc_v += dvp
    np.testing.assert_allclose(acc_k, dk, atol=1e-12)
    np.testing.assert_allclose(acc_v, dv, atol=1e-12)
