"""Pins for the trace-replay generalisation of the oracle (S noisy copies,
SURVEY 8(f) NEXT #1, reading c19): packed axis
[x0 | xt^(1) | ... | xt^(S)], copy s = every block's state before decoding
step s (Eq. 6).  CPU only, fp64.

What pins it (none of these re-types the oracle's own predicate):
* brute-force visibility *sets* built by unioning whole blocks (bruteforce.py);
* closed form: pairs = (1 + S) L (L + B) / 2 in DiRL mode;
* S:227's sequential-replay property: the rows of copy s from ONE expanded
  forward equal the single-copy forward over [x0 | copy s] -- and, via
  torch's SDPA, dense attention over exactly x0[0:kB] U (copy s, block k);
* backward linearity: x0-key gradients of the expanded problem are the sum
  over copies of the single-copy gradients minus the (S-1) repeated x0-row
  contributions; torch autograd on the dense formula; finite differences.
"""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import Problem, attention, mask, tilemap
from bruteforce import visibility_sets


def _p(P, R, B, S, rp=1, Hq=1, Hkv=1, d=8, b=1):
    return Problem(b, P, R, B, Hq, Hkv, d, repeat_prompt=rp, n_copies=S)


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


@pytest.mark.parametrize("L,P,B,rp,S", [(L, P, B, rp, S) for B in (1, 2, 4) for L in (B, 3 * B, 12)
                                        if L % B == 0 for P in (0, B) for rp in (0, 1) for S in (2, 3)])
def test_copies_mask_equals_bruteforce_sets(L, P, B, rp, S):
    prob = _p(P, L - P, B, S, rp)
    m = mask.mask_dense(prob)
    _, vis = visibility_sets(L, P, B, rp, n_copies=S)
    assert m.shape == (len(vis), len(vis))
    for n, s in enumerate(vis):
        e = np.zeros(len(vis), bool)
        e[list(s)] = True
        assert np.array_equal(m[n], e), n
    mask.assert_rows_nonempty(m)


@pytest.mark.parametrize("B,K,S", [(1, 5, 2), (2, 4, 3), (4, 3, 4), (4, 2, 1)])
def test_copies_pairs_closed_form(B, K, S):
    L = B * K
    assert mask.mask_dense(_p(B, L - B, B, S)).sum() == (1 + S) * L * (L + B) // 2


def test_single_copy_unchanged():
    for rp in (0, 1):
        a = mask.mask_dense(Problem(1, 4, 8, 2, 1, 1, 8, repeat_prompt=rp))
        b = mask.mask_dense(_p(4, 8, 2, 1, rp))
        assert np.array_equal(a, b)


def _single(prob):
    return Problem(prob.batch, prob.prompt_len, prob.response_len, prob.block_size, prob.n_q_heads,
                   prob.n_kv_heads, prob.head_dim, prob.repeat_prompt, n_copies=1)


def _take(x, idx):
    return np.ascontiguousarray(x[:, idx])


@pytest.mark.parametrize("P,R,B,S,rp", [(4, 12, 4, 3, 1), (8, 16, 4, 2, 0), (0, 24, 8, 2, 1), (6, 18, 3, 4, 1)])
def test_sequential_replay_forward(P, R, B, S, rp):
    """per-copy outputs of one expanded forward == the single-copy
    forward over [x0 | that copy]; and == dense SDPA over the visible keys."""
    prob = _p(P, R, B, S, rp, Hq=2, Hkv=1, d=16)
    N = prob.ntot
    q, k, v = _rand((1, N, 2, 16), 1), _rand((1, N, 1, 16), 2), _rand((1, N, 1, 16), 3)
    o, lse = attention.forward(prob, q, k, v)
    one = _single(prob)
    L, Ln = prob.L, prob.n_noisy
    for s in range(1, S + 1):
        idx = np.concatenate([np.arange(L), L + (s - 1) * Ln + np.arange(Ln)])
        o1, l1 = attention.forward(one, _take(q, idx), _take(k, idx), _take(v, idx))
        np.testing.assert_allclose(o[:, idx], o1, atol=1e-12)
        np.testing.assert_allclose(lse[:, :, idx], l1, atol=1e-12)
        # dense unmasked attention over x0[0:kB] U (copy s, block k)
        for kb in range(prob.xb // B, L // B):
            rows = L + (s - 1) * Ln + np.arange(kb * B, (kb + 1) * B) - prob.xb
            keys = np.concatenate([np.arange(kb * B), rows])
            t = lambda x: torch.from_numpy(np.ascontiguousarray(x))[None, None]
            for h in range(2):
                ref = F.scaled_dot_product_attention(t(q[0, rows, h]), t(k[0, keys, 0]), t(v[0, keys, 0]))
                np.testing.assert_allclose(o[0, rows, h], ref[0, 0].numpy(), atol=1e-12)


@pytest.mark.parametrize("S", [2, 3])
def test_sequential_replay_backward(S):
    """Gradients by linearity over copies: copy rows' dQ and copy keys' dK/dV
    equal the single-copy problem's; x0 keys collect every copy's
    contribution once and the x0 rows' contribution once."""
    prob = _p(4, 12, 4, S, 1, Hq=2, Hkv=1, d=8)
    N, L, Ln = prob.ntot, prob.L, prob.n_noisy
    q, k, v, do = (_rand((1, N, 2, 8), 11), _rand((1, N, 1, 8), 12), _rand((1, N, 1, 8), 13),
                   _rand((1, N, 2, 8), 14))
    dq, dk, dv = attention.backward(prob, q, k, v, do)
    one = _single(prob)
    dk_x0 = np.zeros_like(dk[:, :L])
    dv_x0 = np.zeros_like(dv[:, :L])
    for s in range(1, S + 1):
        idx = np.concatenate([np.arange(L), L + (s - 1) * Ln + np.arange(Ln)])
        dq1, dk1, dv1 = attention.backward(one, _take(q, idx), _take(k, idx), _take(v, idx), _take(do, idx))
        np.testing.assert_allclose(dq[:, idx], dq1, atol=1e-12)
        np.testing.assert_allclose(dk[:, idx[L:]], dk1[:, L:], atol=1e-12)
        np.testing.assert_allclose(dv[:, idx[L:]], dv1[:, L:], atol=1e-12)
        dk_x0 += dk1[:, :L]
        dv_x0 += dv1[:, :L]
    # the x0 rows' own contribution (dO zero on the noisy rows) was counted S times
    idx = np.concatenate([np.arange(L), L + np.arange(Ln)])
    do_x0only = _take(do, idx)
    do_x0only[:, L:] = 0
    _, dk0, dv0 = attention.backward(one, _take(q, idx), _take(k, idx), _take(v, idx), do_x0only)
    np.testing.assert_allclose(dk[:, :L], dk_x0 - (S - 1) * dk0[:, :L], atol=1e-11)
    np.testing.assert_allclose(dv[:, :L], dv_x0 - (S - 1) * dv0[:, :L], atol=1e-11)


def test_copies_backward_vs_autograd_and_fd():
    prob = _p(2, 6, 2, 2, 1, Hq=2, Hkv=1, d=4)
    N = prob.ntot
    q, k, v, do = (_rand((1, N, 2, 4), 21), _rand((1, N, 1, 4), 22), _rand((1, N, 1, 4), 23),
                   _rand((1, N, 2, 4), 24))
    dq, dk, dv = attention.backward(prob, q, k, v, do)
    m = torch.from_numpy(mask.mask_dense(prob))
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (q, k, v))
    s = torch.einsum("nhd,mhd->hnm", tq[0], tk[0].repeat_interleave(2, 1)) * prob.scale
    s = s.masked_fill(~m, float("-inf"))
    o = torch.einsum("hnm,mhd->nhd", torch.softmax(s, -1), tv[0].repeat_interleave(2, 1))
    (o * torch.from_numpy(do[0])).sum().backward()
    np.testing.assert_allclose(dq, tq.grad.numpy(), atol=1e-12)
    np.testing.assert_allclose(dk, tk.grad.numpy(), atol=1e-12)
    np.testing.assert_allclose(dv, tv.grad.numpy(), atol=1e-12)
    # central finite differences on a few k entries (shared x0 keys)
    h = 1e-6
    for (n, c) in [(0, 1), (3, 2), (prob.L + 1, 0), (N - 1, 3)]:
        kp, km = k.copy(), k.copy()
        kp[0, n, 0, c] += h
        km[0, n, 0, c] -= h
        fp = (attention.forward(prob, q, kp, v)[0] * do).sum()
        fm = (attention.forward(prob, q, km, v)[0] * do).sum()
        assert abs((fp - fm) / (2 * h) - dk[0, n, 0, c]) < 1e-6 * max(1.0, abs(dk[0, n, 0, c]))


@pytest.mark.parametrize("L,B,S", [(384, 4, 2), (256, 8, 3), (200, 4, 2)])
def test_copies_tile_counts(L, B, S):
    """Closed form for L % 128 == 0, B < 128: x0 q-tile i lists i+1 tiles, a
    copy's q-tile i lists i+1 x0 tiles + its own diagonal tile; partial =
    the x0 diagonal (T) + per copy the x0 diagonal and the own tile (2T).
    Ragged L: every q-tile still lists >= 1 tile, EMPTY copy-to-copy tiles."""
    prob = _p(0, L, B, S)
    c = tilemap.classify(prob)
    T = -(-L // 128)
    for e in c:
        if e[0] >= 1 and e[2] >= 1:
            assert e[0] == e[2]  # never across copies
    if L % 128 == 0:
        assert len(c) == T * (T + 1) // 2 + S * (T * (T + 1) // 2 + T)
        assert sum(1 for e in c if e[4] == tilemap.PARTIAL) == T + 2 * S * T
