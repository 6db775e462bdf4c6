"""Pins for oracle/lmhead.py (CPU only): closed forms, invariances, torch fp64
autograd and central finite differences -- none re-types the oracle."""

import math

import numpy as np
import torch

from oracle import lmhead, logprob


def _case(seed, N=5, C=7, V=11):
    g = np.random.default_rng(seed)
    return (g.standard_normal((N, C)), g.standard_normal((V, C)) * 0.7, g.integers(0, V, N),
            g.standard_normal(N))


def test_zero_hidden_closed_form():
    """h = 0 -> uniform softmax: logp = -ln V, dh_n = w_n (W[t_n] - mean_v W_v), dW = 0."""
    _, W, t, w = _case(0)
    h = np.zeros((5, 7))
    lp, lse = lmhead.lmhead_logprob(h, W, t)
    np.testing.assert_allclose(lp, -math.log(11), rtol=1e-14)
    dh, dW = lmhead.lmhead_logprob_grad(h, W, t, w)
    np.testing.assert_allclose(dh, w[:, None] * (W[t] - W.mean(0)[None]), atol=1e-14)
    assert np.abs(dW).max() == 0.0


def test_one_hot_weights_select_hidden_columns():
    """W rows = unit vectors e_{c(v)}: z[n, v] = h[n, c(v)], so the result is the
    (separately pinned) log-softmax of selected hidden columns -- no matmul."""
    h, _, _, _ = _case(1, C=9)
    cols = np.array([3, 0, 8, 8, 5, 1])
    W = np.eye(9)[cols]
    t = np.array([0, 2, 5, 3, 1])
    lp, _ = lmhead.lmhead_logprob(h, W, t)
    ref, _ = logprob.logprob(h[:, cols], t)
    np.testing.assert_allclose(lp, ref, atol=1e-14)


def test_row_shift_invariance():
    """Adding one vector u to every vocabulary row shifts row n's logits by h_n.u:
    log-probs unchanged, dh changes by exactly 0 (sum_v dz = 0), dW unchanged."""
    h, W, t, w = _case(2)
    u = np.random.default_rng(9).standard_normal(7)
    lp0, _ = lmhead.lmhead_logprob(h, W, t)
    lp1, _ = lmhead.lmhead_logprob(h, W + u[None], t)
    np.testing.assert_allclose(lp1, lp0, atol=1e-12)
    dh0, dW0 = lmhead.lmhead_logprob_grad(h, W, t, w)
    dh1, dW1 = lmhead.lmhead_logprob_grad(h, W + u[None], t, w)
    np.testing.assert_allclose(dh1, dh0, atol=1e-12)
    np.testing.assert_allclose(dW1, dW0, atol=1e-12)


def test_dw_rows_sum_to_zero():
    """sum_v dW_v = (sum_v dz_{n,v}) h_n summed over n = 0."""
    h, W, t, w = _case(3, N=8, V=13)
    _, dW = lmhead.lmhead_logprob_grad(h, W, t, w)
    np.testing.assert_allclose(dW.sum(0), 0.0, atol=1e-13)


def test_vs_torch_autograd():
    h, W, t, w = _case(4, N=6, C=10, V=17)
    th = torch.from_numpy(h).requires_grad_()
    tW = torch.from_numpy(W).requires_grad_()
    lp = torch.log_softmax(torch.nn.functional.linear(th, tW), -1)[torch.arange(6), torch.from_numpy(t)]
    lp.backward(torch.from_numpy(w))
    got, _ = lmhead.lmhead_logprob(h, W, t)
    np.testing.assert_allclose(got, lp.detach().numpy(), atol=1e-13)
    dh, dW = lmhead.lmhead_logprob_grad(h, W, t, w)
    np.testing.assert_allclose(dh, th.grad.numpy(), atol=1e-13)
    np.testing.assert_allclose(dW, tW.grad.numpy(), atol=1e-13)


def test_finite_differences():
    """Central differences of L = sum_n w_n logp_n, h = 1e-6."""
    h, W, t, w = _case(5, N=3, C=4, V=6)
    dh, dW = lmhead.lmhead_logprob_grad(h, W, t, w)
    L = lambda hh, WW: float(np.dot(w, lmhead.lmhead_logprob(hh, WW, t)[0]))
    eps = 1e-6
    for X, G, is_h in ((h, dh, True), (W, dW, False)):
        num = np.zeros_like(X)
        for idx in np.ndindex(X.shape):
            Xp, Xm = X.copy(), X.copy()
            Xp[idx] += eps
            Xm[idx] -= eps
            num[idx] = ((L(Xp, W) - L(Xm, W)) if is_h else (L(h, Xp) - L(h, Xm))) / (2 * eps)
        assert np.abs(num - G).max() / np.abs(G).max() < 1e-6


def test_brute_force_loops():
    """Tiny case with scalar Python loops (math.fsum): logits, log-sum-exp."""
    h, W, t, _ = _case(6, N=2, C=3, V=4)
    lp, lse = lmhead.lmhead_logprob(h, W, t)
    for n in range(2):
        z = [math.fsum(h[n, c] * W[v, c] for c in range(3)) for v in range(4)]
        s = math.log(math.fsum(math.exp(x) for x in z))
        assert abs(lse[n] - s) < 1e-13 and abs(lp[n] - (z[t[n]] - s)) < 1e-13


def test_shape_errors():
    import pytest
    with pytest.raises(ValueError):
        lmhead.logits(np.zeros((2, 3)), np.zeros((4, 5)))
    with pytest.raises(IndexError):
        lmhead.lmhead_logprob(np.zeros((1, 3)), np.zeros((4, 3)), [4])
