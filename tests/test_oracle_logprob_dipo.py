"""Pins for oracle/logprob.py and oracle/dipo.py (CPU only)."""

import math

import numpy as np
import pytest
import torch

from oracle import logprob, dipo


def test_uniform_logits():
    """S:75 uniform logits -> CE = ln V, i.e. logp = -ln V."""
    for V in (4, 1024, 151_936):
        z = np.full((3, V), 2.5)
        lp, lse = logprob.logprob(z, [0, V // 2, V - 1])
        np.testing.assert_allclose(lp, -math.log(V), rtol=1e-13)
        np.testing.assert_allclose(lse, 2.5 + math.log(V), rtol=1e-13)


def test_vs_torch_log_softmax_and_autograd():
    g = np.random.default_rng(0)
    z = g.standard_normal((6, 11)) * 3
    t = g.integers(0, 11, 6)
    w = g.standard_normal(6)
    lp, _ = logprob.logprob(z, t)
    tz = torch.from_numpy(z).requires_grad_()
    ref = torch.log_softmax(tz, -1)[torch.arange(6), torch.from_numpy(t)]
    np.testing.assert_allclose(lp, ref.detach().numpy(), atol=1e-13)
    ref.backward(torch.from_numpy(w))
    dz = logprob.logprob_grad(z, t, w)
    np.testing.assert_allclose(dz, tz.grad.numpy(), atol=1e-13)
    np.testing.assert_allclose(dz.sum(1), 0.0, atol=1e-13)  # sum_v dz = 0


def test_one_hot_limit():
    """S:76 one-hot logit magnitude -> loss -> 0."""
    z = np.zeros((1, 8))
    z[0, 3] = 60.0
    lp, _ = logprob.logprob(z, [3])
    assert abs(lp[0]) < 1e-20


def test_target_out_of_range():
    with pytest.raises(IndexError):
        logprob.logprob(np.zeros((2, 4)), [0, 4])


# -------------------------------------------------------------------- DiPO


def test_advantages():
    """S:466-470 examples."""
    np.testing.assert_array_equal(dipo.advantages([1, 1, 1, 1], [0, 0, 0, 0]), [0, 0, 0, 0])
    np.testing.assert_array_equal(dipo.advantages([1, 0], [0, 0]), [0.5, -0.5])
    r = np.random.default_rng(1).random(16)
    a = dipo.advantages(r, np.repeat(np.arange(4), 4))
    np.testing.assert_allclose(a.reshape(4, 4).sum(1), 0.0, atol=1e-15)


def test_reinforce_toy_hand_computed():
    """rho = 1 -> gradient = (1/sum|tau|) sum_i sum_k A_i grad logp.
    Toy: one group, rewards [1, 0], lengths [2, 3]: A = [0.5, -0.5], N_g = 5,
    dloss/dlogp = -A_i/5 = [-0.1, -0.1, 0.1, 0.1, 0.1]; loss = -(0.5*2 - 0.5*3)/5 = 0.1."""
    logp = np.array([-1.0, -2.0, -0.5, -0.7, -3.0])
    loss, dl, st = dipo.dipo_loss(logp, logp.copy(), [0, 0, 1, 1, 1], [1.0, 0.0], [0, 0])
    assert abs(loss - 0.1) < 1e-15
    np.testing.assert_allclose(dl, [-0.1, -0.1, 0.1, 0.1, 0.1], atol=1e-15)
    assert st["clip_frac"] == 0.0


def test_two_groups_mean_over_groups():
    """Reading c11: per-group token normaliser, then mean over groups."""
    logp = np.zeros(5)
    # group 0: trajs 0,1 (rewards 1,0) lengths 1,1 ; group 1: trajs 2,3 (0,1) lengths 1,2
    loss, dl, st = dipo.dipo_loss(logp, logp, [0, 1, 2, 3, 3], [1, 0, 0, 1], [0, 0, 1, 1])
    # group0: A=[.5,-.5], N=2 -> J0 = (0.5-0.5)/2 = 0 ; grads -A/(2*2) = [-.125, .125]
    # group1: A=[-.5,.5], N=3 -> J1 = (-0.5 + 2*0.5)/3 = 1/6 ; grads -A/(3*2)
    assert abs(loss - (-(0 + 1 / 6) / 2)) < 1e-15
    np.testing.assert_allclose(dl, [-0.125, 0.125, 0.5 / 6, -0.5 / 6, -0.5 / 6], atol=1e-15)
    assert st["n_groups"] == 2 and st["n_tokens"] == 5


def test_zero_advantage_zero_gradient():
    """S:476 all A_i = 0 -> gradient exactly 0."""
    logp = np.random.default_rng(2).standard_normal(7)
    _, dl, _ = dipo.dipo_loss(logp, logp, [0, 0, 1, 1, 1, 2, 2], [1, 1, 1], [0, 0, 0])
    assert np.all(dl == 0)


def test_gradient_matches_finite_difference_and_clip():
    """dloss/dlogp vs central differences of the loss (logp_old fixed = sg),
    both at rho = 1 and with rho outside the clip range (gradient 0 there)."""
    g = np.random.default_rng(3)
    logp = g.standard_normal(6)
    old = logp.copy()
    old[0] -= math.log(1.5)   # rho_0 = 1.5 > 1 + eps
    old[4] += math.log(2.0)   # rho_4 = 0.5 < 1 - eps
    tt = [0, 0, 1, 1, 2, 2]
    r = [1.0, 0.0, 0.5]
    gr = [0, 0, 0]
    loss, dl, st = dipo.dipo_loss(logp, old, tt, r, gr)
    h = 1e-7
    for i in range(6):
        lp, lm = logp.copy(), logp.copy()
        lp[i] += h
        lm[i] -= h
        num = (dipo.dipo_loss(lp, old, tt, r, gr)[0] - dipo.dipo_loss(lm, old, tt, r, gr)[0]) / (2 * h)
        assert abs(num - dl[i]) < 1e-7, (i, num, dl[i])
    adv = dipo.advantages(r, gr)
    assert adv[0] > 0 and dl[0] == 0.0  # A>0, rho clipped from above
    assert st["clip_frac"] > 0


def test_nonfinite_ratio_aborts():
    with pytest.raises(FloatingPointError):
        dipo.dipo_loss([0.0, np.inf], [0.0, 0.0], [0, 0], [1.0], [0])
