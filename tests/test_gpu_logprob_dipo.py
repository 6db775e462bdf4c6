"""GPU parity of bd_logprob / bd_logprob_bwd / DiPO kernels vs the fp64 oracle."""

import numpy as np
import pytest
import torch

import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import ops, dipo as bdipo
from oracle import logprob as olp, dipo as odipo
from parity import LOGP_MAX_ABS, DZ_REL_L2, metrics, t2np
from workloads import logits_inputs, rl_batch, VOCAB_QWEN3


@pytest.mark.gpu
@pytest.mark.parametrize("n,V,peaked", [(64, 1024, False), (64, VOCAB_QWEN3, False), (33, VOCAB_QWEN3, True),
                                        (17, 1001, False), (1, 8, False)])
def test_logprob_fwd_bwd(cuda_ok, n, V, peaked):
    z, t = logits_inputs(n, V, seed=n + V, peaked=peaked)
    w = torch.randn(n, generator=torch.Generator().manual_seed(5), dtype=torch.float32)
    zc, tc, wc = z.cuda(), t.cuda(), w.cuda()
    logp, lse = ops.logprob(zc, tc)
    logp2, lse2, dz = ops.logprob(zc, tc, dlogp=wc)
    dz2 = ops.logprob_bwd(zc, tc, lse, wc)
    torch.cuda.synchronize()
    ref_lp, ref_lse = olp.logprob(z, t.long())
    ref_dz = olp.logprob_grad(z, t.long(), w.double().numpy())
    m = metrics(t2np(logp), ref_lp)
    assert m["finite"] and m["max_abs"] <= LOGP_MAX_ABS, m
    assert metrics(t2np(lse), ref_lse)["max_abs"] <= LOGP_MAX_ABS
    np.testing.assert_allclose(t2np(logp2), t2np(logp), atol=1e-5)  # fused path (V % 32 == 0) vs 2-pass
    for d in (dz, dz2):
        md = metrics(t2np(d), ref_dz)
        assert md["finite"] and md["rel_l2"] <= DZ_REL_L2, md
    # sum_v dz = 0 per row (up to bf16 rounding of dz)
    assert t2np(dz).sum(1).__abs__().max() < 1e-2 * max(1.0, np.abs(w.numpy()).max())


@pytest.mark.gpu
def test_logprob_inplace_strided_and_bad_target(cuda_ok):
    n, V, S = 8, 1000, 1024
    z, t = logits_inputs(n, V, seed=3)
    big = torch.zeros(n, S, dtype=torch.bfloat16)
    big[:, :V] = z
    bc = big.cuda()
    view = bc[:, :V]
    t_bad = t.clone()
    t_bad[2] = V  # out of range -> NaN for that row
    w = torch.ones(n)
    logp, lse = ops.logprob(view, t_bad.cuda())
    lp = t2np(logp)
    assert np.isnan(lp[2]) and np.isfinite(np.delete(lp, 2)).all()
    ref_lp, _ = olp.logprob(z, t.long())
    assert np.abs(np.delete(lp, 2) - np.delete(ref_lp, 2)).max() <= LOGP_MAX_ABS
    # in-place gradient over the strided view
    ops.logprob(view, t.cuda(), dlogp=w.cuda(), dlogits=view)
    torch.cuda.synchronize()
    ref_dz = olp.logprob_grad(z, t.long(), w.double().numpy())
    assert metrics(t2np(view), ref_dz)["rel_l2"] <= DZ_REL_L2
    assert torch.all(bc[:, V:] == 0)


@pytest.mark.gpu
@pytest.mark.parametrize("clip", [False, True])
def test_dipo_kernels_vs_oracle(cuda_ok, clip):
    n_groups, G = 4, 8
    g = torch.Generator().manual_seed(11)
    lens = torch.randint(1, 40, (n_groups * G,), generator=g).tolist()
    rewards, group_of_traj, traj_of_token = rl_batch(n_groups, G, lens, seed=2)
    n_tok = traj_of_token.numel()
    logp = -torch.rand(n_tok, generator=g, dtype=torch.float64) * 3
    old = logp.clone()
    if clip:
        old += torch.randn(n_tok, generator=g, dtype=torch.float64) * 0.3
    loss, dl, st = odipo.dipo_loss(logp.numpy(), old.numpy(), traj_of_token.numpy(), rewards.numpy(),
                                   group_of_traj.numpy())
    lp32, old32 = logp.float(), old.float()
    # the kernel computes rho from fp32 inputs; feed the oracle the same fp32 values
    loss32, dl32, _ = odipo.dipo_loss(lp32.double().numpy(), old32.double().numpy(), traj_of_token.numpy(),
                                      rewards.numpy(), group_of_traj.numpy())
    cu = lambda x, dt: x.to(dt).cuda()
    gloss, gdl, parts = bdipo.dipo_loss(cu(lp32, torch.float32), cu(old32, torch.float32),
                                        cu(traj_of_token, torch.int32), cu(rewards, torch.float32),
                                        cu(group_of_traj, torch.int32), cu(torch.tensor(lens), torch.int32),
                                        n_groups)
    torch.cuda.synchronize()
    assert abs(gloss.item() - loss32) < 1e-6 * max(1.0, abs(loss32))
    np.testing.assert_allclose(t2np(gdl), dl32, rtol=1e-5, atol=1e-9)
    assert parts[1].item() == n_tok
    if not clip:
        np.testing.assert_allclose(t2np(gdl), dl, rtol=1e-5, atol=1e-9)
        assert parts[2].item() == 0


@pytest.mark.gpu
@pytest.mark.parametrize("V", [1024, VOCAB_QWEN3])
def test_logprob_fused_inplace_strided(cuda_ok, V):
    """Cluster-fused forward + gradient, in place over a strided view."""
    n, S = 9, V + 64
    z, t = logits_inputs(n, V, seed=V)
    big = torch.zeros(n, S, dtype=torch.bfloat16)
    big[:, :V] = z
    bc = big.cuda()
    view = bc[:, :V]
    w = torch.linspace(-1, 2, n)
    logp, lse, _ = ops.logprob(view, t.cuda(), dlogp=w.cuda(), dlogits=view)
    torch.cuda.synchronize()
    ref_lp, ref_lse = olp.logprob(z, t.long())
    ref_dz = olp.logprob_grad(z, t.long(), w.double().numpy())
    assert metrics(t2np(logp), ref_lp)["max_abs"] <= LOGP_MAX_ABS
    assert metrics(t2np(lse), ref_lse)["max_abs"] <= LOGP_MAX_ABS
    assert metrics(t2np(view), ref_dz)["rel_l2"] <= DZ_REL_L2
    assert torch.all(bc[:, V:] == 0)


@pytest.mark.gpu
def test_dipo_online_rho_one(cuda_ok):
    """logp = logp_old = None: the Eq. 7 online setting, rho == 1 (weights = -A/(N_g n_groups))."""
    rewards, group_of_traj, traj_of_token = rl_batch(2, 4, [3, 1, 4, 1, 5, 9, 2, 6], seed=4)
    lens = [3, 1, 4, 1, 5, 9, 2, 6]
    lp = np.zeros(traj_of_token.numel())
    loss, dl, _ = odipo.dipo_loss(lp, lp, traj_of_token.numpy(), rewards.numpy(), group_of_traj.numpy())
    cu = lambda x, dt: x.to(dt).cuda()
    gloss, gdl, _ = bdipo.dipo_loss(None, None, cu(traj_of_token, torch.int32), cu(rewards, torch.float32),
                                    cu(group_of_traj, torch.int32), cu(torch.tensor(lens), torch.int32), 2)
    torch.cuda.synchronize()
    assert abs(gloss.item() - loss) < 1e-9
    np.testing.assert_allclose(t2np(gdl), dl, rtol=1e-6, atol=1e-9)


@pytest.mark.gpu
def test_fused_logprob_masked_vocab(cuda_ok):
    """-inf logits (masked vocabulary entries) through the one-barrier fused
    kernel: a whole cluster slice masked (its (max, sum) pair is (-inf, 0)), the
    slice holding the row max masked, half the vocabulary masked at random;
    targets stay on finite entries.  Masked entries get dz = 0 exactly."""
    n, V = 4, VOCAB_QWEN3
    z, t = logits_inputs(n, V, seed=21)
    q = V // 4  # the fused kernel's slice per CTA of the 4-CTA cluster
    z[0, :q] = float("-inf")
    z[1, 2 * q:3 * q] = float("-inf")
    g = torch.Generator().manual_seed(4)
    z[2, torch.rand(V, generator=g) < 0.5] = float("-inf")
    for i in range(n):  # targets on finite logits
        while not torch.isfinite(z[i, t[i]]):
            t[i] = (t[i] + 997) % V
    w = torch.randn(n, generator=torch.Generator().manual_seed(6), dtype=torch.float32)
    zc = z.cuda()
    logp, lse, dz = ops.logprob(zc, t.cuda(), dlogp=w.cuda())
    torch.cuda.synchronize()
    ref_lp, ref_lse = olp.logprob(z, t.long())
    ref_dz = olp.logprob_grad(z, t.long(), w.double().numpy())
    assert metrics(t2np(logp), ref_lp)["max_abs"] <= LOGP_MAX_ABS
    assert metrics(t2np(lse), ref_lse)["max_abs"] <= LOGP_MAX_ABS
    d = t2np(dz)
    assert np.isfinite(d).all()
    assert (d[~np.isfinite(t2np(z))] == 0).all()
    assert metrics(d, ref_dz)["rel_l2"] <= DZ_REL_L2


@pytest.mark.gpu
@pytest.mark.parametrize("low", [-60.0, -200.0])
def test_fused_logprob_wide_spread(cuda_ok, low):
    """The fused kernel takes each thread's FIRST vector's max as its exponent
    reference and redoes the thread from global memory against its exact max
    when a later element lies so far above it that the thread's sum leaves
    [0, 2^64).  Rows whose every slice starts with 8 KB of very low logits
    (every thread's first vector) followed by N(0, 3^2) logits and a +40 spike
    take that path for every thread; a -inf-led row and a row with the spike
    in the first vectors take the common path.  Element-wise vs the oracle."""
    n, V = 6, VOCAB_QWEN3
    z, t = logits_inputs(n, V, seed=31)
    q = V // 4
    for r in range(4):
        for c in range(4):
            z[r, c * q:c * q + 2048] = low  # bf16-exact for both values
        z[r, (r * 7919 + 5000) % V] = 40.0
    z[4, :2048] = float("-inf")
    z[5, 100] = 40.0
    w = torch.randn(n, generator=torch.Generator().manual_seed(8), dtype=torch.float32)
    zc = z.cuda()
    logp, lse, dz = ops.logprob(zc, t.cuda(), dlogp=w.cuda())
    torch.cuda.synchronize()
    ref_lp, ref_lse = olp.logprob(z, t.long())
    ref_dz = olp.logprob_grad(z, t.long(), w.double().numpy())
    assert metrics(t2np(logp), ref_lp)["max_abs"] <= LOGP_MAX_ABS
    assert metrics(t2np(lse), ref_lse)["max_abs"] <= LOGP_MAX_ABS
    d = t2np(dz)
    assert np.isfinite(d).all()
    for i in range(n):
        assert metrics(d[i:i + 1], ref_dz[i:i + 1])["rel_l2"] <= DZ_REL_L2, i


@pytest.mark.gpu
def test_fused_logprob_target_positions(cuda_ok):
    """Targets at slice edges and inside the register-held tail of the fused
    kernel's slices (at Qwen3 V the last 1,280 vectors of every 37,984-element
    slice live in registers, the rest in shared memory): logp, LSE and dz
    element-wise vs the oracle, the target entry included."""
    V = VOCAB_QWEN3
    q = V // 4
    tail0 = q - 1280 * 8  # first register-held element of a slice
    pos = [0, 7, 8, tail0 - 1, tail0, tail0 + 9, q - 1, q, 2 * q + tail0 + 3, 3 * q - 1, V - 8, V - 1]
    n = len(pos)
    z, _ = logits_inputs(n, V, seed=41)
    t = torch.tensor(pos, dtype=torch.int32)
    w = torch.randn(n, generator=torch.Generator().manual_seed(9), dtype=torch.float32)
    logp, lse, dz = ops.logprob(z.cuda(), t.cuda(), dlogp=w.cuda())
    torch.cuda.synchronize()
    ref_lp, ref_lse = olp.logprob(z, t.long())
    ref_dz = olp.logprob_grad(z, t.long(), w.double().numpy())
    assert metrics(t2np(logp), ref_lp)["max_abs"] <= LOGP_MAX_ABS
    assert metrics(t2np(lse), ref_lse)["max_abs"] <= LOGP_MAX_ABS
    d = t2np(dz)
    for i in range(n):
        assert metrics(d[i:i + 1], ref_dz[i:i + 1])["rel_l2"] <= DZ_REL_L2, i
        # the target entry itself: w (1 - p_t) within bf16 rounding
        assert abs(d[i, pos[i]] - ref_dz[i, pos[i]]) <= 1e-2 * abs(w[i].item()) + 1e-3, (i, d[i, pos[i]], ref_dz[i, pos[i]])


@pytest.mark.gpu
@pytest.mark.parametrize("V", [49120, 49152, 50176, 65536 + 32])
def test_fused_logprob_register_tail_boundary(cuda_ok, V):
    """Vocabularies at the fused kernel's register-tail threshold (a slice of
    >= 6 x 256 16-byte vectors keeps 5 x 256 of them in registers): 49,152 is
    the first size on the register path with ONE shared-memory vector per
    thread; 49,120 the last without.  logp / LSE / dz vs the oracle."""
    n = 5
    z, t = logits_inputs(n, V, seed=V)
    t[0] = V - 1
    t[1] = 0
    w = torch.randn(n, generator=torch.Generator().manual_seed(V), dtype=torch.float32)
    logp, lse, dz = ops.logprob(z.cuda(), t.cuda(), dlogp=w.cuda())
    torch.cuda.synchronize()
    ref_lp, ref_lse = olp.logprob(z, t.long())
    ref_dz = olp.logprob_grad(z, t.long(), w.double().numpy())
    assert metrics(t2np(logp), ref_lp)["max_abs"] <= LOGP_MAX_ABS
    assert metrics(t2np(lse), ref_lse)["max_abs"] <= LOGP_MAX_ABS
    md = metrics(t2np(dz), ref_dz)
    assert md["finite"] and md["rel_l2"] <= DZ_REL_L2, md


@pytest.mark.gpu
def test_fused_logprob_in_place_qwen3(cuda_ok):
    """The fused kernel in place (dlogits = logits) at the Qwen3 vocabulary --
    the bench's and a training step's use: each CTA reads its slice (shared
    memory part by bulk copy, register tail by streaming loads) before writing
    dz over it; a wide-spread row takes the global-memory redo path, which must
    still see the original logits.  Bit-identical to the out-of-place call."""
    n, V = 6, VOCAB_QWEN3
    z, t = logits_inputs(n, V, seed=55)
    z[0, :2048] = -60.0  # the redo path (first vectors far below the rest)
    w = torch.randn(n, generator=torch.Generator().manual_seed(3), dtype=torch.float32)
    zc, tc, wc = z.cuda(), t.cuda(), w.cuda()
    lp1, ls1, dz1 = ops.logprob(zc, tc, dlogp=wc)
    zi = zc.clone()
    lp2, ls2, dz2 = ops.logprob(zi, tc, dlogp=wc, dlogits=zi)
    torch.cuda.synchronize()
    assert dz2.data_ptr() == zi.data_ptr()
    assert torch.equal(lp1, lp2) and torch.equal(ls1, ls2)
    assert torch.equal(dz1.view(torch.int16), zi.view(torch.int16))
    ref_dz = olp.logprob_grad(z, t.long(), w.double().numpy())
    assert metrics(t2np(zi), ref_dz)["rel_l2"] <= DZ_REL_L2
