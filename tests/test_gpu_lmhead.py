"""GPU parity of the fused LM head + logprob through the
C ABI against the fp64 oracle (oracle/lmhead.py), and of the CTA-pair GEMM
engine behind it.

Tolerances: the forward keeps fp32 logits and fp32 softmax sums (no bf16
rounding of z), so logp uses the path's 1e-3 max-abs bound (parity.py).  The
backward rounds dz to bf16 before the two gradient GEMMs and dh to bf16 on
output: dh, dW rel-L2 <= 1e-2 (the dz bound of bd_logprob, parity.py)."""

import numpy as np
import pytest
import torch

from oracle import lmhead as olm
from parity import metrics, t2np, LOGP_MAX_ABS, DZ_REL_L2
from workloads import lmhead_inputs, LMHEAD_SHAPES

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2512_22234_b200 import ops
    return ops


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K", [(392, 520, 200), (256, 2048, 64), (136, 264, 1032)])
def test_gemm_engine(cuda_ok, a_mn, b_mn, M, N, K):
    g = torch.Generator().manual_seed(M + N + K)
    a = torch.randn((M, K), generator=g).to(torch.bfloat16)
    b = torch.randn((N, K), generator=g).to(torch.bfloat16)
    ref = a.double() @ b.double().T
    ad = (a.T.contiguous() if a_mn else a).cuda()
    bd = (b.T.contiguous() if b_mn else b).cuda()
    out = _ops().selftest_gemm(ad, bd, a_mn, b_mn)
    torch.cuda.synchronize()
    m = metrics(t2np(out), ref.numpy())
    assert m["finite"] and m["rel_l2"] < 1e-5, m


@pytest.mark.parametrize("n,C,V", [(64, 256, 1000), (300, 256, 1000), (1000, 512, 4104), (517, 128, 33000)])
def test_lmhead_fwd(cuda_ok, n, C, V):
    h, W, t, _ = lmhead_inputs(n, C, V, seed=n)
    logp, lse = _ops().lmhead_logprob(h.cuda(), W.cuda(), t.cuda())
    torch.cuda.synchronize()
    lp_ref, lse_ref = olm.lmhead_logprob(h, W, t.long())
    m = metrics(t2np(logp), lp_ref)
    assert m["finite"] and m["max_abs"] <= LOGP_MAX_ABS, m
    m2 = metrics(t2np(lse), lse_ref)
    assert m2["max_abs"] <= LOGP_MAX_ABS, m2


def test_lmhead_fwd_bad_target_nan(cuda_ok):
    h, W, t, _ = lmhead_inputs(40, 128, 512, seed=3)
    t[5] = 512
    t[7] = -1
    logp, _ = _ops().lmhead_logprob(h.cuda(), W.cuda(), t.cuda())
    lp = t2np(logp)
    assert np.isnan(lp[5]) and np.isnan(lp[7])
    ok = np.ones(40, bool)
    ok[[5, 7]] = False
    assert np.isfinite(lp[ok]).all()


@pytest.mark.parametrize("n,C,V,chunk", [(300, 256, 1000, 0), (300, 256, 1000, 128), (1000, 512, 4104, 384)])
def test_lmhead_bwd(cuda_ok, n, C, V, chunk):
    h, W, t, w = lmhead_inputs(n, C, V, seed=n + 1)
    ops = _ops()
    hc, Wc, tc, wc = h.cuda(), W.cuda(), t.cuda(), w.cuda()
    _, lse = ops.lmhead_logprob(hc, Wc, tc)
    dh, dW = ops.lmhead_logprob_bwd(hc, Wc, tc, lse, wc, chunk_rows=chunk)
    torch.cuda.synchronize()
    dh_ref, dW_ref = olm.lmhead_logprob_grad(h, W, t.long(), w.double())
    for name, got, ref in (("dh", dh, dh_ref), ("dW", dW, dW_ref)):
        m = metrics(t2np(got), ref)
        assert m["finite"] and m["rel_l2"] <= DZ_REL_L2, (name, m)


def test_lmhead_fullsize_sampled(cuda_ok):
    """SDAR-8B LM-head shape (131,072 rows x 4,096 x 151,936) in the bench launch
    configuration; logp / LSE of 14 seeded rows and dh of 4 rows vs
    oracle.lmhead row by row (each row is independent of the others); dW over
    all rows satisfies sum_v dW_v = 0 (every row of dz sums to zero)."""
    n, C, V = LMHEAD_SHAPES["sdar_8b"]
    h, W, t, w = lmhead_inputs(n, C, V, device="cuda", seed=11)
    ops = _ops()
    logp, lse = ops.lmhead_logprob(h, W, t)
    torch.cuda.synchronize()
    rows = torch.randint(0, n, (12,), generator=torch.Generator().manual_seed(5)).tolist() + [0, n - 1]
    Wc = W.cpu()
    hs, ts = h[rows].cpu(), t[rows].cpu().long()
    lp_ref, lse_ref = olm.lmhead_logprob(hs, Wc, ts.numpy())
    m = metrics(t2np(logp[rows]), lp_ref)
    assert m["finite"] and m["max_abs"] <= LOGP_MAX_ABS, m
    assert metrics(t2np(lse[rows]), lse_ref)["max_abs"] <= LOGP_MAX_ABS
    dh, dW = ops.lmhead_logprob_bwd(h, W, t, lse, w, chunk_rows=16384)
    torch.cuda.synchronize()
    sub = rows[:4]
    dh_ref, _ = olm.lmhead_logprob_grad(hs[:4], Wc, ts[:4].numpy(), w[sub].double().cpu().numpy())
    m = metrics(t2np(dh[sub]), dh_ref)
    assert m["finite"] and m["rel_l2"] <= DZ_REL_L2, m
    assert torch.isfinite(dW).all()
    col = dW.double().sum(0)
    assert col.abs().max().item() <= 1e-3 * dW.double().abs().sum(0).max().item()


def test_lmhead_full_vocab_and_hidden(cuda_ok):
    """Full Qwen3 / SDAR-8B vocabulary and hidden size (V 151,936, C 4,096) with
    64 rows processed in four chunks: dh and the whole dW [V, C] element by
    element vs oracle.lmhead (every N tile, K chunk and row chunk of the four
    GEMMs), logp / LSE of every row."""
    n, C, V = 64, 4096, 151936
    h, W, t, w = lmhead_inputs(n, C, V, seed=17)
    ops = _ops()
    hc, Wc, tc, wc = h.cuda(), W.cuda(), t.cuda(), w.cuda()
    logp, lse = ops.lmhead_logprob(hc, Wc, tc)
    dh, dW = ops.lmhead_logprob_bwd(hc, Wc, tc, lse, wc, chunk_rows=16)
    torch.cuda.synchronize()
    lp_ref, lse_ref = olm.lmhead_logprob(h, W, t.long().numpy())
    assert metrics(t2np(logp), lp_ref)["max_abs"] <= LOGP_MAX_ABS
    assert metrics(t2np(lse), lse_ref)["max_abs"] <= LOGP_MAX_ABS
    dh_ref, dW_ref = olm.lmhead_logprob_grad(h, W, t.long().numpy(), w.double().numpy())
    for name, got, ref in (("dh", dh, dh_ref), ("dW", dW, dW_ref)):
        m = metrics(t2np(got), ref)
        assert m["finite"] and m["rel_l2"] <= DZ_REL_L2, (name, m)
