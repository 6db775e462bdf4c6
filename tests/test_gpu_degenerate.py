"""GPU parity on the method's degenerate cases (SURVEY §8(c) pins, run
through the C ABI): an empty noisy copy with B = 1 is causal attention
(compared with torch fp64 SDPA, is_causal=True, and with the oracle), a
single block with no prompt is bidirectional attention within each copy,
and B = L makes every x0 row see the whole clean sequence."""

import math

import numpy as np
import pytest
import torch

import paper_2512_22234_b200 as bd
from oracle import Problem as OP, attention
from parity import assert_fwd, assert_grad, t2np
from workloads import AttnConfig, attn_inputs

pytestmark = pytest.mark.gpu


def _run(cfg):
    q, k, v, do = attn_inputs(cfg, device="cpu")
    prob = bd.Problem.from_cfg(cfg)
    qc, kc, vc, doc = q.cuda(), k.cuda(), v.cuda(), do.cuda()
    o, lse = bd.attn_fwd(prob, qc, kc, vc)
    dq, dk, dv = bd.attn_bwd(prob, qc, kc, vc, o, lse, doc)
    torch.cuda.synchronize()
    return (q, k, v, do), (o, lse, dq, dk, dv)


@pytest.mark.parametrize("P,d,H", [(256, 128, 2), (200, 64, 1), (72, 128, 4)])
def test_empty_noisy_copy_is_causal_attention(cuda_ok, P, d, H):
    """repeat_prompt = 0, R = 0: Ntot = P rows of x0 only, B = 1 -> causal."""
    cfg = AttnConfig("causal", 1, H, H, d, P, 0, 1, repeat_prompt=0)
    (q, k, v, do), (o, lse, dq, dk, dv) = _run(cfg)
    assert o.shape[1] == P
    for h in range(H):
        qh, kh, vh = (x[0, :, h].double().requires_grad_() for x in (q, k, v))
        ref = torch.nn.functional.scaled_dot_product_attention(qh[None], kh[None], vh[None], is_causal=True)[0]
        assert_fwd("o_vs_sdpa", t2np(o[0, :, h]), ref.detach().numpy())
        ref.backward(do[0, :, h].double())
        assert_grad("dq_vs_sdpa", t2np(dq[0, :, h]), qh.grad.numpy())
        assert_grad("dk_vs_sdpa", t2np(dk[0, :, h]), kh.grad.numpy())
        assert_grad("dv_vs_sdpa", t2np(dv[0, :, h]), vh.grad.numpy())
        lse_ref = torch.logsumexp((qh @ kh.T / math.sqrt(d)).masked_fill(
            torch.ones(P, P, dtype=torch.bool).triu(1), float("-inf")), -1)
        assert_fwd("lse_vs_sdpa", t2np(lse[0, h]), lse_ref.detach().numpy())


@pytest.mark.parametrize("B,copies", [(128, 1), (64, 1), (128, 2)])
def test_single_block_is_bidirectional(cuda_ok, B, copies):
    """P = 0, R = B: one block; x0 rows = bidirectional SDPA over x0, each noisy
    copy = bidirectional SDPA over itself."""
    cfg = AttnConfig("one_block", 1, 2, 1, 128, 0, B, B, n_copies=copies)
    (q, k, v, do), (o, lse, dq, dk, dv) = _run(cfg)
    for seg in range(1 + copies):
        rows = slice(seg * B, (seg + 1) * B)
        for h in range(2):
            ref = torch.nn.functional.scaled_dot_product_attention(
                q[0, rows, h].double()[None], k[0, rows, 0].double()[None], v[0, rows, 0].double()[None])[0]
            assert_fwd(f"o_seg{seg}", t2np(o[0, rows, h]), ref.numpy())


def test_block_equals_sequence_and_oracle_grads(cuda_ok):
    """B = L = 256 (prompt 64 + response 192): x0 rows see all of x0, every xt
    row sees only xt (its block is the whole sequence); full oracle check of
    the forward and the gradients."""
    cfg = AttnConfig("BeqL", 1, 4, 2, 128, 64, 192, 256)
    (q, k, v, do), (o, lse, dq, dk, dv) = _run(cfg)
    op = OP(1, 64, 192, 256, 4, 2, 128, 1)
    o_ref, lse_ref = attention.forward(op, q, k, v)
    assert_fwd("o", t2np(o), o_ref)
    assert_fwd("lse", t2np(lse), lse_ref)
    dq_r, dk_r, dv_r = attention.backward(op, q, k, v, do)
    for name, got, ref in (("dq", dq, dq_r), ("dk", dk, dk_r), ("dv", dv, dv_r)):
        assert_grad(name, t2np(got), ref)
