"""Varlen batches: per-sequence (P_i, R_i) in the padded
[b, Ntot, H, d] layout.  Each sequence's valid rows [0, N_i) are compared with
the fp64 oracle run on that sequence alone (a varlen batch is a set of
independent problems, so the oracle is the per-sequence definition); rows past
N_i hold a poison value on input (any leak into a valid output breaks parity)
and must be left untouched on output.  The varlen launch is also bit-identical
to a uniform launch of each sequence alone (same tile lists, same order)."""

import numpy as np
import pytest
import torch

import paper_2512_22234_b200 as bd
from oracle import Problem as OProblem, attention
from parity import assert_fwd, assert_grad, t2np

POISON = 64.0

CASES = [
    # (Hq, Hkv, d, B, rp, S, [(P_i, R_i)])
    ("dirl_gqa2", 4, 2, 128, 4, 1, 1, [(64, 320), (32, 96), (0, 200), (64, 64)]),
    ("resp_only_ragged", 2, 1, 128, 8, 0, 1, [(40, 200), (16, 48), (40, 8)]),
    ("copies2_d64", 2, 2, 64, 4, 1, 2, [(16, 176), (8, 40), (16, 112)]),
    ("single_seq", 4, 2, 128, 4, 1, 1, [(32, 96)]),
    # more dQ units than SMs with many skipped (short sequences): the
    # persistent dQ kernel's publisher skips units past a sequence's tile count
    ("many_seqs_units", 8, 2, 64, 4, 1, 1,
     [(64, 448), (8, 24), (32, 160), (0, 512), (16, 80), (64, 320), (24, 40), (48, 208), (0, 96), (40, 472)]),
]


def _setup(Hq, Hkv, d, B, rp, S, lens, seed=0):
    Pm, Rm = max(p for p, _ in lens), max(r for _, r in lens)
    prob = bd.Problem(len(lens), Pm, Rm, B, Hq, Hkv, d, repeat_prompt=rp, n_copies=S,
                      seq_prompt_lens=tuple(p for p, _ in lens), seq_response_lens=tuple(r for _, r in lens))
    N = prob.ntot
    g = torch.Generator().manual_seed(seed)
    q = torch.randn((len(lens), N, Hq, d), generator=g)
    k = torch.randn((len(lens), N, Hkv, d), generator=g)
    v = torch.randn((len(lens), N, Hkv, d), generator=g)
    do = torch.randn((len(lens), N, Hq, d), generator=g)
    for i in range(len(lens)):
        n_i = prob.seq_packed_len(i)
        for x in (q, k, v, do):
            x[i, n_i:] = POISON
    return prob, q.bfloat16(), k.bfloat16(), v.bfloat16(), do.bfloat16()


def _oprob(prob, i):
    return OProblem(1, prob.seq_prompt_lens[i], prob.seq_response_lens[i], prob.block_size, prob.n_q_heads,
                    prob.n_kv_heads, prob.head_dim, prob.repeat_prompt, n_copies=prob.n_copies)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_varlen_parity_and_untouched_padding(cuda_ok, case):
    _, Hq, Hkv, d, B, rp, S, lens = case
    prob, q, k, v, do = _setup(Hq, Hkv, d, B, rp, S, lens)
    qc, kc, vc, doc = q.cuda(), k.cuda(), v.cuda(), do.cuda()
    SENT = -7.0
    o = torch.full_like(qc, SENT)
    lse = torch.full((prob.batch, Hq, prob.ntot), SENT, device="cuda")
    o, lse = bd.attn_fwd(prob, qc, kc, vc, o, lse)
    dq, dk, dv = torch.full_like(qc, SENT), torch.full_like(kc, SENT), torch.full_like(vc, SENT)
    dq, dk, dv = bd.attn_bwd(prob, qc, kc, vc, o, lse, doc, dq, dk, dv)
    torch.cuda.synchronize()
    for i in range(prob.batch):
        n = prob.seq_packed_len(i)
        op = _oprob(prob, i)
        sl = lambda x: x[i:i + 1, :n]
        o_r, l_r = attention.forward(op, sl(q), sl(k), sl(v))
        assert_fwd(f"o[{i}]", t2np(o[i:i + 1, :n]), o_r)
        assert_fwd(f"lse[{i}]", t2np(lse[i:i + 1, :, :n]), l_r)
        dq_r, dk_r, dv_r = attention.backward(op, sl(q), sl(k), sl(v), sl(do))
        assert_grad(f"dq[{i}]", t2np(dq[i:i + 1, :n]), dq_r)
        assert_grad(f"dk[{i}]", t2np(dk[i:i + 1, :n]), dk_r)
        assert_grad(f"dv[{i}]", t2np(dv[i:i + 1, :n]), dv_r)
        for x in (o[i, n:], lse[i, :, n:], dq[i, n:], dk[i, n:], dv[i, n:]):
            assert torch.all(x == SENT), f"padding of sequence {i} was written"


@pytest.mark.gpu
def test_varlen_bit_identical_to_uniform_launches(cuda_ok, monkeypatch):
    # varlen batches take the recompute backward; so must the uniform
    # single-sequence launches compared bit for bit (the stored-dS path
    # computes dS from S^T / dP^T instead of S / dP: same values to fp32
    # rounding, not bit for bit)
    monkeypatch.setenv("BD_BWD_DS", "0")
    prob, q, k, v, do = _setup(4, 2, 128, 4, 1, 1, [(64, 320), (32, 96), (0, 200)], seed=3)
    qc, kc, vc, doc = q.cuda(), k.cuda(), v.cuda(), do.cuda()
    o, lse = bd.attn_fwd(prob, qc, kc, vc)
    dq, dk, dv = bd.attn_bwd(prob, qc, kc, vc, o, lse, doc)
    for i in range(prob.batch):
        n = prob.seq_packed_len(i)
        one = bd.Problem(1, prob.seq_prompt_lens[i], prob.seq_response_lens[i], 4, 4, 2, 128)
        s = lambda x: x[i:i + 1, :n].contiguous()
        o1, l1 = bd.attn_fwd(one, s(qc), s(kc), s(vc))
        dq1, dk1, dv1 = bd.attn_bwd(one, s(qc), s(kc), s(vc), o1, l1, s(doc))
        assert torch.equal(o[i:i + 1, :n], o1) and torch.equal(lse[i:i + 1, :, :n], l1)
        assert torch.equal(dq[i:i + 1, :n], dq1) and torch.equal(dk[i:i + 1, :n], dk1)
        assert torch.equal(dv[i:i + 1, :n], dv1)
