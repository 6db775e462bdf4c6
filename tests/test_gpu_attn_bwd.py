"""GPU parity of bd_attn_bwd vs the fp64 oracle (element by element)."""

import numpy as np
import pytest
import torch

import paper_2512_22234_b200 as bd
from oracle import Problem as OProblem, attention
from parity import assert_grad, t2np
from workloads import CONFIGS, AttnConfig, attn_inputs

CASES = [
    ("tiny", CONFIGS["tiny"]),
    ("gqa2_d128_aligned", AttnConfig("c1", 2, 4, 2, 128, 64, 320, 4)),
    ("gqa4_d128_ragged", AttnConfig("c2", 1, 8, 2, 128, 40, 160, 8)),
    ("resp_only_ragged", AttnConfig("c3", 1, 4, 2, 128, 100, 300, 4, repeat_prompt=0)),
    ("mha_d64_B1", AttnConfig("c4", 1, 3, 3, 64, 16, 240, 1)),
    ("odd_group_d128", AttnConfig("c5", 1, 3, 1, 128, 0, 256, 16)),
    ("B128", AttnConfig("c6", 1, 2, 1, 128, 128, 256, 128)),
    ("B32_d64_gqa2", AttnConfig("c7", 1, 4, 2, 64, 96, 416, 32)),
    ("tiny_L_lt_tile", AttnConfig("c8", 1, 2, 1, 128, 8, 24, 8)),
    ("big_block_B256", AttnConfig("c9", 1, 2, 2, 128, 0, 512, 256)),
    # trace replay: S noisy copies (reading c19)
    ("copies2_gqa2_aligned", AttnConfig("t1", 1, 4, 2, 128, 64, 320, 4, n_copies=2)),
    ("copies3_resp_only_ragged", AttnConfig("t2", 1, 2, 1, 128, 40, 200, 8, repeat_prompt=0, n_copies=3)),
    ("copies4_d64_B1", AttnConfig("t3", 1, 2, 2, 64, 0, 136, 1, n_copies=4)),
    ("copies2_B128", AttnConfig("t4", 1, 2, 1, 128, 128, 256, 128, n_copies=2)),
    # block sizes that do not divide 128 (a block straddles a tile edge: PARTIAL
    # tiles whose block boundaries are not tile-aligned) and response-only mode
    # with P % B != 0 (the first noisy row starts mid-block)
    ("B12_gqa2", AttnConfig("n1", 1, 4, 2, 128, 36, 264, 12)),
    ("B48_resp_only_P50", AttnConfig("n2", 1, 4, 2, 128, 50, 334, 48, repeat_prompt=0)),
    ("B96_d64", AttnConfig("n3", 1, 2, 1, 64, 96, 288, 96)),
    ("B200_resp_only_P130", AttnConfig("n4", 1, 2, 2, 128, 130, 470, 200, repeat_prompt=0)),
    ("resp_only_P42_B8", AttnConfig("n5", 2, 4, 2, 128, 42, 214, 8, repeat_prompt=0)),
    ("resp_only_P33_B3_odd_group", AttnConfig("n6", 1, 3, 1, 128, 33, 267, 3, repeat_prompt=0)),
    ("copies3_B12", AttnConfig("n7", 1, 4, 2, 128, 36, 264, 12, n_copies=3)),
    ("copies2_resp_only_B12_P42", AttnConfig("n8", 1, 2, 1, 128, 42, 258, 12, repeat_prompt=0, n_copies=2)),
    # more dQ units than SMs: the persistent dQ kernel walks several units per
    # CTA (unit ring slot reuse, Q / dO reload, accumulator drain between
    # units); 16 / 12 (sequence, kv head) groups exercise the merged LPT tail
    # of the dK/dV grid
    ("many_units_d64", AttnConfig("m1", 8, 8, 2, 64, 64, 320, 4)),
    ("many_units_d128", AttnConfig("m2", 6, 8, 2, 128, 32, 352, 8)),
]


def _oprob(cfg):
    return OProblem(cfg.batch, cfg.prompt_len, cfg.response_len, cfg.block_size, cfg.n_q_heads,
                    cfg.n_kv_heads, cfg.head_dim, cfg.repeat_prompt, n_copies=cfg.n_copies)


def run_bwd(cfg, stress=False, structured_do=False):
    q, k, v, do = attn_inputs(cfg, device="cpu", stress=stress, structured_do=structured_do)
    prob = bd.Problem.from_cfg(cfg)
    qc, kc, vc, doc = q.cuda(), k.cuda(), v.cuda(), do.cuda()
    o, lse = bd.attn_fwd(prob, qc, kc, vc)
    dq, dk, dv = bd.attn_bwd(prob, qc, kc, vc, o, lse, doc)
    torch.cuda.synchronize()
    dq_r, dk_r, dv_r = attention.backward(_oprob(cfg), q, k, v, do)
    return (t2np(dq), t2np(dk), t2np(dv)), (dq_r, dk_r, dv_r)


def _check(cfg, **kw):
    (dq, dk, dv), (dq_r, dk_r, dv_r) = run_bwd(cfg, **kw)
    L = cfg.L
    m = {}
    for name, got, ref in (("dq", dq, dq_r), ("dk", dk, dk_r), ("dv", dv, dv_r)):
        m[name] = assert_grad(name, got, ref)
        if np.linalg.norm(ref[:, :L]) > 0:
            m[name + "_x0"] = assert_grad(name + "_x0", got[:, :L], ref[:, :L])
        if np.linalg.norm(ref[:, L:]) > 0:
            m[name + "_xt"] = assert_grad(name + "_xt", got[:, L:], ref[:, L:])
    return m


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg", CASES, ids=[c[0] for c in CASES])
def test_bwd_parity_full(cuda_ok, name, cfg):
    m = _check(cfg)
    print(name, {k: round(v["rel_l2"], 5) for k, v in m.items()})


@pytest.mark.gpu
def test_bwd_parity_stress_and_structured(cuda_ok):
    _check(AttnConfig("s", 1, 4, 2, 128, 64, 448, 4), stress=True)
    _check(AttnConfig("s2", 1, 4, 2, 128, 64, 448, 4), structured_do=True)


@pytest.mark.gpu
def test_bwd_invariants(cuda_ok):
    """sum_j dK_j ~ 0 per head (sum_j dS_ij = 0); x0 rows' dQ does not depend
    on xt inputs (up to atomic-order rounding)."""
    cfg = AttnConfig("inv", 1, 4, 2, 128, 64, 320, 4)
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, do = attn_inputs(cfg, device="cuda")
    o, lse = bd.attn_fwd(prob, q, k, v)
    dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
    s = dk.float().sum(dim=1)
    assert s.abs().max().item() < 0.05 * dk.float().abs().sum(dim=1).max().item() + 1e-3
    L = cfg.L
    q2, k2, v2 = q.clone(), k.clone(), v.clone()
    for x in (q2, k2, v2):
        x[:, L:] += 0.5
    o2, lse2 = bd.attn_fwd(prob, q2, k2, v2)
    dq2, _, _ = bd.attn_bwd(prob, q2, k2, v2, o2, lse2, do)
    assert torch.allclose(dq[:, :L].float(), dq2[:, :L].float(), atol=1e-2, rtol=0)
