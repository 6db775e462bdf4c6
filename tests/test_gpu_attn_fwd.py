"""GPU parity of bd_attn_fwd vs the fp64 oracle (element by element)."""

import numpy as np
import pytest
import torch

import paper_2512_22234_b200 as bd
from oracle import Problem as OProblem, attention
from parity import assert_fwd, t2np
from workloads import CONFIGS, AttnConfig, attn_inputs

CASES = [
    # name, cfg (b, Hq, Hkv, d, P, R, B, repeat_prompt)
    ("tiny", CONFIGS["tiny"]),
    ("gqa2_d128_aligned", AttnConfig("c1", 2, 4, 2, 128, 64, 320, 4)),
    ("gqa4_d128_ragged", AttnConfig("c2", 1, 8, 2, 128, 40, 160, 8)),
    ("resp_only_ragged", AttnConfig("c3", 2, 4, 2, 128, 100, 300, 4, repeat_prompt=0)),
    ("mha_d64_B1", AttnConfig("c4", 1, 3, 3, 64, 16, 240, 1)),
    ("odd_group_d128", AttnConfig("c5", 1, 3, 1, 128, 0, 256, 16)),
    ("B128", AttnConfig("c6", 1, 2, 1, 128, 128, 256, 128)),
    ("B32_d64_gqa2", AttnConfig("c7", 2, 4, 2, 64, 96, 416, 32)),
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
]


def _oprob(cfg):
    return OProblem(cfg.batch, cfg.prompt_len, cfg.response_len, cfg.block_size, cfg.n_q_heads,
                    cfg.n_kv_heads, cfg.head_dim, cfg.repeat_prompt, n_copies=cfg.n_copies)


def _check_full(cfg, stress=False, seed=None):
    q, k, v, _ = attn_inputs(cfg, device="cpu", stress=stress, with_do=False, seed=seed)
    prob = bd.Problem.from_cfg(cfg)
    o, lse = bd.attn_fwd(prob, q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    o_ref, lse_ref = attention.forward(_oprob(cfg), q, k, v)
    o_np, lse_np = t2np(o), t2np(lse)
    L = cfg.L
    out = {}
    out["o"] = assert_fwd("o", o_np, o_ref)
    out["lse"] = assert_fwd("lse", lse_np, lse_ref)
    # per segment (a bug in one mask kind must not hide in a global norm)
    out["o_x0"] = assert_fwd("o_x0", o_np[:, :L], o_ref[:, :L])
    out["o_xt"] = assert_fwd("o_xt", o_np[:, L:], o_ref[:, L:])
    out["lse_xt"] = assert_fwd("lse_xt", lse_np[:, :, L:], lse_ref[:, :, L:])
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg", CASES, ids=[c[0] for c in CASES])
def test_fwd_parity_full(cuda_ok, name, cfg):
    m = _check_full(cfg)
    print(name, {k: (round(v["max_abs"], 5), round(v["rel_l2"], 6)) for k, v in m.items()})


@pytest.mark.gpu
def test_fwd_parity_stress(cuda_ok):
    """q x 8: peaky softmax, exercises the lazy-rescale path."""
    _check_full(AttnConfig("s", 1, 4, 2, 128, 64, 448, 4), stress=True)


@pytest.mark.gpu
def test_fwd_deterministic_and_x0_independent_of_xt(cuda_ok):
    cfg = AttnConfig("d", 1, 4, 2, 128, 64, 320, 4)
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, _ = attn_inputs(cfg, device="cuda", with_do=False)
    o1, l1 = bd.attn_fwd(prob, q, k, v)
    o1, l1 = o1.clone(), l1.clone()
    o2, l2 = bd.attn_fwd(prob, q, k, v)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    L = cfg.L
    q2, k2, v2 = q.clone(), k.clone(), v.clone()
    for x in (q2, k2, v2):
        x[:, L:] += 1.0
    o3, l3 = bd.attn_fwd(prob, q2, k2, v2)
    assert torch.equal(o1[:, :L], o3[:, :L]) and torch.equal(l1[:, :, :L], l3[:, :, :L])


@pytest.mark.gpu
def test_fwd_copies_equal_single_copy_runs(cuda_ok):
    """Trace replay (reading c19): the rows of copy s from one expanded
    launch are bit-identical to a single-copy launch over [x0 | copy s] (same
    tile list in the same order)."""
    cfg = AttnConfig("r", 2, 4, 2, 128, 64, 320, 4, n_copies=3)
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, _ = attn_inputs(cfg, device="cuda", with_do=False)
    o, lse = bd.attn_fwd(prob, q, k, v)
    one = prob.with_(n_copies=1)
    L, Lx = cfg.L, cfg.L - cfg.xb
    for s in range(3):
        idx = torch.cat([torch.arange(L), L + s * Lx + torch.arange(Lx)]).cuda()
        o1, l1 = bd.attn_fwd(one, q[:, idx].contiguous(), k[:, idx].contiguous(), v[:, idx].contiguous())
        assert torch.equal(o[:, idx], o1) and torch.equal(lse[:, :, idx], l1)
