"""The Python binding validates every tensor before its pointer crosses the
C ABI (fp32 logits read as bf16 or int64 targets read as int32
pairs gave silently wrong results; undersized q / k / v / o / lse made the TMA
descriptors read and write out of bounds): wrong dtype, shape, strides or
device raise BdError and enqueue nothing.  Also: per-call workspaces on two
streams do not interfere, and the DiPO kernels flag invalid ids / empty
groups with NaN instead of reading out of bounds."""

import math

import pytest
import torch

import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import ops
from paper_2512_22234_b200._lib import BdError
from workloads import AttnConfig, attn_inputs, logits_inputs

pytestmark = pytest.mark.gpu


def _setup():
    cfg = AttnConfig("v", 2, 4, 2, 128, 32, 224, 4)
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, do = [x.cuda() for x in attn_inputs(cfg)]
    return cfg, prob, q, k, v, do


def test_attention_argument_checks(cuda_ok):
    cfg, prob, q, k, v, do = _setup()
    n0 = ops.launch_count()
    with pytest.raises(BdError, match="bfloat16"):
        bd.attn_fwd(prob, q.float(), k, v)
    with pytest.raises(BdError, match="shape"):
        bd.attn_fwd(prob, q[:, :-1], k[:, :-1], v[:, :-1])
    with pytest.raises(BdError, match="shape"):
        bd.attn_fwd(prob.with_(batch=3), q, k, v)
    with pytest.raises(BdError, match="strides"):
        bd.attn_fwd(prob, q.transpose(1, 2).contiguous().transpose(1, 2), k, v)
    with pytest.raises(BdError, match="CUDA"):
        bd.attn_fwd(prob, q.cpu(), k, v)
    o, lse = bd.attn_fwd(prob, q, k, v)
    with pytest.raises(BdError, match="lse"):
        bd.attn_bwd(prob, q, k, v, o, lse[:, :1], do)
    with pytest.raises(BdError, match="float32"):
        bd.attn_bwd(prob, q, k, v, o, lse.double(), do)
    assert ops.launch_count() == n0 + 2  # only the one valid forward (map + kernel)


def test_logprob_argument_checks(cuda_ok):
    z, t = logits_inputs(8, 1024, device="cuda")
    with pytest.raises(BdError, match="bf16"):
        ops.logprob(z.float(), t)  # _check_logits says "bf16"
    with pytest.raises(BdError, match="int32"):
        ops.logprob(z, t.long())
    with pytest.raises(BdError, match="shape"):
        ops.logprob(z, t[:4])
    with pytest.raises(BdError, match="shape"):
        ops.logprob(z, t, dlogp=torch.ones(7, device="cuda"))
    with pytest.raises(BdError, match="unit inner stride"):
        ops.logprob(z.t(), t)


def test_per_call_workspace_two_streams(cuda_ok):
    """Two problems with different tile maps on two streams at once give the
    same results as serial runs (each call gets its own stream-ordered
    workspace; the round-1 binding shared one per device)."""
    cfg, prob, q, k, v, do = _setup()
    cfg2 = AttnConfig("w", 1, 4, 2, 128, 0, 512, 16, repeat_prompt=0)
    prob2 = bd.Problem.from_cfg(cfg2)
    q2, k2, v2, _ = [x.cuda() for x in attn_inputs(cfg2, with_do=False) if x is not None] + [None]
    ref1 = bd.attn_fwd(prob, q, k, v)[0].clone()
    ref2 = bd.attn_fwd(prob2, q2, k2, v2)[0].clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            o1, _ = bd.attn_fwd(prob, q, k, v)
        with torch.cuda.stream(s2):
            o2, _ = bd.attn_fwd(prob2, q2, k2, v2)
    torch.cuda.synchronize()
    assert torch.equal(o1, ref1) and torch.equal(o2, ref2)


def test_dipo_invalid_ids_give_nan(cuda_ok):
    rew = torch.tensor([1.0, 0.0], device="cuda")
    gid = torch.tensor([0, 0], dtype=torch.int32, device="cuda")
    tlen = torch.tensor([3, 2], dtype=torch.int32, device="cuda")
    stats = ops.dipo_group_stats(rew, gid, tlen, 2)  # group 1 stays empty
    tok = torch.tensor([0, 0, 0, 1, 1], dtype=torch.int32, device="cuda")
    d, p = ops.dipo_token_loss(None, None, tok, rew, gid, stats, 1)
    assert torch.isfinite(d).all() and math.isfinite(p[0].item()) and p[1].item() == 5
    bad = torch.tensor([0, 5, 0, 1, -1], dtype=torch.int32, device="cuda")  # trajectory ids out of range
    d, p = ops.dipo_token_loss(None, None, bad, rew, gid, stats, 1)
    assert torch.isnan(d[1]) and torch.isnan(d[4]) and torch.isfinite(d[[0, 2, 3]]).all()
    assert math.isnan(p[0].item())
    gid_bad = torch.tensor([0, 1], dtype=torch.int32, device="cuda")  # trajectory 1 in the empty group 1
    d, p = ops.dipo_token_loss(None, None, tok, rew, gid_bad, stats, 1)
    assert torch.isnan(d[3:]).all() and math.isnan(p[0].item())


def test_dipo_deterministic(cuda_ok):
    """No floating-point atomics: repeated reductions are bitwise equal."""
    g = torch.Generator(device="cuda").manual_seed(0)
    n_traj, n_tok = 64, 100_000
    rew = torch.rand(n_traj, generator=g, device="cuda")
    gid = (torch.arange(n_traj, device="cuda") // 8).to(torch.int32)
    tok = torch.randint(0, n_traj, (n_tok,), generator=g, device="cuda", dtype=torch.int32)
    tlen = torch.bincount(tok.long(), minlength=n_traj).to(torch.int32)
    lp = torch.randn(n_tok, generator=g, device="cuda") * 0.1
    lo = lp + torch.randn(n_tok, generator=g, device="cuda") * 0.3
    outs = []
    for _ in range(3):
        st = ops.dipo_group_stats(rew, gid, tlen, 8)
        outs.append((st.clone(),) + ops.dipo_token_loss(lp, lo, tok, rew, gid, st, 8))
    for o in outs[1:]:
        assert all(torch.equal(a, b) for a, b in zip(o, outs[0]))
