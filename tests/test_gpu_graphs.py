"""The hot path is CUDA-graph capturable: no host synchronisation, no host->
device copies and no allocation inside the ABI calls (tile maps are rebuilt
on device, TMA descriptors and varlen lengths travel as kernel parameters).
A captured step (attention fwd -> DiPO weights -> fused logprob -> attention
bwd, plus a decode step) replays bit-identically to the eager run, and the
eager run itself matches the fp64 oracle (checked by the other parity tests;
here the attention output is re-checked against the oracle once)."""

import numpy as np
import pytest
import torch

from oracle import Problem as OP, attention
from parity import assert_fwd, t2np
from workloads import CONFIGS, attn_inputs, logits_inputs, decode_inputs

pytestmark = pytest.mark.gpu


def _step(bd, ops, dipo, prob, t):
    o, lse = bd.attn_fwd(prob, t["q"], t["k"], t["v"], t["o"], t["lse"])
    _, dlogp, parts = dipo.dipo_loss(None, None, t["tok"], t["rew"], t["gid"], t["tlen"], 1)
    ops.logprob(t["z"], t["tgt"], dlogp=dlogp, dlogits=t["z"])
    bd.attn_bwd(prob, t["q"], t["k"], t["v"], o, lse, t["do"], t["dq"], t["dk"], t["dv"])
    ops.decode_attn(t["dq_q"], t["kc"], t["vc"], t["kvl"], o=t["dec_o"], lse=t["dec_lse"])
    return parts


@pytest.mark.parametrize("varlen", [False, True])
def test_capture_replay_bitwise(cuda_ok, varlen):
    import paper_2512_22234_b200 as bd
    from paper_2512_22234_b200 import ops, dipo
    cfg = CONFIGS["tiny"].with_(batch=2, response_len=160, n_q_heads=4, n_kv_heads=2, head_dim=128)
    if varlen:
        cfg = cfg.with_(resp_lens=(160, 96))
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, do = [x.cuda() for x in attn_inputs(cfg)]
    n_rows, V = cfg.batch * cfg.response_len, 1024
    z0, tgt = logits_inputs(n_rows, V, seed=3)
    qd, kc, vc, kvl = decode_inputs(2, 4, 4, 2, 128, 512, seed=4)
    t = dict(q=q, k=k, v=v, do=do, o=torch.empty_like(q),
             lse=torch.empty((cfg.batch, cfg.n_q_heads, cfg.ntot), device="cuda"),
             dq=torch.zeros_like(q), dk=torch.zeros_like(k), dv=torch.zeros_like(v),
             z=z0.cuda().clone(), tgt=tgt.cuda(),
             tok=torch.arange(cfg.batch, device="cuda", dtype=torch.int32).repeat_interleave(cfg.response_len),
             rew=torch.tensor([1.0, 0.0], device="cuda"), gid=torch.zeros(2, dtype=torch.int32, device="cuda"),
             tlen=torch.full((2,), cfg.response_len, dtype=torch.int32, device="cuda"),
             dq_q=qd.cuda(), kc=kc.cuda(), vc=vc.cuda(), kvl=kvl.cuda(),
             dec_o=torch.empty_like(qd.cuda()), dec_lse=torch.empty((2, 4, 4), device="cuda"))
    for n in ("o", "dq", "dk", "dv", "dec_o"):
        t[n].zero_()  # varlen padding rows are never written: start from zeros
    # eager reference (also grows the shared workspace to its final size)
    _step(bd, ops, dipo, prob, t)
    torch.cuda.synchronize()
    eager = {n: t[n].clone() for n in ("o", "lse", "dq", "dk", "dv", "z", "dec_o", "dec_lse")}
    # capture, reset the in-place logits, replay twice
    t["z"].copy_(z0.cuda())
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            _step(bd, ops, dipo, prob, t)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        t["z"].copy_(z0.cuda())
        for n in ("o", "dq", "dk", "dv", "dec_o"):
            t[n].zero_()
        g.replay()
        torch.cuda.synchronize()
        for n, ref in eager.items():
            assert torch.equal(t[n].view(torch.uint8) if t[n].dtype == torch.bfloat16 else t[n],
                               ref.view(torch.uint8) if ref.dtype == torch.bfloat16 else ref), n
    if not varlen:
        oprob = OP(cfg.batch, cfg.prompt_len, cfg.response_len, cfg.block_size, cfg.n_q_heads, cfg.n_kv_heads,
                   cfg.head_dim, cfg.repeat_prompt)
        o_ref, _ = attention.forward(oprob, q.cpu(), k.cpu(), v.cpu())
        assert_fwd("O", t2np(t["o"]), o_ref)
