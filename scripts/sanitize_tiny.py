"""Tiny end-to-end run of every ABI entry point, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): attention fwd + bwd (uniform,
varlen, trace replay, d = 64, blocks not aligned to tiles, head-sharded
strided slices, a small SDAR-8B-like slice, the opt-in stored-dS backward), fused (incl. the
Qwen3-vocabulary register-tail variant) and two-pass logprob, DiPO, LM head fwd + bwd, decode
attention + select.  Exits 0 when every call returned BD_OK."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import ops, dipo
from workloads import CONFIGS, attn_inputs, logits_inputs, lmhead_inputs, decode_inputs

torch.cuda.set_device(0)
base = CONFIGS["tiny"].with_(response_len=160, n_q_heads=4, n_kv_heads=2, head_dim=128)
for cfg in (base, base.with_(resp_lens=(160,), batch=1), base.with_(n_copies=2), base.with_(head_dim=64)):
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, do = [x.cuda() for x in attn_inputs(cfg)]
    o, lse = bd.attn_fwd(prob, q, k, v)
    bd.attn_bwd(prob, q, k, v, o, lse, do)
# block sizes that straddle tile edges / xb % B != 0 (response-only), and a
# head-sharded problem on strided head slices of full-width tensors
for cfg in (base.with_(prompt_len=50, response_len=334, block_size=48, repeat_prompt=0),
            base.with_(prompt_len=36, response_len=264, block_size=12, n_copies=2)):
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, do = [x.cuda() for x in attn_inputs(cfg)]
    o, lse = bd.attn_fwd(prob, q, k, v)
    bd.attn_bwd(prob, q, k, v, o, lse, do)
# a small SDAR-8B-like slice: one sequence, GQA 4, L = 2,048, B = 4
cfg = base.with_(batch=1, n_q_heads=4, n_kv_heads=1, prompt_len=256, response_len=1792, block_size=4)
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = [x.cuda() for x in attn_inputs(cfg)]
o, lse = bd.attn_fwd(prob, q, k, v)
bd.attn_bwd(prob, q, k, v, o, lse, do)
cfg = base.with_(n_q_heads=8, n_kv_heads=4)
full = bd.Problem.from_cfg(cfg)
q, k, v, do = [x.cuda() for x in attn_inputs(cfg)]
sh = full.head_shard(1, 2)
qs, dos = sh.head_slice_q(q), sh.head_slice_q(do)
ks, vs = sh.head_slice_kv(k), sh.head_slice_kv(v)
o, lse = bd.attn_fwd(sh, qs, ks, vs)
bd.attn_bwd(sh, qs, ks, vs, o, lse, dos)
z, t = logits_inputs(64, 1024, seed=1)
z, t = z.cuda(), t.cuda()
logp, lz = ops.logprob(z, t)
w = torch.randn(64, device="cuda")
ops.logprob_bwd(z, t, lz, w)
ops.logprob(z.clone(), t, dlogp=w, dlogits=torch.empty_like(z))
# the Qwen3 vocabulary: the fused kernel with register-held slice tails
zq, tq = logits_inputs(8, 151936, seed=4)
zq, tq = zq.cuda(), tq.cuda()
ops.logprob(zq, tq, dlogp=torch.randn(8, device="cuda"), dlogits=torch.empty_like(zq))
# the opt-in stored-dS backward, two chunks of one sequence
cfg = base.with_(batch=2)
prob = bd.Problem.from_cfg(cfg)
os.environ["BD_BWD_DS"], os.environ["BD_BWD_DS_BUDGET_MB"] = "1", "1"
q, k, v, do = [x.cuda() for x in attn_inputs(cfg)]
o, lse = bd.attn_fwd(prob, q, k, v)
bd.attn_bwd(prob, q, k, v, o, lse, do)
os.environ["BD_BWD_DS"] = "0"
rew = torch.tensor([1.0, 0.0], device="cuda")
gid = torch.zeros(2, dtype=torch.int32, device="cuda")
tl = torch.full((2,), 32, dtype=torch.int32, device="cuda")
tok = torch.arange(2, device="cuda", dtype=torch.int32).repeat_interleave(32)
dipo.dipo_loss(logp, logp.clone(), tok, rew, gid, tl, 1)
h, W, tt, ww = [x.cuda() for x in lmhead_inputs(300, 256, 1000, seed=2)]
lp, ls = ops.lmhead_logprob(h, W, tt)
ops.lmhead_logprob_bwd(h, W, tt, ls, ww, chunk_rows=128)
qd, kc, vc, kvl = [x.cuda() for x in decode_inputs(2, 4, 4, 2, 128, 300, seed=3)]
ops.decode_attn(qd, kc, vc, kvl)
zz = torch.randn((2, 4, 512), device="cuda").to(torch.bfloat16)
ops.decode_select(zz, torch.ones((2, 4), dtype=torch.uint8, device="cuda"), 0.9)
torch.cuda.synchronize()
print("sanitize run ok", ops.launch_count(), "launches")
