"""One hot-path step at a reduced batch for ncu captures (never a bench value).

    ncu --set full -k regex:attn_ -c 2 python scripts/profile_step.py [config] [batch]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_22234_b200 as bd  # noqa: E402
from paper_2512_22234_b200 import ops  # noqa: E402
from workloads import CONFIGS, attn_inputs, logits_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sdar_8b"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = CONFIGS[name].with_(batch=batch)
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = attn_inputs(cfg, device="cuda")
o, lse = bd.attn_fwd(prob, q, k, v)
dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
z, t = logits_inputs(2048, 151936, device="cuda")
logp, lz = ops.logprob(z, t)
ops.logprob_bwd(z, t, lz, torch.ones_like(logp), dlogits=z)
ops.logprob(z, t, dlogp=torch.ones_like(logp), dlogits=z)  # cluster-fused path
torch.cuda.synchronize()
print("done", name, batch)
