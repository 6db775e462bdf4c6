"""One fwd+bwd at a BJ config (for ncu launch lists; never a bench value)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_22234_b200 as bd
from workloads import CONFIGS, attn_inputs
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "sdar_8b"]
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = attn_inputs(cfg, device="cuda")
for _ in range(2):
    o, lse = bd.attn_fwd(prob, q, k, v)
    bd.attn_bwd(prob, q, k, v, o, lse, do)
torch.cuda.synchronize()
