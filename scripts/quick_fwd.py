"""Quick forward timing at a BJ config (dev helper; bench.py is the contract)."""
import sys, time
import torch
import paper_2512_22234_b200 as bd
from workloads import CONFIGS, attn_inputs, useful_flops

name = sys.argv[1] if len(sys.argv) > 1 else "sdar_8b"
cfg = CONFIGS[name]
prob = bd.Problem.from_cfg(cfg)
q, k, v, _ = attn_inputs(cfg, device="cuda", with_do=False)
o, lse = bd.attn_fwd(prob, q, k, v)
torch.cuda.synchronize()
for _ in range(2):
    bd.attn_fwd(prob, q, k, v, o, lse)
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 5
st.record()
for _ in range(n):
    bd.attn_fwd(prob, q, k, v, o, lse)
en.record()
torch.cuda.synchronize()
ms = st.elapsed_time(en) / n
f, _ = useful_flops(cfg)
print(f"{name}: fwd {ms:.3f} ms  {f / ms / 1e9:.1f} TFLOP/s useful")
