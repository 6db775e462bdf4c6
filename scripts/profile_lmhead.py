"""One forward + backward of the fused LM head at a LMHEAD_SHAPES config, for
ncu (--set full -k regex:gemm2sm|lse_combine)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_22234_b200 import ops
from workloads import lmhead_inputs, LMHEAD_SHAPES
name = sys.argv[1] if len(sys.argv) > 1 else "sdar_1_7b"
n, C, V = LMHEAD_SHAPES[name]
h, W, t, w = lmhead_inputs(n, C, V, device="cuda", seed=7)
logp, lse = ops.lmhead_logprob(h, W, t)
ops.lmhead_logprob_bwd(h, W, t, lse, w, chunk_rows=n)
torch.cuda.synchronize()
print("ok", name)
