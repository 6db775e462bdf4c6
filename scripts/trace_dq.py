"""Print the dQ kernel's event trace (run with BD_TRACE=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import _lib
from workloads import CONFIGS, attn_inputs

cfg = CONFIGS["sdar_8b"].with_(batch=2)
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = attn_inputs(cfg, device="cuda")
o, lse = bd.attn_fwd(prob, q, k, v)
for _ in range(2):
    bd.attn_bwd(prob, q, k, v, o, lse, do)
torch.cuda.synchronize()
buf = (ctypes.c_int64 * 8192)()
_lib.lib().bd_debug_trace(buf, 8192)
t = list(buf)
print("compute(j): s_full p1end dp_full dp_read done | mma: dP(j) issue, dQ(j) issue, S(j) issue | period (dP issues)")
for j in range(20, 34):
    c = t[4096 + 8 * j: 4096 + 8 * j + 5]
    c = [c[0], c[4], c[1], c[2], c[3]]
    m = t[5120 + 8 * j: 5120 + 8 * j + 3]
    z = m[0]
    print(j, [x - z for x in c], [x - z for x in m], m[0] - t[5120 + 8 * (j - 1)])
