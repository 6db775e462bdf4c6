"""Print the forward kernel's event trace (run with BD_TRACE=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import _lib
from workloads import CONFIGS, attn_inputs

cfg = CONFIGS["sdar_8b"].with_(batch=2)
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = attn_inputs(cfg, device="cuda")
for _ in range(3):
    bd.attn_fwd(prob, q, k, v)
torch.cuda.synchronize()
buf = (ctypes.c_int64 * 8192)()
_lib.lib().bd_debug_trace_fwd(buf, 8192)
t = list(buf)
print("softmax q0: start s_full p_arrive | q1: start s_full p_arrive || mma: V(j) P0 P1 S0(j+1) S1(j+1) | period")
for j in range(20, 36):
    s0 = t[8 * j: 8 * j + 3]
    s1 = t[8 * j + 4: 8 * j + 7]
    m = t[1024 + 8 * j: 1024 + 8 * j + 5]
    z = m[0]
    print(j, [x - z for x in s0], [x - z for x in s1], [x - z for x in m], m[0] - t[1024 + 8 * (j - 1)])
