"""Print the dK/dV kernel's event trace (run with BD_TRACE=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import _lib
from workloads import CONFIGS, attn_inputs

cfg = CONFIGS["sdar_8b"].with_(batch=1)
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = attn_inputs(cfg, device="cuda")
o, lse = bd.attn_fwd(prob, q, k, v)
for _ in range(2):
    bd.attn_bwd(prob, q, k, v, o, lse, do)
torch.cuda.synchronize()
buf = (ctypes.c_int64 * 8192)()
_lib.lib().bd_debug_trace(buf, 8192)
t = list(buf)
print("compute: vec s_full p1end dp_full ds_arrive | mma: p1 pt dvwait ds dOfull dkissued Qfull | tma issue Q(i+1) dO(i+1) | period")
for i in range(20, 34):
    c = t[8 * i: 8 * i + 5]
    m = t[1024 + 8 * i: 1024 + 8 * i + 7]
    p = t[2048 + 8 * (i + 1): 2048 + 8 * (i + 1) + 2]
    z = m[0]
    print(i, [x - z for x in c], [x - z for x in m], [x - z for x in p], m[0] - t[1024 + 8 * (i - 1)])
