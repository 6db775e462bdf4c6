"""Pass timings of the device tile-map builder (dev diagnostic; needs a build
with -DBD_MAP_TRACE=1, e.g. BD_NVCC_EXTRA=-DBD_MAP_TRACE=1 BD_LIB_OUT=...)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import _lib, ops
from workloads import CONFIGS

cfg = CONFIGS["sdar_8b"].with_(batch=1, n_q_heads=1, n_kv_heads=1)
prob = bd.Problem.from_cfg(cfg)
N = bd.packed_len(prob)
q = torch.zeros((1, N, 1, 128), dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    ops.attn_fwd(prob, q, q, q)
torch.cuda.synchronize()
buf = (ctypes.c_int64 * 8)()
assert _lib.lib().bd_debug_map_trace(buf, 8) == 0
t = list(buf)
names = ["init", "pass1 classify", "row scan", "pass2 fill", "(nothing)", "col scan", "pass3 columns", "pass4 LPT"]
for i in range(1, 8):
    print(f"{names[i]:16s} {t[i] - t[i - 1]:8d} clk")
print("total", t[7] - t[0])
