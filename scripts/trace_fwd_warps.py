"""Per-warp forward event trace (dev helper; build with -DBD_FWD_WTRACE, run with BD_TRACE=1).
For tiles 20-27 of CTA 0 (SDAR-8B heads, batch 2), relative to the MMA thread's
V(j) wait: per softmax warp, [s_full seen, max done, p_half arrived, P stored, S loaded, first P part issued],
and the MMA thread's [V wait start, p_half[0] seen, p_full[0] seen, p_half[1] seen, p_full[1] seen]."""
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
for j in range(20, 28):
    z = t[1024 + 8 * j]
    mma = t[3072 + 8 * (j & 15): 3072 + 8 * (j & 15) + 3]
    print(f"tile {j}: mma Vwait {mma[0] - z}, p_half0 {mma[1] - z}, p_full0 {t[1024 + 8 * j + 1] - z}, "
          f"p_half1 {mma[2] - z}, p_full1 {t[1024 + 8 * j + 2] - z}, S0 {t[1024 + 8 * j + 3] - z}, S1 {t[1024 + 8 * j + 4] - z}")
    for w in range(8):
        e = t[2048 + 64 * (j & 15) + 8 * w: 2048 + 64 * (j & 15) + 8 * w + 6]
        print(f"   warp {w} (q{w // 4}): " + " ".join(f"{x - z:6d}" for x in e))
# split-row softmax (NQ = 2): every warp takes both heads; slots 4096 + 128 (j % 16) + 16 warp + 4 q + e
if any(t[4096:4096 + 2048]):
    print("split rows: per warp [s_full seen, max exchanged, p_half arrived, P stored] for q0 | q1")
    for j in range(20, 28):
        z = t[1024 + 8 * j]
        mma = t[3072 + 8 * (j & 15): 3072 + 8 * (j & 15) + 3]
        print(f"tile {j}: mma Vwait {mma[0] - z}, p_half0 {mma[1] - z}, p_full0 {t[1024 + 8 * j + 1] - z}, "
              f"p_half1 {mma[2] - z}, p_full1 {t[1024 + 8 * j + 2] - z}, S0 {t[1024 + 8 * j + 3] - z}, "
              f"S1 {t[1024 + 8 * j + 4] - z}")
        for w in range(8):
            b = 4096 + 128 * (j & 15) + 16 * w
            e0 = [x - z for x in t[b: b + 4]]
            e1 = [x - z for x in t[b + 4: b + 8]]
            print(f"   warp {w} (h{w // 4}): " + " ".join(f"{x:6d}" for x in e0) + "  | " + " ".join(f"{x:6d}" for x in e1))
