"""Per-CTA timeline of the dK/dV kernel (run with BD_TRACE=3): SM busy
fraction over the kernel span and the tail (time from the first SM going idle
for good to the kernel end).  Dev diagnostic."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import _lib
from workloads import CONFIGS, attn_inputs

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = CONFIGS["sdar_8b"].with_(batch=batch)
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = attn_inputs(cfg, device="cuda")
o, lse = bd.attn_fwd(prob, q, k, v)
for _ in range(2):
    bd.attn_bwd(prob, q, k, v, o, lse, do)
torch.cuda.synchronize()
n = 144 * batch * 8
buf = (ctypes.c_int64 * (4 * n))()
assert _lib.lib().bd_debug_cta_timeline(buf, 4 * n) == 0
t = np.array(buf, dtype=np.int64).reshape(n, 4)
t0, t1, nit, sm = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
span = t1.max() - t0.min()
busy = np.zeros(sm.max() + 1)
np.add.at(busy, sm, t1 - t0)
last_end = np.zeros(sm.max() + 1)
np.maximum.at(last_end, sm, t1 - t0.min())
print(f"CTAs {n}, span {span / 1e3:.1f} us, SM busy fraction mean {busy.mean() / span:.3f}")
print(f"SM finish times (us from start): min {last_end.min() / 1e3:.1f}, median {np.median(last_end) / 1e3:.1f}, max {last_end.max() / 1e3:.1f}")
dur = (t1 - t0)
A = np.stack([np.ones(n), nit], 1)
coef, *_ = np.linalg.lstsq(A, dur.astype(float), rcond=None)
print(f"duration ~ {coef[0] / 1e3:.2f} us + {coef[1] / 1e3:.4f} us x iterations; longest CTA {dur.max() / 1e3:.1f} us")
