"""Per-unit timeline of the (persistent) dQ kernel (run with BD_TRACE=2): how
much of the kernel's span the SMs' compute warps spend inside work units, and
per-unit cost vs tile count (fixed overhead + per-tile time, least squares).
Dev diagnostic.  (The one-CTA-per-unit kernel it was first written for gave
98.3% busy, ~5.3 us + 1.13 us per tile at SDAR-8B batch 2.)"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import _lib
from workloads import CONFIGS, attn_inputs

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = CONFIGS["sdar_8b"].with_(batch=batch)
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = attn_inputs(cfg, device="cuda")
o, lse = bd.attn_fwd(prob, q, k, v)
for _ in range(3):
    bd.attn_bwd(prob, q, k, v, o, lse, do)
torch.cuda.synchronize()
n = 144 * batch * 32
buf = (ctypes.c_int64 * (4 * n))()
assert _lib.lib().bd_debug_cta_timeline(buf, 4 * n) == 0
t = np.array(buf, dtype=np.int64).reshape(n, 4)
t0, t1, nk, sm = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
span = t1.max() - t0.min()
dur = t1 - t0
print(f"units {n}, span {span / 1e3:.1f} us, mean unit {dur.mean() / 1e3:.2f} us, tiles/unit {nk.mean():.1f}")
busy = np.zeros(sm.max() + 1)
np.add.at(busy, sm, dur)
print(f"SM busy fraction of span: mean {busy.mean() / span:.3f} min {busy.min() / span:.3f}")
A = np.stack([np.ones(n), nk], 1)
coef, *_ = np.linalg.lstsq(A, dur.astype(float), rcond=None)
print(f"duration ~ {coef[0] / 1e3:.2f} us + {coef[1] / 1e3:.3f} us x tiles; fixed share {coef[0] * n / dur.sum():.3f}")
# gaps between consecutive CTAs on one SM
gaps = []
for s_ in np.unique(sm):
    idx = np.where(sm == s_)[0]
    o_ = np.argsort(t0[idx])
    a0, a1 = t0[idx][o_], t1[idx][o_]
    gaps += list(a0[1:] - a1[:-1])
gaps = np.array(gaps)
print(f"gap between units on an SM: median {np.median(gaps) / 1e3:.2f} us, mean {gaps.mean() / 1e3:.2f} us")
for lo, hi in [(1, 5), (5, 20), (20, 40), (40, 80)]:
    m = (nk >= lo) & (nk < hi)
    if m.any():
        print(f"tiles [{lo},{hi}): {m.sum()} CTAs, us/tile {np.mean(dur[m] / nk[m]) / 1e3:.3f}")
