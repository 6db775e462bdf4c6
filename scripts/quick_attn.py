"""Quick fwd / bwd timing at a BJ config (dev helper; bench.py is the contract).
Reports the median of 5 repeats of 4 back-to-back calls each."""
import statistics
import sys
import torch
import paper_2512_22234_b200 as bd
from workloads import CONFIGS, attn_inputs, useful_flops

name = sys.argv[1] if len(sys.argv) > 1 else "sdar_8b"
cfg = CONFIGS[name]
prob = bd.Problem.from_cfg(cfg)
q, k, v, do = attn_inputs(cfg, device="cuda")
o, lse = bd.attn_fwd(prob, q, k, v)
dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
torch.cuda.synchronize()


def timeit(fn, n=4, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(n):
            fn()
        en.record()
        torch.cuda.synchronize()
        out.append(st.elapsed_time(en) / n)
    return statistics.median(out), min(out)


f, fb = useful_flops(cfg)
tf, tfm = timeit(lambda: bd.attn_fwd(prob, q, k, v, o, lse))
tb, tbm = timeit(lambda: bd.attn_bwd(prob, q, k, v, o, lse, do, dq, dk, dv))
print(f"{name}: fwd {tf:.3f} ms (min {tfm:.3f}) {f/tf/1e9:.0f} TF/s | bwd {tb:.3f} ms (min {tbm:.3f}) "
      f"{fb/tb/1e9:.0f} TF/s | fwd+bwd {(f+fb)/(tf+tb)/1e9:.0f} TF/s")
