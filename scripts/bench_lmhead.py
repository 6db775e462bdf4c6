"""Time the fused LM head + logprob at a LMHEAD_SHAPES
config: forward (bd_lmhead_logprob) and backward (bd_lmhead_logprob_bwd),
CUDA events on the launching stream, median of the timed reps.
Useful FLOPs: forward 2 n C V; backward 3 x forward (logit recompute, dh, dW).
Prints one JSON line."""
import json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_22234_b200 import ops
from workloads import lmhead_inputs, LMHEAD_SHAPES

name = sys.argv[1] if len(sys.argv) > 1 else "sdar_8b"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
n, C, V = LMHEAD_SHAPES[name]
h, W, t, w = lmhead_inputs(n, C, V, device="cuda", seed=7)
st = torch.cuda.current_stream()


def timed(fn):
    ts = []
    for i in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


logp, lse = ops.lmhead_logprob(h, W, t)
dh = torch.empty_like(h)
dw = torch.empty((V, C), dtype=torch.float32, device="cuda")
fwd_ms, fwd_min = timed(lambda: ops.lmhead_logprob(h, W, t))
bwd_ms, bwd_min = timed(lambda: ops.lmhead_logprob_bwd(h, W, t, lse, w, chunk_rows=chunk, dh=dh, dw=dw))
F = 2.0 * n * C * V
print(json.dumps({"workload": f"lmhead_{name}", "n_rows": n, "hidden": C, "vocab": V, "chunk_rows": chunk,
                  "fwd_ms": round(fwd_ms, 3), "fwd_tflops": round(F / fwd_ms / 1e9, 1),
                  "bwd_ms": round(bwd_ms, 3), "bwd_tflops": round(3 * F / bwd_ms / 1e9, 1),
                  "fwd_min_ms": round(fwd_min, 3), "bwd_min_ms": round(bwd_min, 3),
                  "logits_bytes_avoided": n * V * 2}))
