"""Time bd_decode_attn at a DECODE_SHAPES config:
CUDA events, median of reps; algorithmic bytes = the K/V cache rows each
sequence reads (sum_b kv_len_b x Hkv x d x 2 B x 2) + q + o."""
import json, sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_22234_b200 import ops
from workloads import decode_inputs, DECODE_SHAPES

name = sys.argv[1] if len(sys.argv) > 1 else "sdar_8b"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
sh = DECODE_SHAPES[name]
q, k, v, kv_len = decode_inputs(**sh, device="cuda", seed=21, min_len=1028)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
o, lse = ops.decode_attn(q, k, v, kv_len)
ts = []
for i in range(reps + 3):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ops.decode_attn(q, k, v, kv_len, o=o, lse=lse)
    e1.record(st)
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
byts = int(kv_len.sum().item()) * sh["n_kv_heads"] * sh["head_dim"] * 4 + 2 * q.numel() * 2
print(json.dumps({"workload": f"decode_{name}", **sh, "mean_kv_len": float(kv_len.float().mean()),
                  "ms": round(ms, 4), "GBps": round(byts / ms / 1e6, 1), "bytes": byts}))
