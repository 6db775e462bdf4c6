"""Quick timing of the fused logprob forward + gradient at the SDAR-8B shape (dev helper)."""
import statistics, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_22234_b200 import ops
n, V = int(sys.argv[1]) if len(sys.argv) > 1 else 131072, 151936
z = torch.empty((n, V), dtype=torch.bfloat16, device="cuda")
for r0 in range(0, n, 8192):
    z[r0:r0 + 8192].normal_(0, 3)
t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32)
w = torch.randn(n, device="cuda")
ts = []
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.logprob(z, t, dlogp=w, dlogits=z)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(f"logprob fused {n}x{V}: {ms:.3f} ms, {4 * n * V / ms / 1e6:.0f} GB/s")
