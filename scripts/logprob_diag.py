"""Fused logprob timing under different power states (dev helper).

  python scripts/logprob_diag.py [n_rows]

Prints the median time of the fused kernel (131,072 x 151,936 by default)
  * cold: standalone, in place (dz over z) and to a separate buffer,
  * hot: each launch right after ~25 ms of bf16 GEMMs (the forward's power
    draw in the bench step), with the SM clock sampled by NVML.
"""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_22234_b200 import ops

try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
except Exception:  # noqa: BLE001
    _h = None


def clocks_during(fn):
    samples, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            if _h is not None:
                samples.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.01)

    th = threading.Thread(target=poll)
    th.start()
    try:
        r = fn()
    finally:
        stop.set()
        th.join()
    return r, (statistics.median(samples) if samples else None)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
V = 151936
z = torch.empty((n, V), dtype=torch.bfloat16, device="cuda")
for r0 in range(0, n, 8192):
    z[r0:r0 + 8192].normal_(0, 3)
dz = torch.empty_like(z)
t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32)
w = torch.randn(n, device="cuda")
a = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
bm = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
cm = torch.empty(8192, 8192, dtype=torch.bfloat16, device="cuda")


def timed(pre, out, reps):
    ts = []
    for i in range(reps):
        for _ in range(pre):
            torch.matmul(a, bm, out=cm)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.logprob(z, t, dlogp=w, dlogits=out)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


cases = (("cold in-place", 0, z, 8), ("cold separate", 0, dz, 8),
         ("sustained separate", 0, dz, 60), ("after 36 GEMMs separate", 36, dz, 12))
if os.environ.get("LP_SHORT"):
    cases = (cases[1], cases[3])
for name, pre, out, reps in cases:
    ms, mhz = clocks_during(lambda: timed(pre, out, reps))
    print(f"{name:28s} {ms:7.3f} ms  {4 * n * V / ms / 1e6:6.0f} GB/s  sm {mhz} MHz", flush=True)
