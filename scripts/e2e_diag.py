"""Dev diagnostic: where the end-to-end step's time goes (compute alone, with
concurrent H2D of the next inputs, with concurrent D2H of the gradients, both)."""
import sys, os, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

job = bench.JOBS["sdar_8b"]
step = bench.Step(job, 0, 1)
names_in = ("q", "k", "v", "do", "targets")
names_out = ("dq", "dk", "dv")
host_in = {n: torch.empty(getattr(step, n).shape, dtype=getattr(step, n).dtype, pin_memory=True) for n in names_in}
host_out = {n: torch.empty(getattr(step, n).shape, dtype=getattr(step, n).dtype, pin_memory=True) for n in names_out}
spare = {n: torch.empty_like(getattr(step, n)) for n in names_in}
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def run(n, h2d, d2h):
    main = torch.cuda.current_stream()
    for _ in range(2):
        step.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        if h2d:
            s_in.wait_stream(main)
            with torch.cuda.stream(s_in):
                for nm in names_in:
                    spare[nm].copy_(host_in[nm], non_blocking=True)
        step.run()
        if d2h:
            s_out.wait_stream(main)
            with torch.cuda.stream(s_out):
                for nm in names_out:
                    host_out[nm].copy_(getattr(step, nm), non_blocking=True)
    main.wait_stream(s_in)
    main.wait_stream(s_out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for h2d, d2h in ((0, 0), (1, 0), (0, 1), (1, 1)):
    print(f"h2d {h2d} d2h {d2h}: {run(6, h2d, d2h):.1f} ms per step")

# the bench's own e2e pipeline, for comparison
args = types.SimpleNamespace(steps=6, warmup=3, no_e2e=False)
f, fb = bench.rank_flops(job, 1, 0)
r = bench.run_e2e(step, args, 1, f + fb)
print("bench.run_e2e:", r["ms_per_step"], "ms per step,", r["value"], "TF/s")
