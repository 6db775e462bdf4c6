#!/usr/bin/env python
"""bench.py -- one JSON line for the DiRL/DiPO block-diffusion hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config sdar_8b] [--impl ours|reference]

A STEP is one pass of the whole hot path over one batch of
synthetic, device-resident inputs, per rank:
    bd_attn_fwd (tile map a1 + a2) -> DiPO group stats + token weights + NCCL
    all-reduce of the scalar partials (a7; online update, rho == 1, Eq. 7) ->
    bd_logprob forward + gradient fused in one pass, in place (a6 + a8) ->
    bd_attn_bwd (a3-a5, tile map rebuilt on device).
The transformer between attention and the logits is the caller's (out of
scope): the logits are a resident synthetic stand-in for the LM-head output at
the response positions (N = b R rows x V = 151,936).

Metric (BASELINE.json): bd-attn fwd+bwd useful TFLOP/s (& % BF16 peak) and
train tokens/s.  `value` = useful attention FLOPs of the step summed over all
ranks / step time (max over ranks), i.e. the whole step's time including
logprob and DiPO.  Useful FLOPs count only visible (query, key) pairs:
fwd = 4 d Hq b pairs, bwd = 2.5 fwd, pairs = L (L + B), or
(1 + S) L (L + B) / 2 for the trace-replay config with S noisy copies.
Multi-GPU: one process per GPU (torchrun), each rank runs its own GRPO
group(s) of sequences -> weak scaling; NCCL only all-reduces DiPO scalars.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIGS, VOCAB_QWEN3, useful_flops, useful_pairs  # noqa: E402

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {k: float(d[k]) for k in FALLBACK_PEAKS}, "measured"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sms, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


# ------------------------------------------------------------------ setup
def dist_setup(gpus, backend="nccl"):
    """One process per GPU.  backend="gloo" with BD_BENCH_SHARE_GPU=1 maps every
    rank onto cuda:0 -- a dry run of the multi-rank path on a 1-GPU box (NCCL
    refuses two ranks on one GPU); never a scaling measurement."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        if os.environ.get("BD_BENCH_SHARE_GPU") == "1":
            local = 0
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    if gpus != world and rank == 0:
        print(f"[bench] warning: --gpus {gpus} but WORLD_SIZE {world}", file=sys.stderr)
    return world, rank, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def barrier(world):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


class Step:
    """Device-resident buffers and one hot-path step for this rank."""

    def __init__(self, cfg, rank, world):
        import paper_2512_22234_b200 as bd
        from paper_2512_22234_b200 import ops
        self.bd, self.ops = bd, ops
        self.cfg, self.rank, self.world = cfg, rank, world
        self.prob = bd.Problem.from_cfg(cfg)
        dev = torch.device("cuda")
        g = torch.Generator(device=dev)
        g.manual_seed(cfg.seed * 1000 + rank)
        N, b = cfg.ntot, cfg.batch
        sq, sk = (b, N, cfg.n_q_heads, cfg.head_dim), (b, N, cfg.n_kv_heads, cfg.head_dim)
        self.q = torch.randn(sq, generator=g, device=dev, dtype=torch.bfloat16)
        self.k = torch.randn(sk, generator=g, device=dev, dtype=torch.bfloat16)
        self.v = torch.randn(sk, generator=g, device=dev, dtype=torch.bfloat16)
        self.do = torch.randn(sq, generator=g, device=dev, dtype=torch.bfloat16)
        self.o = torch.empty_like(self.q)
        self.lse = torch.empty((b, cfg.n_q_heads, N), dtype=torch.float32, device=dev)
        self.dq, self.dk, self.dv = torch.empty_like(self.q), torch.empty_like(self.k), torch.empty_like(self.v)
        # logits stand-in for the response rows (the LM head is the caller's)
        self.V = VOCAB_QWEN3
        self.n_rows = b * cfg.response_len
        self.logits = torch.empty((self.n_rows, self.V), dtype=torch.bfloat16, device=dev)
        for r0 in range(0, self.n_rows, 4096):
            r1 = min(self.n_rows, r0 + 4096)
            self.logits[r0:r1] = torch.randn((r1 - r0, self.V), generator=g, device=dev) * 3.0
        self.targets = torch.randint(0, self.V, (self.n_rows,), generator=g, device=dev, dtype=torch.int32)
        # one GRPO group of b trajectories per rank (global group id = rank)
        self.rewards = torch.bernoulli(torch.full((b,), 0.5, device=dev), generator=g).float()
        self.group_of_traj = torch.full((b,), rank, dtype=torch.int32, device=dev)
        self.traj_len = torch.full((b,), cfg.response_len, dtype=torch.int32, device=dev)
        self.traj_of_token = torch.arange(b, device=dev, dtype=torch.int32).repeat_interleave(cfg.response_len)
        self.n_groups = world
        self.loss = None
        torch.cuda.synchronize()

    def run(self, ev=None):
        """One step.  ev: optional list of 6 CUDA events bracketing the phases."""
        from paper_2512_22234_b200 import dipo
        bd, ops = self.bd, self.ops
        rec = (lambda i: ev[i].record()) if ev is not None else (lambda i: None)
        rec(0)
        bd.attn_fwd(self.prob, self.q, self.k, self.v, self.o, self.lse)
        rec(1)
        # DiRL's online update: pi_old = sg(pi_theta) (Eq. 7), so rho == 1 and
        # the DiPO token weights are known before the log-probs; one fused logprob pass
        # (forward + gradient, in place) follows.
        loss, dlogp, parts = dipo.dipo_loss(None, None, self.traj_of_token, self.rewards,
                                            self.group_of_traj, self.traj_len, self.n_groups, straddle=False)
        rec(2)
        self.logp, _, _ = ops.logprob(self.logits, self.targets, dlogp=dlogp, dlogits=self.logits)
        rec(3)
        rec(4)
        bd.attn_bwd(self.prob, self.q, self.k, self.v, self.o, self.lse, self.do, self.dq, self.dk, self.dv)
        rec(5)
        self.loss = parts
        return parts


def run_ours(args):
    world, rank, local = dist_setup(args.gpus, args.dist_backend)
    cfg = CONFIGS[args.config]
    peaks, peak_src = load_peaks()
    step = Step(cfg, rank, world)
    ops = step.ops
    fwd_f, bwd_f = useful_flops(cfg)
    flops_step = (fwd_f + bwd_f)  # per rank
    tokens_step = cfg.batch * cfg.L
    for _ in range(args.warmup):
        step.run()
    barrier(world)

    # ---- device-resident timed region
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = ops.launch_count()
    with ClockSampler(local) as clk:
        barrier(world)
        start.record()
        for i in range(args.steps):
            step.run(evs[i])
        end.record()
        barrier(world)
    launches = (ops.launch_count() - n0) // args.steps
    ms_local = start.elapsed_time(end) / args.steps
    ms = max_over_ranks(ms_local, world)
    phase = {n: statistics.mean(e[i].elapsed_time(e[i + 1]) for e in evs)
             for i, n in enumerate(["attn_fwd", "dipo", "logprob_fused", "unused", "attn_bwd"])}
    phase.pop("unused")
    loss_val = float(step.loss[0].item())

    # ---- end-to-end through the public API with pinned host buffers.  Every
    # step's inputs are copied H2D inside the timed region and its loss partials
    # read back D2H; the copy of step i+1 runs on a side stream into the second
    # of two device input buffers while step i computes (double buffering).
    e2e = None
    e2e_ok = not args.no_e2e
    if e2e_ok:
        names = ("q", "k", "v", "do", "targets", "rewards")
        try:  # pinned host inputs (~6 GB per rank at SDAR-8B); agreed across ranks before any collective
            host = {n: torch.empty(getattr(step, n).shape, dtype=getattr(step, n).dtype, pin_memory=True)
                    for n in names}
        except Exception as ex:  # noqa: BLE001 -- reported, the device-resident line still prints
            print(f"[bench] e2e skipped: pinned host allocation failed: {ex}", file=sys.stderr)
            e2e_ok = False
        if world > 1:
            flag = torch.tensor([1 if e2e_ok else 0], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            e2e_ok = bool(flag.item())
    if e2e_ok:
        for n, h in host.items():
            h.copy_(getattr(step, n))
        bufs = [{n: getattr(step, n) for n in names}, {n: torch.empty_like(getattr(step, n)) for n in names}]
        out_host = torch.empty((2, 3), dtype=torch.float64, pin_memory=True)
        h2d = sum(h.numel() * h.element_size() for h in host.values())
        d2h = out_host[0].numel() * out_host.element_size()
        e2e_steps = max(2, min(args.steps, 8))
        main, side = torch.cuda.current_stream(), torch.cuda.Stream()
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]

        def copy_in(slot):
            side.wait_event(free[slot])
            with torch.cuda.stream(side):
                for n, h in host.items():
                    bufs[slot][n].copy_(h, non_blocking=True)
                copied[slot].record(side)

        def run_e2e(n_steps):
            for ev in free:
                ev.record(main)
            copy_in(0)
            for i in range(n_steps):
                cur = i % 2
                if i + 1 < n_steps:
                    copy_in(1 - cur)
                main.wait_event(copied[cur])
                for n in names:
                    setattr(step, n, bufs[cur][n])
                parts = step.run()
                out_host[cur].copy_(parts, non_blocking=True)
                free[cur].record(main)

        run_e2e(2)  # warm path
        barrier(world)
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        es.record()
        run_e2e(e2e_steps)
        ee.record()
        barrier(world)
        for n in names:
            setattr(step, n, bufs[0][n])
        e2e_ms = max_over_ranks(es.elapsed_time(ee) / e2e_steps, world)
        e2e = {"value": round(world * flops_step / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
               "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": e2e_steps,
               "inputs": "q,k,v,dO,targets,rewards H2D from pinned host every step (side stream, double-buffered: "
                         "step i+1's copy overlaps step i); DiPO loss partials D2H every step; logits are the "
                         "caller's LM-head output and stay device-resident"}

    nxt = None
    if not args.no_next:
        # decode first: measured right after the step, before the long LM-head GEMMs
        dec = bench_decode(peaks, peak_src)
        nxt = {"lmhead_logprob": bench_lmhead(peaks, peak_src), "decode_attn": dec}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, target_s=args.cpu_seconds)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    value = world * flops_step / (ms * 1e-3) / 1e12
    attn_ms = phase["attn_fwd"] + phase["attn_bwd"]
    peak_b, peak_s = peaks["bf16_tflops"], peaks["bf16_tflops_sustained"]
    bwd_achieved = bwd_f / (phase["attn_bwd"] * 1e-3) / 1e12
    fwd_achieved = fwd_f / (phase["attn_fwd"] * 1e-3) / 1e12
    lp_bytes = step.n_rows * step.V * 2
    traffic = load_traffic() if cfg.name == "sdar_8b" else {}  # the ncu capture is at the SDAR-8B bench shape
    roofline = {"kernel": "bd_attn_bwd (attn_bwd_dkdv_kernel + attn_bwd_dqp_kernel (persistent dQ) + bwd_pre + tile map)",
                "bound": "tensor",
                "achieved": round(bwd_achieved, 1), "peak": peak_s, "unit": "TFLOP/s",
                "frac": round(bwd_achieved / peak_s, 4), "traffic": traffic.get("attn_bwd"),
                "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/ncu_traffic.json)",
                "peak_kind": f"bf16 sustained ({peak_src}); kernel timed inside a long step",
                "algorithmic": f"useful bwd FLOPs per launch = 10 d Hq b L(L+B) = {bwd_f:.4e}"}
    others = {
        "attn_fwd": {"bound": "tensor", "achieved": round(fwd_achieved, 1), "peak": peak_s, "unit": "TFLOP/s",
                     "frac": round(fwd_achieved / peak_s, 4), "frac_of_burst": round(fwd_achieved / peak_b, 4),
                     "traffic": traffic.get("attn_fwd_kernel")},
        "attn_fwd_bwd": {"achieved": round((fwd_f + bwd_f) / (attn_ms * 1e-3) / 1e12, 1), "unit": "TFLOP/s",
                         "frac_sustained": round((fwd_f + bwd_f) / (attn_ms * 1e-3) / 1e12 / peak_s, 4),
                         "frac_burst": round((fwd_f + bwd_f) / (attn_ms * 1e-3) / 1e12 / peak_b, 4)},
        "logprob_fused": {"bound": "hbm",
                          "achieved": round(2 * lp_bytes / (phase["logprob_fused"] * 1e-3) / 1e9, 1),
                          "peak": peaks["hbm_gbs"], "unit": "GB/s",
                          "frac": round(2 * lp_bytes / (phase["logprob_fused"] * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                          "algorithmic": "read + write of the bf16 logits (2 x 2 B per element)",
                          "traffic": (traffic["logprob_fused_ratio"] * 2 * lp_bytes)
                          if "logprob_fused_ratio" in traffic else None},
    }
    clocks = clk.summary()
    line = {
        "metric": "bd-attn fwd+bwd useful TFLOP/s & % BF16 peak; train tokens/s at 1/2/4/8 B200",
        "value": round(value, 2),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) q/k/v/dO, N(0,3^2) logits, Bernoulli(0.5) rewards)",
        "config": {"workload": cfg.name, "batch_per_gpu": cfg.batch, "global_batch": cfg.batch * world,
                   "n_q_heads": cfg.n_q_heads, "n_kv_heads": cfg.n_kv_heads, "head_dim": cfg.head_dim,
                   "prompt_len": cfg.prompt_len, "response_len": cfg.response_len, "block_size": cfg.block_size,
                   "packed_len": cfg.ntot, "n_copies": cfg.n_copies, "vocab": step.V, "logprob_rows_per_gpu": step.n_rows,
                   "parallelism": f"dp{world} (sequence-sharded, one GRPO group per rank)",
                   "l2": "inputs larger than L2 (q alone %.1f GB >> 126 MB)" % (step.q.numel() * 2 / 1e9)},
        "pct_bf16_peak": round(value / world / peak_s * 100, 2),
        "pct_bf16_peak_burst": round(value / world / peak_b * 100, 2),
        "peak_source": peak_src,
        "tokens_per_s": round(world * tokens_step / (ms * 1e-3), 1),
        # also response tokens/s of the step and the fused
        # logprob's rows/s inside it (its own phase time)
        "response_tokens_per_s": round(world * (sum(cfg.resp_lens) if cfg.resp_lens else cfg.batch * cfg.response_len)
                                       / (ms * 1e-3), 1),
        "logprob_rows_per_s": (round(world * step.n_rows / (phase["logprob_fused"] * 1e-3), 1)
                               if phase.get("logprob_fused") else None),
        "phase_ms": {k: round(v, 3) for k, v in phase.items()},
        "dipo_loss": loss_val,
        "roofline": roofline,
        "roofline_other": others,
        "clocks": clocks,
        "gpu_launches": int(launches) * world,
        "gpu_launches_per_rank": int(launches),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "next_rows": nxt,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def bench_lmhead(peaks, peak_src, reps=3):
    """SURVEY 8(f) NEXT #2, measured beside the step (not part of it): the fused
    LM head + logprob at the SDAR-8B shape, 131,072 response rows x hidden 4,096
    x V 151,936 (LMHEAD_SHAPES).  Useful FLOPs: fwd 2 n C V (logits never
    materialised), bwd 3 x fwd (logit recompute, dh = dz W, dW = dz^T h).
    CUDA events on the launching stream; median of `reps` after one warm-up."""
    from paper_2512_22234_b200 import ops
    from workloads import lmhead_inputs, LMHEAD_SHAPES
    n, C, V = LMHEAD_SHAPES["sdar_8b"]
    h, W, t, w = lmhead_inputs(n, C, V, device="cuda", seed=7)
    dh, dw = torch.empty_like(h), torch.empty((V, C), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()

    def timed(fn):
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    _, lse = ops.lmhead_logprob(h, W, t)
    fwd_ms = timed(lambda: ops.lmhead_logprob(h, W, t))
    bwd_ms = timed(lambda: ops.lmhead_logprob_bwd(h, W, t, lse, w, chunk_rows=16384, dh=dh, dw=dw))
    F = 2.0 * n * C * V
    peak = peaks["bf16_tflops_sustained"]
    fa, ba = F / (fwd_ms * 1e-3) / 1e12, 3 * F / (bwd_ms * 1e-3) / 1e12
    del h, W, t, w, dh, dw
    torch.cuda.empty_cache()
    return {"workload": f"lmhead_sdar_8b ({n} rows x hidden {C} x V {V})", "bound": "tensor", "unit": "TFLOP/s",
            "fwd_ms": round(fwd_ms, 3), "fwd_achieved": round(fa, 1), "fwd_frac": round(fa / peak, 4),
            "bwd_ms": round(bwd_ms, 3), "bwd_achieved": round(ba, 1), "bwd_frac": round(ba / peak, 4),
            "peak": peak, "peak_kind": f"bf16 sustained ({peak_src})",
            "algorithmic": "fwd 2 n C V, bwd 6 n C V useful FLOPs",
            "logits_bytes_not_materialised": n * V * 2}


def bench_decode(peaks, peak_src, reps=20):
    """SURVEY 8(f) NEXT #4, measured beside the step: bd_decode_attn at the 8xB200
    RL step's per-GPU rollout shape (128 sequences, SDAR-8B heads, B = 4, cache
    capacity 9,216, kv_len ~ U[1,028, 9,216] in block multiples).  HBM-bound:
    algorithmic bytes = cached K/V rows read (sum kv_len x Hkv x d x 4 B) + q + o.
    L2 flushed (256 MB write) before each timed call; median of `reps`."""
    from paper_2512_22234_b200 import ops
    from workloads import decode_inputs, DECODE_SHAPES
    sh = DECODE_SHAPES["sdar_8b"]
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
    gbs = byts / ms / 1e6
    del q, k, v, flush
    torch.cuda.empty_cache()
    return {"workload": "decode_sdar_8b (128 seqs x Hq 32 / Hkv 8 x d 128, B 4, cap 9216)", "bound": "hbm",
            "ms": round(ms, 4), "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(gbs / peaks["hbm_gbs"], 4), "peak_kind": f"HBM ({peak_src})",
            "algorithmic_bytes": byts, "l2": "flushed before each call"}


def load_traffic():
    """Per-launch DRAM bytes (dram__bytes_read.sum + write) from the committed
    ncu --set full summary, if one exists."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------- oracle baseline
def _oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def oracle_sample(cfg, n_rows, seed=0):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload:
    fwd + bwd of `n_rows` query rows of one (sequence, q-head) at the full
    packed length.  Returns (seconds, useful_flops, description)."""
    import numpy as np
    from oracle import Problem as OP, attention, mask
    prob = OP(1, cfg.prompt_len, cfg.response_len, cfg.block_size, 1, 1, cfg.head_dim, cfg.repeat_prompt,
              n_copies=cfg.n_copies)
    g = torch.Generator().manual_seed(seed)
    N, d = prob.ntot, prob.head_dim
    q = torch.randn((1, N, 1, d), generator=g).to(torch.bfloat16)
    k = torch.randn((1, N, 1, d), generator=g).to(torch.bfloat16)
    v = torch.randn((1, N, 1, d), generator=g).to(torch.bfloat16)
    do = torch.randn((1, N, 1, d), generator=g).to(torch.bfloat16)
    rows = np.linspace(0, N - 1, n_rows).astype(np.int64)
    pairs = int(mask.mask_rows(prob, rows).sum())
    t0 = time.perf_counter()
    attention.forward_rows(prob, q, k, v, 0, 0, rows)
    attention.backward_rows(prob, q, k, v, do, 0, 0, rows)
    dt = time.perf_counter() - t0
    return dt, 14 * d * pairs, f"fwd+bwd of {n_rows} of {N} query rows of one (sequence, head) of {cfg.name}"


def cpu_baseline(cfg, target_s=15.0):
    n = 256
    dt, fl, desc = oracle_sample(cfg, n)
    # scale the row count so the sample costs about target_s seconds
    n2 = int(min(cfg.ntot, max(n, n * target_s / max(dt, 1e-3))))
    if n2 > n:
        dt, fl, desc = oracle_sample(cfg, n2)
    return {"value": round(fl / dt / 1e12, 6), "unit": "TFLOP/s", "cores": _oracle_threads(), "kind": "oracle",
            "sample": desc, "seconds": round(dt, 2), "host_cpu_count": os.cpu_count()}


def run_reference(args):
    """--impl reference: the fp64 CPU oracle timed on the host cores on this
    arm's workload / metric (each step a bounded row sample)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    n_rows = args.ref_rows
    for _ in range(args.warmup):
        oracle_sample(cfg, n_rows)
    tot_t, tot_f = 0.0, 0
    desc = ""
    for i in range(args.steps):
        dt, fl, desc = oracle_sample(cfg, n_rows, seed=i)
        tot_t += dt
        tot_f += fl
    value = tot_f / tot_t / 1e12
    line = {
        "impl": "reference",
        "metric": "bd-attn fwd+bwd useful TFLOP/s & % BF16 peak; train tokens/s at 1/2/4/8 B200",
        "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot_t / args.steps, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": _oracle_threads(), "kind": "oracle",
                         "sample": desc + f" per step"},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="sdar_8b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the SURVEY 8(f) next-row measurements")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo + BD_BENCH_SHARE_GPU=1: multi-rank dry run on one GPU (not a measurement)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-rows", type=int, default=512)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("[bench] warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
