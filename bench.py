#!/usr/bin/env python
"""bench.py -- one JSON line for the DiRL/DiPO block-diffusion hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config sdar_8b] [--impl ours|reference]

A STEP is one pass of the whole hot path over one batch of
synthetic, device-resident inputs, per rank:
    DiPO group statistics + token weights + NCCL all-reduce of the scalar
    partials (a7; online update, rho == 1, Eq. 7 -- the weights are known
    before the log-probs) -> for each micro-batch of this rank's work units:
    bd_attn_fwd (tile map a1 + a2) -> bd_logprob forward + gradient fused in
    one pass (a6 + a8) -> bd_attn_bwd (a3-a5, tile map rebuilt on device).
The transformer between attention and the logits is the caller's (out of
scope): the logits are a resident synthetic stand-in for the LM-head output at
the response positions (N = R rows per sequence x V = 151,936); dlogits go to
a separate buffer, so every step reads the same N(0, 3^2) logits.

Jobs (--config): the BASELINE.json configs.  Work is partitioned over ranks
in (sequence, kv-head group) units (paper_2512_22234_b200/shard.py):
  sdar_8b (default)  SDAR-8B shape, one GRPO group of 16 per rank, weak scaling
  rl8                BJ configs[4]: 128 prompts x G = 8 = 1,024 sequences,
                     micro-batches of 16, strong scaling (128 per rank at W = 8)
  fig6               the paper's Fig. 6 run: batch 4, SDAR-8B; at W = 8
                     each rank runs 4 of one sequence's 8 kv heads (head sharding)
  sdar_8b_strong     one group of 16 split over the ranks (groups straddle)
  any other CONFIGS  one group of `batch` sequences per rank, weak scaling

Metric (BASELINE.json): bd-attn fwd+bwd useful TFLOP/s (& % BF16 peak) and
train tokens/s.  `value` = useful attention FLOPs of the whole job (all ranks)
/ step time (max over ranks), the whole step's time including logprob and
DiPO.  Useful FLOPs count only visible (query, key) pairs: fwd = 4 d Hq pairs,
bwd = 2.5 fwd, pairs = L (L + B) per sequence, (1 + S) L
(L + B) / 2 with S noisy copies.  The line also carries, measured in the same
process with clocks, every other BASELINE config (`configs`), the roofline of
the dominant kernel, an end-to-end number through the public API with host
buffers (`e2e`) and the fp64 oracle timed on the host cores (`cpu_baseline`).
"""

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import dataclass

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIGS, VOCAB_QWEN3, useful_pairs  # noqa: E402

METRIC = "bd-attn fwd+bwd useful TFLOP/s & % BF16 peak; train tokens/s at 1/2/4/8 B200"
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


# ------------------------------------------------------------------- jobs
@dataclass(frozen=True)
class Job:
    """A BASELINE workload: per-sequence attention shape + how many sequences
    the whole job has at world size W, their GRPO grouping and micro-batch."""
    name: str
    cfg: str
    scaling: str          # "weak": per-rank work fixed; "strong": whole job fixed
    n_seq_fixed: int = 0  # strong scaling: sequences of the whole job
    group: int = 0        # GRPO group size (0 = cfg.batch)
    micro_batch: int = 0  # sequences per attention launch (0 = cfg.batch)
    note: str = ""

    def attn_cfg(self):
        return CONFIGS[self.cfg]

    def n_seq(self, world):
        return self.n_seq_fixed if self.scaling == "strong" else self.attn_cfg().batch * world

    def group_size(self):
        return self.group or self.attn_cfg().batch

    def mb(self):
        return self.micro_batch or self.attn_cfg().batch


JOBS = {
    "sdar_8b": Job("sdar_8b", "sdar_8b", "weak", note="BJ configs[2]: one GRPO group of 16 per rank"),
    "rl8": Job("rl8", "sdar_8b", "strong", n_seq_fixed=1024, group=8, micro_batch=16,
               note="BJ configs[4]: 128 prompts x G 8 = 1,024 sequences, micro-batches of 16"),
    "fig6": Job("fig6", "sdar_8b", "strong", n_seq_fixed=4, group=4, micro_batch=4,
                note="P:294 Fig. 6: batch 4, input 1024, output 8192, SDAR-8B; head-sharded when W > 4"),
    "sdar_8b_strong": Job("sdar_8b_strong", "sdar_8b", "strong", n_seq_fixed=16, group=16, micro_batch=16,
                          note="one group of 16 split over the ranks (straddling group statistics)"),
}
for _n in CONFIGS:
    JOBS.setdefault(_n, Job(_n, _n, "weak", note="one group of `batch` sequences per rank"))


def seq_resp_len(cfg, s):
    """Response length of job sequence s (varlen configs repeat their pattern)."""
    return cfg.resp_lens[s % cfg.batch] if cfg.resp_lens else cfg.response_len


def piece_pairs(cfg, seqs):
    """Visible pairs per head summed over job sequences `seqs`."""
    return sum(useful_pairs(cfg.with_(response_len=seq_resp_len(cfg, s), resp_lens=None)) for s in seqs)


def rank_flops(job, world, rank):
    """Useful (fwd, bwd) FLOPs of one rank's pieces."""
    from paper_2512_22234_b200 import shard
    cfg = job.attn_cfg()
    G = cfg.n_q_heads // cfg.n_kv_heads
    f = 0
    for p in shard.plan(job.n_seq(world), cfg.n_kv_heads, world, rank, job.mb()):
        f += 4 * cfg.head_dim * p.n_kv * G * piece_pairs(cfg, range(p.seq0, p.seq1))
    return f, 2.5 * f


def job_flops(job, world):
    t = [rank_flops(job, world, r) for r in range(world)]
    return sum(a for a, _ in t), sum(b for _, b in t)


class Step:
    """Device-resident buffers and one hot-path step for this rank."""

    def __init__(self, job, rank, world):
        import paper_2512_22234_b200 as bd
        from paper_2512_22234_b200 import ops, shard
        self.bd, self.ops = bd, ops
        self.job, self.rank, self.world = job, rank, world
        cfg = self.cfg = job.attn_cfg()
        self.n_seq = job.n_seq(world)
        Hkv, Hq, d, N = cfg.n_kv_heads, cfg.n_q_heads, cfg.head_dim, cfg.ntot
        self.G = Hq // Hkv
        self.pieces = shard.plan(self.n_seq, Hkv, world, rank, job.mb())
        self.straddle = shard.groups_straddle(self.n_seq, job.group_size(), world, Hkv)
        mbs = max([p.n_seq for p in self.pieces] + [1])
        dev = torch.device("cuda")
        g = torch.Generator(device=dev)
        g.manual_seed(cfg.seed * 1000 + rank)
        sq, sk = (mbs, N, Hq, d), (mbs, N, Hkv, d)
        self.q = torch.randn(sq, generator=g, device=dev, dtype=torch.bfloat16)
        self.k = torch.randn(sk, generator=g, device=dev, dtype=torch.bfloat16)
        self.v = torch.randn(sk, generator=g, device=dev, dtype=torch.bfloat16)
        self.do = torch.randn(sq, generator=g, device=dev, dtype=torch.bfloat16)
        self.o = torch.empty_like(self.q)
        self.lse = torch.empty(mbs * Hq * N, dtype=torch.float32, device=dev)
        self.dq, self.dk, self.dv = torch.empty_like(self.q), torch.empty_like(self.k), torch.empty_like(self.v)
        # logprob rows of each piece: sequence s, kv heads [kv0, kv1) -> rows
        # [R kv0 / Hkv, R kv1 / Hkv) of s (shard.row_range)
        self.piece_rows = []
        tok_traj = []
        for p in self.pieces:
            n = 0
            for s in range(p.seq0, p.seq1):
                a, b = shard.row_range(p.kv0, p.kv1, Hkv, seq_resp_len(cfg, s))
                n += b - a
                tok_traj.append(torch.full((b - a,), s, dtype=torch.int32))
            self.piece_rows.append(n)
        self.n_rows = sum(self.piece_rows)
        self.max_rows = max(self.piece_rows + [1])
        self.V = VOCAB_QWEN3
        self.logits = torch.empty((self.max_rows, self.V), dtype=torch.bfloat16, device=dev)
        for r0 in range(0, self.max_rows, 4096):
            r1 = min(self.max_rows, r0 + 4096)
            self.logits[r0:r1] = torch.randn((r1 - r0, self.V), generator=g, device=dev) * 3.0
        self.dlogits = torch.empty_like(self.logits)
        self.targets = torch.randint(0, self.V, (self.max_rows,), generator=g, device=dev, dtype=torch.int32)
        # DiPO over the job's trajectories (one per sequence): rewards of every
        # trajectory (Bernoulli(0.5), one seed for the whole job), group ids;
        # the group statistics take only the trajectories this rank owns
        gr = torch.Generator().manual_seed(cfg.seed * 7919 + 1)
        self.rewards = torch.bernoulli(torch.full((self.n_seq,), 0.5), generator=gr).float().to(dev)
        self.group_of_traj = (torch.arange(self.n_seq, dtype=torch.int32) // job.group_size()).to(dev)
        self.traj_len = torch.tensor([seq_resp_len(cfg, s) for s in range(self.n_seq)], dtype=torch.int32,
                                     device=dev)
        own = torch.tensor(shard.owners(self.n_seq, Hkv, world)[rank], dtype=torch.long)
        self.own_rewards = self.rewards[own.to(dev)].contiguous()
        self.own_gid = self.group_of_traj[own.to(dev)].contiguous()
        self.own_len = self.traj_len[own.to(dev)].contiguous()
        self.traj_of_token = (torch.cat(tok_traj) if tok_traj else torch.zeros(0, dtype=torch.int32)).to(dev)
        self.n_groups = -(-self.n_seq // job.group_size())
        self.loss = None
        torch.cuda.synchronize()

    def piece_problem(self, p):
        cfg = self.cfg
        lens = None
        if cfg.resp_lens:
            lens = tuple(seq_resp_len(cfg, s) for s in range(p.seq0, p.seq1))
        prob = self.bd.Problem(p.n_seq, cfg.prompt_len, cfg.response_len, cfg.block_size, cfg.n_q_heads,
                               cfg.n_kv_heads, cfg.head_dim, cfg.repeat_prompt, n_copies=cfg.n_copies,
                               seq_prompt_lens=None if lens is None else (cfg.prompt_len,) * p.n_seq,
                               seq_response_lens=lens)
        if p.n_kv != cfg.n_kv_heads:
            prob = prob.head_shard(p.kv0, p.n_kv)
        return prob

    def dipo(self):
        from paper_2512_22234_b200 import dipo
        ops = self.ops
        stats = ops.dipo_group_stats(self.own_rewards, self.own_gid, self.own_len, self.n_groups)
        dipo.reduce_stats(stats, self.straddle)
        dlogp, parts = ops.dipo_token_loss(None, None, self.traj_of_token, self.rewards, self.group_of_traj, stats,
                                           self.n_groups)
        dipo.reduce_partials(parts)
        return dlogp, parts

    def run_piece(self, i, dlogp, r0, ev=None, bufs=None):
        """Attention fwd -> fused logprob -> attention bwd of piece i (its logprob
        rows start at r0 in this rank's token order)."""
        bd, ops = self.bd, self.ops
        b = bufs or self.__dict__
        p = self.pieces[i]
        prob = self.piece_problem(p)
        n = p.n_seq
        q, k, v, do = b["q"][:n], b["k"][:n], b["v"][:n], b["do"][:n]
        o, dq, dk, dv = self.o[:n], b["dq"][:n], b["dk"][:n], b["dv"][:n]
        if p.n_kv != self.cfg.n_kv_heads:
            q, do, o, dq = (prob.head_slice_q(t) for t in (q, do, o, dq))
            k, v, dk, dv = (prob.head_slice_kv(t) for t in (k, v, dk, dv))
        lse = self.lse[:n * prob.n_q_heads * prob.ntot].view(n, prob.n_q_heads, prob.ntot)
        rec = (lambda j: ev[j].record()) if ev is not None else (lambda j: None)
        rec(0)
        bd.attn_fwd(prob, q, k, v, o, lse)
        rec(1)
        nr = self.piece_rows[i]
        logp = None
        if nr:
            logp, _, _ = ops.logprob(self.logits[:nr], b["targets"][:nr], dlogp=dlogp[r0:r0 + nr],
                                     dlogits=self.dlogits[:nr])
        rec(2)
        bd.attn_bwd(prob, q, k, v, o, lse, do, dq, dk, dv)
        rec(3)
        return logp

    def run(self, evs=None, dipo_ev=None):
        """One step.  evs: optional per-piece lists of 4 CUDA events."""
        if dipo_ev is not None:
            dipo_ev[0].record()
        dlogp, parts = self.dipo()
        if dipo_ev is not None:
            dipo_ev[1].record()
        r0 = 0
        for i in range(len(self.pieces)):
            self.run_piece(i, dlogp, r0, None if evs is None else evs[i])
            r0 += self.piece_rows[i]
        self.loss = parts
        return parts


# ------------------------------------------------------------- timed runs
def run_ours(args):
    world, rank, local = dist_setup(args.gpus, args.dist_backend)
    job = JOBS[args.config]
    cfg = job.attn_cfg()
    peaks, peak_src = load_peaks()
    step = Step(job, rank, world)
    ops = step.ops
    fwd_f, bwd_f = rank_flops(job, world, rank)
    job_fwd, job_bwd = job_flops(job, world)
    for _ in range(args.warmup):
        step.run()
    barrier(world)

    # ---- device-resident timed region
    npc = len(step.pieces)
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(npc)] for _ in range(args.steps)]
    devs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = ops.launch_count()
    with ClockSampler(local) as clk:
        barrier(world)
        start.record()
        for i in range(args.steps):
            step.run(evs[i], devs[i])
        end.record()
        barrier(world)
    launches = (ops.launch_count() - n0) // args.steps
    ms_local = start.elapsed_time(end) / args.steps
    ms = max_over_ranks(ms_local, world)
    phase = {"dipo": statistics.mean(e[0].elapsed_time(e[1]) for e in devs)}
    for j, n in enumerate(["attn_fwd", "logprob_fused", "attn_bwd"]):
        phase[n] = statistics.mean(sum(pe[j].elapsed_time(pe[j + 1]) for pe in se) for se in evs)
    bwd_launch_ms = statistics.mean(pe[2].elapsed_time(pe[3]) for se in evs for pe in se)
    loss_val = float(step.loss[0].item())
    clocks = clk.summary()

    e2e = None if args.no_e2e else run_e2e(step, args, world, job_fwd + job_bwd)

    if rank != 0:
        del step
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    n_pieces = npc
    rows_r0 = step.n_rows
    del step
    torch.cuda.empty_cache()

    cfg_runs = None
    if world == 1 and not args.no_configs:
        cfg_runs = bench_configs(peaks, args.config_names.split(",") if args.config_names else None)
    nxt = None
    if world == 1 and not args.no_next:
        dec = bench_decode(peaks, peak_src)  # right after the step, before the long LM-head GEMMs
        nxt = {"lmhead_logprob": bench_lmhead(peaks, peak_src), "decode_attn": dec}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, target_s=args.cpu_seconds)

    value = (job_fwd + job_bwd) / (ms * 1e-3) / 1e12
    attn_ms = phase["attn_fwd"] + phase["attn_bwd"]
    peak_b, peak_s = peaks["bf16_tflops"], peaks["bf16_tflops_sustained"]
    bwd_per_launch = bwd_f / max(n_pieces, 1)
    bwd_achieved = bwd_f / (phase["attn_bwd"] * 1e-3) / 1e12  # = per-launch FLOPs / mean launch time
    fwd_achieved = fwd_f / (phase["attn_fwd"] * 1e-3) / 1e12
    lp_bytes = rows_r0 * VOCAB_QWEN3 * 2  # rank 0's logits (its logprob phase time is rank 0's)
    traffic = load_traffic() if cfg.name == "sdar_8b" and job.mb() == 16 else {}
    roofline = {"kernel": "bd_attn_bwd (attn_bwd_dkdv_kernel + attn_bwd_dqp_kernel (persistent dQ) + bwd_pre + tile map)",
                "bound": "tensor",
                "achieved": round(bwd_achieved, 1), "peak": peak_s, "unit": "TFLOP/s",
                "frac": round(bwd_achieved / peak_s, 4), "traffic": traffic.get("attn_bwd"),
                "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/ncu_traffic.json)",
                "peak_kind": f"bf16 sustained ({peak_src}); kernel timed inside a long step",
                "algorithmic": f"useful bwd FLOPs per launch = 10 d Hq b L(L+B) = {bwd_per_launch:.4e}",
                "launch_ms": round(bwd_launch_ms, 3)}
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
                          "algorithmic": "read of the bf16 logits + write of the bf16 dlogits (2 x 2 B per element)",
                          "traffic": (traffic["logprob_fused_ratio"] * 2 * lp_bytes)
                          if "logprob_fused_ratio" in traffic else None},
    }
    tokens = sum(cfg.prompt_len + seq_resp_len(cfg, s) for s in range(job.n_seq(world)))
    resp = sum(seq_resp_len(cfg, s) for s in range(job.n_seq(world)))
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": job.scaling,
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) q/k/v/dO, N(0,3^2) logits (read-only: dlogits to a separate buffer), "
                "Bernoulli(0.5) rewards; micro-batches reuse one resident buffer set)",
        "config": config_dict(job, world),
        "pct_bf16_peak": round(value / world / peak_s * 100, 2),
        "pct_bf16_peak_burst": round(value / world / peak_b * 100, 2),
        "peak_source": peak_src,
        "tokens_per_s": round(tokens / (ms * 1e-3), 1),
        "response_tokens_per_s": round(resp / (ms * 1e-3), 1),
        "logprob_rows_per_s": round(resp / (phase["logprob_fused"] * 1e-3), 1) if world == 1 else None,
        "phase_ms": {k: round(v, 3) for k, v in phase.items()},
        "dipo_loss": loss_val,
        "roofline": roofline,
        "roofline_other": others,
        "clocks": clocks,
        "gpu_launches": int(launches) * world,
        "gpu_launches_per_rank": int(launches),
        "e2e": e2e,
        "configs": cfg_runs,
        "cpu_baseline": cpu,
        "next_rows": nxt,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def config_dict(job, world):
    cfg = job.attn_cfg()
    return {"workload": job.name, "attn_shape": cfg.name, "n_sequences": job.n_seq(world),
            "grpo_group": job.group_size(), "micro_batch": job.mb(), "batch_per_gpu": job.n_seq(world) / world,
            "global_batch": job.n_seq(world), "n_q_heads": cfg.n_q_heads, "n_kv_heads": cfg.n_kv_heads,
            "head_dim": cfg.head_dim, "prompt_len": cfg.prompt_len, "response_len": cfg.response_len,
            "block_size": cfg.block_size, "packed_len": cfg.ntot, "n_copies": cfg.n_copies, "vocab": VOCAB_QWEN3,
            "parallelism": f"dp{world} over (sequence, kv-head group) units ({job.scaling} scaling)",
            "note": job.note, "l2": "inputs larger than L2 (q of one micro-batch >> 126 MB)"}


def run_e2e(step, args, world, flops_step):
    """End to end through the public API with pinned host buffers: every
    micro-batch's inputs (q, k, v, dO, targets) are copied H2D and its results
    (dQ, dK, dV, logp) D2H inside the timed region, plus the rewards H2D and
    the loss partials D2H once per step.  Two device buffer slots: the copy-in
    of micro-batch i+1 (H2D stream) and the copy-out of micro-batch i-1 (D2H
    stream) overlap the compute of micro-batch i."""
    names_in = ("q", "k", "v", "do", "targets")
    names_out = ("dq", "dk", "dv")
    ok = True
    try:
        host_in = {n: torch.empty(getattr(step, n).shape, dtype=getattr(step, n).dtype, pin_memory=True)
                   for n in names_in}
        host_out = {n: torch.empty(getattr(step, n).shape, dtype=getattr(step, n).dtype, pin_memory=True)
                    for n in names_out}
        host_logp = torch.empty(step.max_rows, dtype=torch.float32, pin_memory=True)
        host_rew = torch.empty(step.rewards.shape, dtype=torch.float32, pin_memory=True)
        host_loss = torch.empty(3, dtype=torch.float64, pin_memory=True)
        slots = [{n: getattr(step, n) for n in names_in + names_out},
                 {n: torch.empty_like(getattr(step, n)) for n in names_in + names_out}]
    except Exception as ex:  # noqa: BLE001 -- reported, the device-resident line still prints
        print(f"[bench] e2e skipped: allocation failed: {ex}", file=sys.stderr)
        ok = False
    if world > 1:
        flag = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok = bool(flag.item())
    if not ok:
        return None
    for n in names_in:
        host_in[n].copy_(getattr(step, n))
    host_rew.copy_(step.rewards)
    main = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    computed = [torch.cuda.Event(), torch.cuda.Event()]
    drained = [torch.cuda.Event(), torch.cuda.Event()]
    npc = len(step.pieces)
    tally = {"h2d": 0, "d2h": 0}

    def copy_in(i, sl):
        n = step.pieces[i].n_seq
        s_in.wait_event(computed[sl])  # the slot's previous micro-batch no longer reads its inputs
        with torch.cuda.stream(s_in):
            for nm in names_in:
                src = host_in[nm][:step.piece_rows[i]] if nm == "targets" else host_in[nm][:n]
                dst = slots[sl][nm][:step.piece_rows[i]] if nm == "targets" else slots[sl][nm][:n]
                dst.copy_(src, non_blocking=True)
                tally["h2d"] += src.numel() * src.element_size()
            copied[sl].record(s_in)

    def run(n_steps):
        """n_steps steps as one stream of micro-batches: the copy-in of the
        next micro-batch (of this step or the next) overlaps the compute of the
        current one, whose copy-out overlaps the one after."""
        for e in computed + drained:
            e.record(main)
        order = [(s, i) for s in range(n_steps) for i in range(npc)]
        copy_in(0, 0)
        dlogp = parts = None
        r0 = 0
        for idx, (s, i) in enumerate(order):
            sl = idx % 2
            if i == 0:
                step.rewards.copy_(host_rew, non_blocking=True)
                tally["h2d"] += host_rew.numel() * 4
                dlogp, parts = step.dipo()
                r0 = 0
            if idx + 1 < len(order):
                copy_in(order[idx + 1][1], 1 - sl)
            main.wait_event(copied[sl])
            main.wait_event(drained[sl])  # the slot's previous outputs are copied out
            logp = step.run_piece(i, dlogp, r0, bufs=slots[sl])
            computed[sl].record(main)
            s_out.wait_event(computed[sl])
            n = step.pieces[i].n_seq
            with torch.cuda.stream(s_out):
                for nm in names_out:
                    host_out[nm][:n].copy_(slots[sl][nm][:n], non_blocking=True)
                    tally["d2h"] += host_out[nm][:n].numel() * 2
                if logp is not None:
                    host_logp[:logp.numel()].copy_(logp, non_blocking=True)
                    tally["d2h"] += logp.numel() * 4
                if i == npc - 1:
                    host_loss.copy_(parts, non_blocking=True)
                    tally["d2h"] += 24
                drained[sl].record(s_out)
            r0 += step.piece_rows[i]
        main.wait_stream(s_out)

    run(1)  # warm path
    barrier(world)
    # >= ~24 micro-batches: the first copy-in (pipeline fill) is amortised over the run
    n_steps = max(2, min(args.steps, -(-24 // npc)))
    tally["h2d"] = tally["d2h"] = 0
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record()
    run(n_steps)
    ee.record()
    barrier(world)
    h2d, d2h = tally["h2d"] // n_steps, tally["d2h"] // n_steps
    e2e_ms = max_over_ranks(es.elapsed_time(ee) / n_steps, world)
    return {"value": round(flops_step / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
            "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": n_steps,
            "inputs": "q, k, v, dO, targets of every micro-batch and the rewards H2D from pinned host; dQ, dK, dV "
                      "and logp of every micro-batch and the DiPO loss partials D2H (H2D / D2H streams, two "
                      "device slots; micro-batches of consecutive steps form one pipeline, copies overlapped with "
                      "compute); the logits are the caller's LM-head output and stay device-resident"}


def _timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    st = torch.cuda.current_stream()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


CONFIG_RUNS = ["sdar_1_7b", "sweep_b4", "sweep_b8", "sweep_b16", "sweep_b32", "trace_s4", "sdar_8b_varlen", "tiny"]


def bench_configs(peaks, names=None):
    """Every other BASELINE config, measured in this process after the step
    (attention fwd and bwd through the ABI, CUDA events on the launching
    stream, median of 5 after 2 warm-ups; inputs >> L2), each with its own
    nvidia-smi clock summary and its tile-map sparsity."""
    import paper_2512_22234_b200 as bd
    from paper_2512_22234_b200 import ops
    from workloads import attn_inputs, useful_flops, total_pairs, total_tokens
    out = {}
    for name in names or CONFIG_RUNS:
        cfg = CONFIGS[name]
        prob = bd.Problem.from_cfg(cfg)
        q, k, v, do = attn_inputs(cfg, device="cuda")
        o, lse = bd.attn_fwd(prob, q, k, v)
        dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
        # enough repetitions for >= ~1.5 s of timed work, so nvidia-smi (200 ms)
        # samples the clocks of every config
        t0 = _timeit(lambda: (bd.attn_fwd(prob, q, k, v, o, lse), bd.attn_bwd(prob, q, k, v, o, lse, do, dq, dk, dv)),
                     reps=1)
        reps = int(min(200, max(5, 750.0 / max(t0, 1e-3))))
        with ClockSampler(torch.cuda.current_device()) as clk:
            tf = _timeit(lambda: bd.attn_fwd(prob, q, k, v, o, lse), reps)
            tb = _timeit(lambda: bd.attn_bwd(prob, q, k, v, o, lse, do, dq, dk, dv), reps)
        f, fb = useful_flops(cfg)
        if cfg.resp_lens is None:
            st = ops.tilemap_stats(prob)
            tiles_all, nonempty, partial = st["tiles"] ** 2, st["nonempty"], st["partial"]
        else:
            sts = [ops.tilemap_stats(bd.Problem.from_cfg(cfg.with_(batch=1, response_len=r, resp_lens=None)))
                   for r in cfg.resp_lens]
            tiles_all = sum(x["tiles"] ** 2 for x in sts)
            nonempty = sum(x["nonempty"] for x in sts)
            partial = sum(x["partial"] for x in sts)
        pairs = total_pairs(cfg) / (cfg.batch if cfg.resp_lens is None else 1)
        peak = peaks["bf16_tflops_sustained"]
        out[name] = {"batch": cfg.batch, "heads": f"{cfg.n_q_heads}/{cfg.n_kv_heads}", "head_dim": cfg.head_dim,
                     "prompt_len": cfg.prompt_len, "response_len": cfg.response_len, "block_size": cfg.block_size,
                     "n_copies": cfg.n_copies, "varlen": cfg.resp_lens is not None,
                     "fwd_ms": round(tf, 3), "bwd_ms": round(tb, 3), "reps": reps,
                     "fwd_tflops": round(f / tf / 1e9, 1), "bwd_tflops": round(fb / tb / 1e9, 1),
                     "fwd_bwd_tflops": round((f + fb) / (tf + tb) / 1e9, 1),
                     "fwd_bwd_frac_sustained": round((f + fb) / (tf + tb) / 1e9 / peak, 4),
                     "tokens_per_s": round(total_tokens(cfg) / ((tf + tb) * 1e-3), 1),
                     "tile_skip_frac": round(1 - nonempty / tiles_all, 4),
                     "partial_frac_of_listed": round(partial / nonempty, 4),
                     "useful_over_computed": round(pairs / (nonempty * 128 * 128), 4)
                     if cfg.resp_lens is None else None,
                     "clocks": clk.summary()}
        del q, k, v, do, o, lse, dq, dk, dv
        torch.cuda.empty_cache()
    return out


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
    _, lse = ops.lmhead_logprob(h, W, t)
    with ClockSampler(torch.cuda.current_device()) as clk:
        fwd_ms = _timeit(lambda: ops.lmhead_logprob(h, W, t), reps)
        bwd_ms = _timeit(lambda: ops.lmhead_logprob_bwd(h, W, t, lse, w, chunk_rows=16384, dh=dh, dw=dw), reps)
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
            "logits_bytes_not_materialised": n * V * 2, "clocks": clk.summary()}


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
    with ClockSampler(torch.cuda.current_device()) as clk:
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
            "algorithmic_bytes": byts, "l2": "flushed before each call", "clocks": clk.summary()}


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


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
    """The fp64 oracle timed on the host cores on a bounded row sample, plus
    labelled extrapolations to one (sequence, kv-group) slice and to the whole
    config (useful FLOPs / the sample's measured useful FLOP/s)."""
    from workloads import useful_flops
    n = 256
    dt, fl, desc = oracle_sample(cfg, n)
    n2 = int(min(cfg.ntot, max(n, n * target_s / max(dt, 1e-3))))
    if n2 > n:
        dt, fl, desc = oracle_sample(cfg, n2)
    rate = fl / dt
    G = cfg.n_q_heads // cfg.n_kv_heads
    slice_f = 14 * cfg.head_dim * G * (useful_pairs(cfg) if cfg.resp_lens is None else 0)
    f, fb = useful_flops(cfg)
    return {"value": round(rate / 1e12, 6), "unit": "TFLOP/s", "cores": _oracle_threads(), "kind": "oracle",
            "sample": desc, "seconds": round(dt, 2), "host_cpu_count": os.cpu_count(), "cpu_model": cpu_model(),
            "extrapolated_slice_s": round(slice_f / rate, 1) if slice_f else None,
            "extrapolated_config_s": round((f + fb) / rate, 1),
            "extrapolation": "useful FLOPs of one (sequence, kv-group) slice / of the whole config divided by the "
                             "sample's measured useful FLOP/s (labelled estimate, not timed)"}


def run_reference(args):
    """--impl reference: the fp64 CPU oracle timed on the host cores on this
    arm's workload / metric (each step a bounded row sample)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    job = JOBS[args.config]
    cfg = job.attn_cfg()
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
        "metric": METRIC,
        "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot_t / args.steps, 1), "higher_is_better": True, "scaling": job.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(job, world),
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": _oracle_threads(), "kind": "oracle",
                         "sample": desc + " per step", "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="sdar_8b", choices=sorted(JOBS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the SURVEY 8(f) next-row measurements")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs")
    ap.add_argument("--config-names", default="", help="comma-separated subset of the other configs")
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
