"""CPU checks of bench.py's accounting and of its reference arm:
the useful-FLOP closed forms agree with the oracle's mask count, and
`bench.py --impl reference` prints one JSON line with the contract's keys."""

import json
import os
import subprocess
import sys

import pytest

from oracle import Problem as OP, mask
from workloads import CONFIGS, useful_flops, useful_pairs, total_pairs, total_tokens

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("P,R,B,S", [(8, 24, 4, 1), (0, 32, 8, 1), (12, 36, 4, 3), (16, 48, 16, 4)])
def test_pairs_closed_form_vs_oracle_mask(P, R, B, S):
    cfg = CONFIGS["tiny"].with_(prompt_len=P, response_len=R, block_size=B, n_copies=S)
    prob = OP(1, P, R, B, 1, 1, 64, 1, n_copies=S)
    assert useful_pairs(cfg) == mask.visible_pairs(prob)


def test_varlen_totals_sum_sequences():
    cfg = CONFIGS["tiny"].with_(batch=3, prompt_len=8, response_len=24, block_size=4, resp_lens=(24, 8, 16))
    want = sum(mask.visible_pairs(OP(1, 8, r, 4, 1, 1, 64, 1)) for r in (24, 8, 16))
    assert total_pairs(cfg) == want
    assert total_tokens(cfg) == (8 + 24) + (8 + 8) + (8 + 16)


def test_flop_accounting_bench_shape():
    cfg = CONFIGS["sdar_8b"]
    fwd, bwd = useful_flops(cfg)
    L = cfg.prompt_len + cfg.response_len
    pairs = L * (L + cfg.block_size)
    assert fwd == 4 * cfg.head_dim * cfg.n_q_heads * cfg.batch * pairs
    assert bwd == 2.5 * fwd
    assert abs((fwd + bwd) / 1e12 - 77.96) < 0.01  # 77.96 TFLOP per call


def test_reference_arm_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-rows", "16", "--config", "sdar_1_7b"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "gpu_launches"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOP/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"] == "sdar_1_7b"


def test_job_accounting_over_ranks():
    """Strong-scaling jobs keep the whole job's useful FLOPs fixed as W grows
    (units partition the job); BJ configs[4] totals 4,990 TFLOP fwd+bwd
    (SURVEY §8(d)); weak jobs grow linearly."""
    sys.path.insert(0, ROOT)
    import bench
    for name in ("rl8", "fig6", "sdar_8b_strong"):
        job = bench.JOBS[name]
        tot = [sum(bench.job_flops(job, w)) for w in (1, 2, 4, 8)]
        assert max(tot) - min(tot) < 1e-6 * tot[0], (name, tot)
    assert abs(sum(bench.job_flops(bench.JOBS["rl8"], 8)) / 1e12 - 4990) < 1
    w1 = sum(bench.job_flops(bench.JOBS["sdar_8b"], 1))
    assert abs(sum(bench.job_flops(bench.JOBS["sdar_8b"], 8)) - 8 * w1) < 1e-6 * w1
    # fig6 at W = 8: every rank runs half of one sequence's heads
    f = [bench.rank_flops(bench.JOBS["fig6"], 8, r)[0] for r in range(8)]
    assert max(f) == min(f)
