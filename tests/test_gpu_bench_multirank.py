"""The bench's multi-rank path (torchrun, one process per GPU, DiPO scalars
all-reduced, max-over-ranks timing) run end to end as a 2-rank dry run on a
single GPU: gloo backend, both ranks on cuda:0 (BD_BENCH_SHARE_GPU=1).  Checks
the contract keys of the single JSON line rank 0 prints; the throughput of a
shared-GPU run means nothing and is not checked."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_dry_run(cuda_ok):
    env = dict(os.environ, BD_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--config", "tiny", "--dist-backend", "gloo", "--no-next",
           "--no-cpu-baseline", "--no-configs"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 2 * d["config"]["batch_per_gpu"]
    assert d["gpu_launches"] == 2 * d["gpu_launches_per_rank"] > 0
    for key in ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "roofline", "clocks", "e2e"):
        assert key in d, key


def test_eight_rank_fig6_head_sharding_dry_run(cuda_ok):
    """The paper's Fig. 6 job (batch 4, SDAR-8B) on 8 ranks: each rank runs 4 of
    one sequence's 8 kv heads (head-sharded problems on strided head slices) and
    the group statistics are all-reduced (the group straddles ranks)."""
    env = dict(os.environ, BD_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "8",
           "--master-addr", "127.0.0.1", "--master-port", "29519", os.path.join(ROOT, "bench.py"), "--gpus", "8",
           "--steps", "2", "--warmup", "3", "--config", "fig6", "--dist-backend", "gloo", "--no-next",
           "--no-cpu-baseline", "--no-e2e", "--no-configs"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 8 and d["scaling"] == "strong" and d["config"]["n_sequences"] == 4
    assert d["gpu_launches_per_rank"] > 0 and d["dipo_loss"] == d["dipo_loss"]  # not NaN
