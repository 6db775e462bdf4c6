"""Host logic of the multi-GPU partitioning (paper_2512_22234_b200/shard.py):
(sequence, kv-head group) units cover the job exactly once, whole sequences
stay on one rank when the world size divides the batch, heads are split when
it does not (the paper's Fig. 6 run: batch 4 on 8 GPUs), logprob rows
and trajectory ownership partition the job, and straddling GRPO groups are
detected.  A world-size-2 gloo run checks the two all-reduces of the DiPO step
reproduce the 1-rank oracle loss with the plan's row / owner split."""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_22234_b200 import shard, dipo as bdipo
from oracle import dipo as odipo


@pytest.mark.parametrize("n_seq,n_kv,world,mb", [
    (16, 8, 1, 16), (16, 8, 2, 16), (16, 8, 8, 16), (4, 8, 8, 4), (4, 8, 3, 4), (1024, 8, 8, 16),
    (1024, 8, 1, 16), (3, 8, 5, 0), (16, 8, 32, 16), (7, 2, 4, 2),
])
def test_units_cover_job_once(n_seq, n_kv, world, mb):
    seen = np.zeros((n_seq, n_kv), dtype=int)
    for r in range(world):
        for p in shard.plan(n_seq, n_kv, world, r, mb):
            assert 0 <= p.seq0 < p.seq1 <= n_seq and 0 <= p.kv0 < p.kv1 <= n_kv
            if mb and p.kv0 == 0 and p.kv1 == n_kv:
                assert p.n_seq <= mb
            if p.n_seq > 1:
                assert (p.kv0, p.kv1) == (0, n_kv)  # multi-sequence pieces carry every head
            seen[p.seq0:p.seq1, p.kv0:p.kv1] += 1
    assert (seen == 1).all()


def test_whole_sequences_when_world_divides_batch():
    for r in range(8):
        ps = shard.plan(1024, 8, 8, r, 16)
        assert all(p.kv0 == 0 and p.kv1 == 8 for p in ps)
        assert sum(p.n_seq for p in ps) == 128 and len(ps) == 8
    assert not shard.groups_straddle(1024, 8, 8, 8)  # 128 prompts x G = 8 (BJ configs[4])


def test_fig6_head_split():
    """Batch 4 on 8 ranks: each rank holds 4 of the 8 kv heads of one sequence."""
    for r in range(8):
        (p,) = shard.plan(4, 8, 8, r)
        assert p.n_seq == 1 and p.n_kv == 4 and p.seq0 == r // 2 and p.kv0 == 4 * (r % 2)
    assert shard.groups_straddle(4, 4, 8, 8)


def test_rows_and_owners_partition():
    for n_seq, n_kv, world in [(4, 8, 8), (4, 8, 3), (16, 8, 8), (3, 8, 5), (16, 8, 32)]:
        R = 8192
        rows = np.zeros((n_seq, R), dtype=int)
        for r in range(world):
            for p in shard.plan(n_seq, n_kv, world, r):
                a, b = shard.row_range(p.kv0, p.kv1, n_kv, R)
                rows[p.seq0:p.seq1, a:b] += 1
        assert (rows == 1).all()
        own = shard.owners(n_seq, n_kv, world)
        flat = sorted(s for v in own.values() for s in v)
        assert flat == list(range(n_seq))


def test_straddle_detection():
    assert not shard.groups_straddle(16, 16, 1, 8)
    assert shard.groups_straddle(16, 16, 8, 8)      # one group of 16 over 8 ranks
    assert not shard.groups_straddle(128, 16, 8, 8)  # weak: one group per rank
    assert bdipo.groups_straddle(16, 16, 8)


def _job(n_groups, G, R_max, seed=0):
    rng = np.random.default_rng(seed)
    n = n_groups * G
    rewards = rng.integers(0, 2, n).astype(np.float64)
    lens = rng.integers(R_max // 2, R_max + 1, n)
    gid = np.repeat(np.arange(n_groups), G)
    return rewards, lens, gid


def _rank_partials(rank, world, n_kv, rewards, lens, gid, n_groups, straddle):
    """The DiPO step of one rank from the plan: owned trajectories enter the
    group statistics once, each rank's rows carry rho == 1 token terms."""
    n_seq = len(rewards)
    own = shard.owners(n_seq, n_kv, world)[rank]
    stats = torch.zeros((n_groups, 3), dtype=torch.float64)
    for s in own:
        stats[gid[s]] += torch.tensor([rewards[s], 1.0, lens[s]], dtype=torch.float64)
    bdipo.reduce_stats(stats, straddle)
    parts = torch.zeros(3, dtype=torch.float64)
    for p in shard.plan(n_seq, n_kv, world, rank):
        for s in range(p.seq0, p.seq1):
            a, b = shard.row_range(p.kv0, p.kv1, n_kv, int(lens[s]))
            g = gid[s]
            A = rewards[s] - stats[g, 0] / stats[g, 1]
            parts[0] -= (b - a) * A / (stats[g, 2] * n_groups)
            parts[1] += b - a
    bdipo.reduce_partials(parts)
    return parts


def _worker(rank, world, path, out, n_groups, G, n_kv):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    rewards, lens, gid = _job(n_groups, G, 40)
    straddle = shard.groups_straddle(len(rewards), G, world, n_kv)
    parts = _rank_partials(rank, world, n_kv, rewards, lens, gid, n_groups, straddle)
    out[rank] = (float(parts[0]), float(parts[1]), straddle)
    dist.destroy_process_group()


@pytest.mark.parametrize("n_groups,G,n_kv", [(1, 4, 8), (2, 1, 8), (3, 3, 2)])
def test_gloo_two_ranks_plan_loss_equals_one_rank(n_groups, G, n_kv):
    """World size 2 over (sequence, kv-head) units -- heads split when there
    is a single sequence per group -- reproduces the 1-rank oracle loss."""
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mgr = mp.Manager()
        out = mgr.dict()
        mp.spawn(_worker, args=(world, os.path.join(d, "pg"), out, n_groups, G, n_kv), nprocs=world, join=True)
        rewards, lens, gid = _job(n_groups, G, 40)
        traj_of_token = np.repeat(np.arange(len(lens)), lens)
        lp = np.zeros(traj_of_token.size)
        ref, _, _ = odipo.dipo_loss(lp, lp, traj_of_token, rewards, gid)
        for r in range(world):
            assert abs(out[r][0] - ref) < 1e-12, (dict(out), ref)
            assert out[r][1] == lens.sum()
