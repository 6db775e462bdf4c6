"""World-size-2 gloo test of the multi-rank DiPO path (CPU).

The kernels need a GPU, so each rank computes its local per-group statistics
and token partials with the oracle's formulas split by shard; the test checks
the host-side distributed logic of paper_2512_22234_b200.dipo -- contiguous
sharding, straddle detection, the two all-reduces -- reproduces the 1-rank
loss exactly (reduced loss == 1-GPU loss)."""

import os
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_22234_b200 import dipo as bdipo
from oracle import dipo as odipo


def _local_partials(rank, world, rewards, group_of_traj, lens, n_groups, straddle, logp):
    """Per-rank computation mirroring bd_dipo_group_stats / bd_dipo_token_loss."""
    n_traj = len(rewards)
    a, b = bdipo.shard_range(n_traj, world, rank)
    stats = torch.zeros((n_groups, 3), dtype=torch.float64)
    for i in range(a, b):
        stats[group_of_traj[i]] += torch.tensor([rewards[i], 1.0, lens[i]], dtype=torch.float64)
    bdipo.reduce_stats(stats, straddle)
    starts = np.concatenate([[0], np.cumsum(lens)])
    parts = torch.zeros(3, dtype=torch.float64)
    for i in range(a, b):
        gi = group_of_traj[i]
        A = rewards[i] - stats[gi, 0] / stats[gi, 1]
        Ng = stats[gi, 2]
        for k in range(starts[i], starts[i + 1]):
            parts[0] -= A / (Ng * n_groups)  # rho = 1 -> C = A
            parts[1] += 1
    bdipo.reduce_partials(parts)
    return parts


def _worker(rank, world, path, out, straddle_expected, group_size, n_groups):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    rewards = rng.integers(0, 2, n_groups * group_size).astype(float)
    group_of_traj = np.repeat(np.arange(n_groups), group_size)
    lens = rng.integers(1, 9, n_groups * group_size)
    straddle = bdipo.groups_straddle(len(rewards), group_size, world)
    assert straddle == straddle_expected
    parts = _local_partials(rank, world, rewards, group_of_traj, lens, n_groups, straddle, None)
    out[rank] = float(parts[0])
    dist.destroy_process_group()


def _run(group_size, n_groups, straddle_expected):
    world = 2
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "pg")
        mgr = mp.Manager()
        out = mgr.dict()
        mp.spawn(_worker, args=(world, path, out, straddle_expected, group_size, n_groups), nprocs=world, join=True)
        rng = np.random.default_rng(0)
        rewards = rng.integers(0, 2, n_groups * group_size).astype(float)
        group_of_traj = np.repeat(np.arange(n_groups), group_size)
        lens = rng.integers(1, 9, n_groups * group_size)
        traj_of_token = np.repeat(np.arange(len(lens)), lens)
        logp = np.zeros(traj_of_token.size)
        ref, _, _ = odipo.dipo_loss(logp, logp, traj_of_token, rewards, group_of_traj)
        assert abs(out[0] - ref) < 1e-12 and abs(out[1] - ref) < 1e-12, (dict(out), ref)


def test_gloo_two_ranks_groups_straddle():
    _run(group_size=3, n_groups=3, straddle_expected=True)   # 9 trajectories -> [0,4) [4,9)


def test_gloo_two_ranks_whole_groups():
    _run(group_size=4, n_groups=2, straddle_expected=False)  # 8 trajectories -> [0,4) [4,8)


def test_shard_helpers():
    assert bdipo.shard_range(10, 4, 0) == (0, 2) and bdipo.shard_range(10, 4, 3) == (7, 10)
    assert not bdipo.groups_straddle(16, 8, 2)
    assert bdipo.groups_straddle(16, 16, 8)
    assert not bdipo.groups_straddle(1024, 8, 8)
