"""DiPO step driver: sequence sharding across ranks and the scalar NCCL
all-reduce.  The arithmetic runs in the library's kernels
(bd_dipo_group_stats / bd_dipo_token_loss); this module only decides which
tiny tensors cross ranks:

* per-group (sum r, count, sum |tau|) -- only when a GRPO group straddles
  ranks (otherwise every group's statistics are rank-local);
* (loss partial, tokens, clipped tokens) -- always, one fp64[3] all-reduce.

Eq. 8 with the stop-gradient behaviour policy of Eq. 7
(P:179-204); A_i = r_i - mean of the group.
"""

import torch
import torch.distributed as dist

from . import ops, shard


def shard_range(n_units: int, world: int, rank: int):
    """Contiguous sharding of n_units sequences: rank r gets [r n/W, (r+1) n/W)."""
    return shard.shard_range(n_units, world, rank)


def groups_straddle(n_seq: int, group_size: int, world: int, n_kv: int = 1) -> bool:
    """True if some GRPO group is split across ranks (see shard.groups_straddle)."""
    return shard.groups_straddle(n_seq, group_size, world, n_kv)


def _dist_on(pg):
    return dist.is_available() and dist.is_initialized() and dist.get_world_size(pg) > 1


def reduce_stats(stats, straddle: bool, pg=None):
    if straddle and _dist_on(pg):
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=pg)
    return stats


def reduce_partials(partials, pg=None):
    if _dist_on(pg):
        dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=pg)
    return partials


def dipo_loss(logp, logp_old, traj_of_token, rewards, group_of_traj, traj_len, n_groups_global,
              straddle=False, eps=0.2, pg=None):
    """One DiPO reduction on this rank's tokens.

    group_of_traj holds GLOBAL group ids in [0, n_groups_global).  Returns
    (loss fp64 scalar tensor, dlogp, partials) with loss already summed over
    ranks."""
    stats = ops.dipo_group_stats(rewards, group_of_traj, traj_len, n_groups_global)
    reduce_stats(stats, straddle, pg)
    dlogp, partials = ops.dipo_token_loss(logp, logp_old, traj_of_token, rewards, group_of_traj, stats,
                                          n_groups_global, eps)
    reduce_partials(partials, pg)
    return partials[0], dlogp, partials
