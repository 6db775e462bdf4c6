"""Work partitioning across ranks: host logic only.

The hot path shards with no attention-time exchange.  Units are
(sequence, kv-head group) pairs numbered sequence-major, u = s Hkv + g; rank r
takes the contiguous unit range [r U / W, (r + 1) U / W) of the U = n Hkv
units (north star: "sequences and heads are partitioned across the 8 GPUs").
When W divides n every rank gets whole sequences (the usual data-parallel
case); when n < W (e.g. the paper's Fig. 6 run, batch 4 on 8 GPUs) a
sequence's kv heads are split between ranks, which run their heads in place
on head slices of the full-width tensors (bd_problem q_row_heads /
kv_row_heads, Problem.head_shard).

A sequence's response rows (its log-prob tokens) are split between the ranks
that hold its kv heads, in proportion to the heads: the rank with kv heads
[g0, g1) scores rows [R g0 / Hkv, R g1 / Hkv).  The rank holding kv head 0 of
a sequence "owns" the trajectory for the DiPO group statistics (each
trajectory counted once).  A GRPO group whose sequences span more than one
rank straddles: its statistics are all-reduced before the token weights
(paper_2512_22234_b200.dipo.reduce_stats).
"""

from dataclasses import dataclass


def shard_range(n_units: int, world: int, rank: int):
    """Contiguous sharding: rank r gets [r n / W, (r + 1) n / W)."""
    return (rank * n_units) // world, ((rank + 1) * n_units) // world


@dataclass(frozen=True)
class Piece:
    """Sequences [seq0, seq1) with kv heads [kv0, kv1) of each."""
    seq0: int
    seq1: int
    kv0: int
    kv1: int

    @property
    def n_seq(self):
        return self.seq1 - self.seq0

    @property
    def n_kv(self):
        return self.kv1 - self.kv0


def plan(n_seq: int, n_kv: int, world: int, rank: int, micro_batch: int = 0):
    """Pieces of rank `rank`, in order; whole-sequence runs are cut into
    micro-batches of at most `micro_batch` sequences (0 = no limit)."""
    u0, u1 = shard_range(n_seq * n_kv, world, rank)
    out = []
    u = u0
    while u < u1:
        s, g = divmod(u, n_kv)
        if g == 0 and u + n_kv <= u1:
            s_end = u1 // n_kv
            step = micro_batch if micro_batch > 0 else s_end - s
            for a in range(s, s_end, step):
                out.append(Piece(a, min(s_end, a + step), 0, n_kv))
            u = s_end * n_kv
        else:
            g_end = min(n_kv, g + (u1 - u))
            out.append(Piece(s, s + 1, g, g_end))
            u += g_end - g
    return out


def row_range(piece_kv0: int, piece_kv1: int, n_kv: int, n_rows: int):
    """Response rows of a sequence scored by the rank holding kv heads [kv0, kv1)."""
    return (n_rows * piece_kv0) // n_kv, (n_rows * piece_kv1) // n_kv


def owners(n_seq: int, n_kv: int, world: int):
    """rank -> list of sequences whose kv head 0 it holds (trajectory owner)."""
    res = {r: [] for r in range(world)}
    for r in range(world):
        for p in plan(n_seq, n_kv, world, r):
            if p.kv0 == 0:
                res[r].extend(range(p.seq0, p.seq1))
    return res


def ranks_of_sequence(n_seq: int, n_kv: int, world: int):
    """sequence -> sorted list of ranks holding any of its kv heads."""
    res = {s: set() for s in range(n_seq)}
    for r in range(world):
        for p in plan(n_seq, n_kv, world, r):
            for s in range(p.seq0, p.seq1):
                res[s].add(r)
    return {s: sorted(v) for s, v in res.items()}


def groups_straddle(n_seq: int, group_size: int, world: int, n_kv: int = 1) -> bool:
    """True if some GRPO group (group_size consecutive sequences) spans ranks."""
    where = ranks_of_sequence(n_seq, n_kv, world)
    for g0 in range(0, n_seq, group_size):
        ranks = set()
        for s in range(g0, min(n_seq, g0 + group_size)):
            ranks.update(where[s])
        if len(ranks) > 1:
            return True
    return False
