"""Dense block-diffusion visibility mask, written from the paper's rule.

Sources:
* Block partition, blk(p) = p // B (Eq. 1 "partition it into K
  non-overlapping text blocks ... each block contains B tokens").
* Reverse process, Eq. 2: block k is predicted from its noisy
  state b^k_t and the clean history b^{<k}  ->  a noisy (xt) token sees the
  clean (x0) blocks < k and its own noisy block (bidirectionally).
* Clean tokens attend block-causally (own whole block + earlier blocks):
  S:213 "CLEAN block k sees CLEAN blocks <= k", SPEC design decision
  "CLEAN-copy intra-block attention is bidirectional" (reading c3).
* A clean token never sees a noisy token ("NOISY ... sees CLEAN blocks
  < k and NOISY block k (itself, bidirectional) and nothing else"; clean rows
  see only clean blocks).
* DiRL repeats prompt and response blockwise (Fig. 4b);
  TraceRL repeats only the output (Fig. 4a) -> ``repeat_prompt``.

* Trace replay (reading c19, Eq. 6): with S noisy
  copies, copy s of block k is one conditioning state; it "sees CLEAN earlier
  blocks and itself" -- never another copy.

Rule table (query segment, key segment -> visible iff):
    x0    -> x0    : blk(pk) <= blk(pq)
    xt(s) -> x0    : blk(pk) <  blk(pq)
    xt(s) -> xt(u) : s == u and blk(pk) == blk(pq)
    x0    -> xt    : never

ORACLE: test infrastructure only (see oracle/__init__.py).
"""

import numpy as np

from .problem import Problem


def packed_copies(prob: Problem):
    """Return (copy[Ntot] int64, clean_pos[Ntot] int64) for the packed axis.

    Packed index n < L is x0 (copy 0) at clean position n; the noisy copies
    follow, copy s (1..S) occupying [L + (s-1)(L-xb), L + s(L-xb)) at clean
    positions xb.. L-1 (reading c1: concatenated [x0 | xt^(1) | ...]; noisy
    copies keep their source positions, S:139 / S:169)."""
    L, xb, N, Ln = prob.L, prob.xb, prob.ntot, prob.n_noisy
    n = np.arange(N, dtype=np.int64)
    noisy = n >= L
    j = np.where(noisy, n - L, 0)
    copy = np.where(noisy, 1 + j // max(Ln, 1), 0)
    pos = np.where(noisy, xb + j % max(Ln, 1), n)
    return copy, pos


def packed_segments(prob: Problem):
    """Return (is_noisy[Ntot] bool, clean_pos[Ntot] int64)."""
    copy, pos = packed_copies(prob)
    return copy > 0, pos


def mask_rows(prob: Problem, rows) -> np.ndarray:
    """Visibility M[rows, :] (bool) straight from the rule table."""
    copy, pos = packed_copies(prob)
    noisy = copy > 0
    rows = np.asarray(rows, dtype=np.int64)
    B = prob.block_size
    bq = (pos[rows] // B)[:, None]
    bk = (pos // B)[None, :]
    q_noisy = noisy[rows][:, None]
    k_noisy = noisy[None, :]
    same_copy = copy[rows][:, None] == copy[None, :]
    clean_clean = (~q_noisy) & (~k_noisy) & (bk <= bq)
    noisy_clean = q_noisy & (~k_noisy) & (bk < bq)
    noisy_noisy = q_noisy & k_noisy & same_copy & (bk == bq)
    return clean_clean | noisy_clean | noisy_noisy


def mask_dense(prob: Problem) -> np.ndarray:
    """Full [Ntot, Ntot] boolean mask."""
    prob.validate()
    return mask_rows(prob, np.arange(prob.ntot))


def assert_rows_nonempty(m: np.ndarray) -> None:
    """a query row with zero visible keys is a contract violation."""
    empty = np.where(~m.any(axis=1))[0]
    if empty.size:
        raise AssertionError(f"rows with zero visible keys: {empty[:8].tolist()}")


def visible_pairs(prob: Problem) -> int:
    """Number of visible (query, key) pairs per (sequence, head)."""
    total = 0
    for r0 in range(0, prob.ntot, 1024):
        total += int(mask_rows(prob, np.arange(r0, min(prob.ntot, r0 + 1024))).sum())
    return total
