"""Tile classification from the dense mask (the definition the GPU tile map
must equal bit-exactly).

The packed axis of each segment is cut into 128-row tiles starting at the
segment start: x0 tiles cover packed rows [128 j, min(128 j + 128, L)), the
tiles of noisy copy s cover [c_s + 128 j, min(c_s + 128 j + 128, c_s + L - xb))
with c_s = L + (s-1)(L - xb).  For every (q-tile,
k-tile) pair the kind is read off the dense mask restricted to the tile's
valid rows/columns:

    FULL    every pair visible
    EMPTY   no pair visible          (never listed, never loaded)
    PARTIAL otherwise

Kinds are returned as an ordered list of (q_seg, q_tile, k_seg, k_tile, kind)
tuples, q-tiles in packed order and k-tiles in packed order, EMPTY omitted.
This is SPEC's "optional block-skip optimization for fully-masked tiles"
 turned into a schedule; the only requirement the paper puts on it is
that results are unchanged ("accepts fine-grained masks").

ORACLE: test infrastructure only (see oracle/__init__.py).
"""

import numpy as np

from .problem import Problem
from .mask import mask_dense

FULL, PARTIAL = 1, 2


def segment_tiles(prob: Problem, tile: int = 128):
    """[(seg, tile_idx, start, end)] over all segments in packed order
    (seg 0 = x0, seg s = noisy copy s; each segment tiled from its start)."""
    out = []
    L, Ln = prob.L, prob.n_noisy
    bounds = [(0, L)] + [(L + (s - 1) * Ln, L + s * Ln) for s in range(1, prob.n_copies + 1)]
    for seg, (s0, s1) in enumerate(bounds):
        j = 0
        for a in range(s0, s1, tile):
            out.append((seg, j, a, min(a + tile, s1)))
            j += 1
    return out


def classify(prob: Problem, tile: int = 128, m=None):
    if m is None:
        m = mask_dense(prob)
    tiles = segment_tiles(prob, tile)
    out = []
    for qs, qi, q0, q1 in tiles:
        for ks, ki, k0, k1 in tiles:
            blk = m[q0:q1, k0:k1]
            if blk.all():
                out.append((qs, qi, ks, ki, FULL))
            elif blk.any():
                out.append((qs, qi, ks, ki, PARTIAL))
    return out


def counts(prob: Problem, tile: int = 128):
    c = classify(prob, tile)
    full = sum(1 for x in c if x[4] == FULL)
    part = sum(1 for x in c if x[4] == PARTIAL)
    n = len(segment_tiles(prob, tile))
    return {"nonempty": full + part, "full": full, "partial": part, "all": n * n}
