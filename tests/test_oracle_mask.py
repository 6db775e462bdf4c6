"""Pins for oracle/mask.py and oracle/tilemap.py (CPU only)."""

import itertools
import os

import numpy as np
import pytest

from oracle import Problem, mask, tilemap
from bruteforce import visibility_sets, read_grid

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _prob(P, R, B, rp=1):
    return Problem(batch=1, prompt_len=P, response_len=R, block_size=B, n_q_heads=1,
                   n_kv_heads=1, head_dim=8, repeat_prompt=rp)


def _grid_cases():
    for B in (1, 2, 3, 4, 8):
        for L in range(B, 25, B):
            for P in sorted({0, B, L // 2, L - B, 1 if B > 1 else 0, L}):
                if P > L:
                    continue
                for rp in (0, 1):
                    yield L, P, B, rp


@pytest.mark.parametrize("L,P,B,rp", list(_grid_cases()))
def test_mask_equals_bruteforce_sets(L, P, B, rp):
    """S:228-231 independent visibility predicate vs bit-matrix construction."""
    prob = _prob(P, L - P, B, rp)
    m = mask.mask_dense(prob)
    _, vis = visibility_sets(L, P, B, rp)
    assert m.shape == (len(vis), len(vis))
    for n, s in enumerate(vis):
        expect = np.zeros(len(vis), bool)
        expect[list(s)] = True
        assert np.array_equal(m[n], expect), (n, sorted(s))
    mask.assert_rows_nonempty(m)  # every row sees its own block


@pytest.mark.parametrize("B", [1, 2, 4, 8])
@pytest.mark.parametrize("L_blocks", [1, 2, 3, 5])
def test_pairs_closed_form(B, L_blocks):
    """pairs = L (L + B) in DiRL mode (SURVEY §8(c) closed form, derived:
    x0 rows see sum_k (k+1)B^2, xt rows see sum_k k B^2 + B^2)."""
    L = B * L_blocks
    for P in (0, B * (L_blocks // 2)):
        prob = _prob(P, L - P, B, 1)
        assert mask.mask_dense(prob).sum() == L * (L + B)


@pytest.mark.parametrize("fname,P,R,B,rp,pairs", [
    ("fig4_dirl_mask.txt", 2, 6, 2, 1, 80),
    ("fig4_traceRL_mask.txt", 2, 6, 2, 0, 76),
    ("spec_12x12_mask.txt", 2, 4, 2, 1, 48),
])
def test_golden_grids(fname, P, R, B, rp, pairs):
    """Fig. 4 shape and SPEC's 12x12 example."""
    g = np.array(read_grid(os.path.join(GOLD, fname)))
    m = mask.mask_dense(_prob(P, R, B, rp))
    assert g.sum() == pairs
    assert np.array_equal(m, g)


def test_single_block_no_prompt():
    """S:203 'K=1, no prompt: mask is all-ones BxB' on x0; xt sees only itself
    (S:215 '1 block fully masked: NOISY copy sees only itself')."""
    B = 4
    m = mask.mask_dense(_prob(0, B, B, 1))
    assert m[:B, :B].all() and not m[:B, B:].any()
    assert m[B:, B:].all() and not m[B:, :B].any()


def test_response_rows_identical_across_modes():
    """Reading c2: response rows are identical in both modes (no row other than
    a noisy-prompt row ever sees a noisy-prompt key)."""
    for P, R, B in [(4, 8, 2), (8, 16, 4), (6, 6, 3)]:
        a = mask.mask_dense(_prob(P, R, B, 1))
        b = mask.mask_dense(_prob(P, R, B, 0))
        L = P + R
        # x0 rows: identical over x0 keys, nothing in xt
        assert np.array_equal(a[:L, :L], b[:L, :L])
        # noisy response rows in DiRL mode = rows L+P.. ; in TraceRL mode L..
        ra = a[L + P:, :]
        rb = b[L:, :]
        assert np.array_equal(ra[:, :L], rb[:, :L])
        assert np.array_equal(ra[:, L + P:], rb[:, L:])
        assert not ra[:, L:L + P].any()


def test_layout_error():
    with pytest.raises(ValueError):
        mask.mask_dense(_prob(3, 4, 2, 1))  # L=7 not multiple of B


# ---------------------------------------------------------------- tile map


def _tile_counts_bruteforce(prob, tile):
    m = mask.mask_dense(prob)
    tiles = tilemap.segment_tiles(prob, tile)
    nfull = npart = 0
    for _, _, q0, q1 in tiles:
        for _, _, k0, k1 in tiles:
            s = m[q0:q1, k0:k1].sum()
            if s == (q1 - q0) * (k1 - k0):
                nfull += 1
            elif s:
                npart += 1
    return nfull, npart


@pytest.mark.parametrize("T,B,tile", [(1, 4, 8), (2, 4, 8), (3, 2, 8), (4, 4, 16), (3, 8, 32), (2, 16, 32)])
def test_tile_counts_closed_form(T, B, tile):
    """Aligned L with B | tile, DiRL: T^2 + 2T non-empty tiles, 3T of them
    PARTIAL (T^2 + T when B = tile), derived in SURVEY §8(a) a1."""
    L = T * tile
    prob = _prob(0, L, B, 1)
    c = tilemap.counts(prob, tile)
    if B < tile:
        assert c["nonempty"] == T * T + 2 * T
        assert c["partial"] == 3 * T
    assert (c["full"], c["partial"]) == _tile_counts_bruteforce(prob, tile)
    prob2 = _prob(0, L, tile, 1)
    assert tilemap.counts(prob2, tile)["nonempty"] == T * T + T


def test_tile_classification_covers_every_pair():
    """Every visible pair lies in a listed tile; EMPTY tiles hold none."""
    for P, R, B, rp, tile in [(2, 6, 2, 1, 4), (4, 20, 4, 0, 8), (12, 36, 4, 1, 16), (0, 24, 8, 1, 8)]:
        prob = _prob(P, R, B, rp)
        m = mask.mask_dense(prob)
        listed = np.zeros_like(m)
        tiles = {(s, i): (a, b) for s, i, a, b in tilemap.segment_tiles(prob, tile)}
        for qs, qi, ks, ki, kind in tilemap.classify(prob, tile, m):
            q0, q1 = tiles[(qs, qi)]
            k0, k1 = tiles[(ks, ki)]
            listed[q0:q1, k0:k1] = True
            if kind == tilemap.FULL:
                assert m[q0:q1, k0:k1].all()
        assert not (m & ~listed).any()
