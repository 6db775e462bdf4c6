"""Element-level mask: the per-element predicate the kernels evaluate
(tilemap.cuh row_interval -- forward and dQ kernels; key_interval -- dK/dV
kernel), dumped by the host path bd_mask_dump, equals the oracle's dense mask
BIT FOR BIT (BASELINE north star "the mask and tile map must match the oracle
bit-exactly"; "bitmatrix and predicate agree everywhere").

The oracle (oracle/mask.py) builds the mask from the rule table of Fig. 4 /
Eq. 2; it is itself pinned against brute-force
visibility sets and the golden grids (tests/test_oracle_mask.py).  The GPU
probe (tests/test_gpu_mask_probe.py) recovers the same bits from the kernels'
outputs."""

import numpy as np
import pytest

import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import ops
from oracle import Problem as OP, mask as omask

# (P, R, B, repeat_prompt, n_copies): the T2 grid of SURVEY §4 widened to
# block sizes that do not divide 128 (a block straddles a tile edge), P % B != 0
# in response-only mode (the first noisy row starts mid-block), ragged L < 128,
# B > 128 and trace-replay copies with non-power-of-two B
GRID = [
    (2, 6, 2, 1, 1), (2, 6, 2, 0, 1),            # Fig. 4 shape
    (0, 12, 2, 1, 1),                             # SPEC 12x12
    (32, 64, 4, 1, 1), (32, 64, 4, 0, 1),         # tiny
    (0, 96, 1, 1, 1),                             # B = 1
    (36, 264, 12, 1, 1), (42, 258, 12, 0, 1),     # B = 12 straddles tiles; P % B != 0
    (42, 214, 8, 0, 1), (42, 214, 8, 1, 1),       # P = 42, B = 8 (verdict case)
    (48, 336, 48, 1, 1), (50, 334, 48, 0, 1),
    (96, 288, 96, 1, 1), (100, 284, 96, 0, 1),
    (0, 600, 200, 1, 1), (130, 470, 200, 0, 1),
    (7, 121, 128, 1, 1), (64, 448, 256, 1, 1),
    (5, 355, 5, 1, 1), (33, 267, 3, 0, 1),        # odd B, odd P
    (36, 264, 12, 1, 3), (42, 258, 12, 0, 2),     # copies with non-power-of-two B
    (24, 216, 24, 1, 4), (8, 136, 1, 1, 4),
    (0, 2, 2, 1, 1), (1, 0, 1, 1, 1),             # degenerate: one block, prompt only
]


def _probs(P, R, B, rp, S):
    return (bd.Problem(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S),
            OP(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S))


@pytest.mark.parametrize("P,R,B,rp,S", GRID)
def test_kernel_mask_equals_oracle_bitwise(P, R, B, rp, S):
    prob, oprob = _probs(P, R, B, rp, S)
    got = ops.mask_dump(prob)
    ref = omask.mask_dense(oprob)
    assert got.shape == ref.shape
    row_view = (got & 1).astype(bool)
    key_view = (got & 2).astype(bool)
    assert np.array_equal(row_view, ref), np.argwhere(row_view != ref)[:5]
    assert np.array_equal(key_view, ref), np.argwhere(key_view != ref)[:5]


def test_kernel_mask_sdar_1_7b_rows():
    """SDAR-1.7B shape (L = 2,560, Ntot = 5,120): every row, both views."""
    prob, oprob = _probs(512, 2048, 4, 1, 1)
    for r0 in range(0, 5120, 1280):
        got = ops.mask_dump(prob, row0=r0, n_rows=1280)
        ref = omask.mask_rows(oprob, np.arange(r0, r0 + 1280))
        assert np.array_equal((got & 1).astype(bool), ref)
        assert np.array_equal((got & 2).astype(bool), ref)


def test_kernel_mask_sdar_8b_sampled_rows():
    """SDAR-8B shape (Ntot = 18,432): rows around every x0 / xt segment edge,
    tile edges and a seeded random sample, all keys, both views."""
    prob, oprob = _probs(1024, 8192, 4, 1, 1)
    N = 18432
    rng = np.random.default_rng(2)
    rows = sorted(set([0, 1, 3, 4, 127, 128, 1023, 1024, 9215, 9216, 9217, 9219, 9220, N - 1]
                      + rng.integers(0, N, 48).tolist()))
    for r in rows:
        got = ops.mask_dump(prob, row0=r, n_rows=1)[0]
        ref = omask.mask_rows(oprob, [r])[0]
        assert np.array_equal((got & 1).astype(bool), ref), r
        assert np.array_equal((got & 2).astype(bool), ref), r


def test_kernel_mask_varlen_per_sequence():
    """Varlen batch: sequence i's mask is that of its own (P_i, R_i)."""
    P = (36, 24, 0, 12)
    R = (264, 120, 96, 36)
    prob = bd.Problem(4, 36, 264, 12, 1, 1, 64, seq_prompt_lens=P, seq_response_lens=R)
    for i in range(4):
        got = ops.mask_dump(prob, seq=i)
        ref = omask.mask_dense(OP(1, P[i], R[i], 12, 1, 1, 64))
        assert got.shape == ref.shape
        assert np.array_equal((got & 1).astype(bool), ref)
        assert np.array_equal((got & 2).astype(bool), ref)


def test_mask_dump_validation():
    prob, _ = _probs(32, 64, 4, 1, 1)
    with pytest.raises(bd.ops._lib.BdError):
        ops.mask_dump(prob, seq=1)
    with pytest.raises(bd.ops._lib.BdError):
        ops.mask_dump(prob, row0=190, n_rows=5)
