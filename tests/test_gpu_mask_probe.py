"""Bit-exact recovery of the element mask that each attention KERNEL applies
(forward, dK/dV, dQ), compared with the oracle's dense mask (BASELINE north
star: "the mask and tile map must match the oracle bit-exactly").
Float parity cannot stand in for this: one wrongly visible key among 9,216
moves O by ~1e-4, far inside the 2e-2 / 1e-2 tolerances.

Probes (chunk c of d keys / rows is assigned to one (sequence, kv head), all
products are of non-negative numbers, so an output is exactly 0 iff no
visible pair contributes):

* forward: q = 0 (uniform attention over the visible keys), v_j = e_(j - c d)
  for the keys of chunk c, 0 elsewhere  =>  O[i, col] > 0  iff  key c d + col
  is visible from row i; exp(LSE_i) = number of visible keys of row i.
* bwd A (dQ and dK kernels): q_i = e_(i - c d) on the rows of chunk c,
  k_j = e_(j - c d) on its keys, v = dO = e_0, O = 0, LSE = 0 (both are the
  caller's inputs to bd_attn_bwd), so P_ij = exp(S_ij) > 0 and dS_ij = P_ij
  on visible pairs, 0 elsewhere  =>  dQ[i, col] > 0 iff (i, c d + col)
  visible; dK[j, col] > 0 iff (c d + col, j) visible.
* bwd B (dV): q = k = 0, v = 0, dO_i = e_(i - c d) on the rows of chunk c,
  O = 0, LSE = 0  =>  dV[j, col] > 0 iff (c d + col, j) visible.

Shapes: block sizes that do not divide 128 (a block straddles a tile edge),
response-only mode with P % B != 0, trace-replay copies with
non-power-of-two B, a varlen batch, and the SDAR-1.7B / SDAR-8B head shapes
in the launch configuration the bench times (d = 128, GQA 2 / 4)."""

import numpy as np
import pytest
import torch

import paper_2512_22234_b200 as bd
from oracle import Problem as OP, mask as omask

pytestmark = pytest.mark.gpu


def _oracle_mask(P, R, B, rp, S, device):
    op = OP(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S)
    N = op.ntot
    out = torch.empty((N, N), dtype=torch.bool, device=device)
    for r0 in range(0, N, 2048):
        r1 = min(N, r0 + 2048)
        out[r0:r1] = torch.from_numpy(omask.mask_rows(op, np.arange(r0, r1))).to(device)
    return out


def _onehot_rows(b, N, H, d, chunk_of, device, rows_valid=None):
    """t[bi, n, h, :] = e_(n - c d) if row n lies in chunk c = chunk_of(bi, h), else 0."""
    t = torch.zeros((b, N, H, d), dtype=torch.bfloat16, device=device)
    n = torch.arange(N, device=device)
    for bi in range(b):
        for h in range(H):
            c = chunk_of(bi, h)
            if c is None:
                continue
            lo, hi = c * d, min(N, c * d + d)
            if lo >= N:
                continue
            t[bi, n[lo:hi], h, n[lo:hi] - lo] = 1.0
    return t


def _bits(out, G, b, N, Hkv, d, chunks, which):
    """Recover the visibility bits from an output [b, N, H, d]: for heads of
    kv head g (first q head of its group when which == 'q'), chunk c =
    chunks[(bi, g)] -> columns [c d, c d + d) of the [N, N] bit matrix."""
    bits = torch.zeros((N, N), dtype=torch.bool, device=out.device)
    for (bi, g), c in chunks.items():
        lo, hi = c * d, min(N, c * d + d)
        if lo >= N:
            continue
        if which == "q":
            blk = out[bi, :, g * G:(g + 1) * G, :hi - lo] != 0          # [N, G, w]
            assert bool((blk == blk[:, :1]).all()), "q heads of one group disagree"
            bits[:, lo:hi] = blk[:, 0]
        else:
            bits[:, lo:hi] = out[bi, :, g, :hi - lo] != 0
    return bits


def _probe(P, R, B, rp=1, S=1, Hkv=8, G=2, d=128):
    dev = torch.device("cuda")
    L = P + R
    N = L + S * (L - (0 if rp else P))
    n_chunks = -(-N // d)
    b = -(-n_chunks // Hkv)
    Hq = Hkv * G
    prob = bd.Problem(b, P, R, B, Hq, Hkv, d, repeat_prompt=rp, n_copies=S)
    assert prob.ntot == N
    chunks = {(bi, g): bi * Hkv + g for bi in range(b) for g in range(Hkv) if bi * Hkv + g < n_chunks}
    ref = _oracle_mask(P, R, B, rp, S, dev)
    kv_chunk = lambda bi, g: chunks.get((bi, g))
    q_chunk = lambda bi, h: chunks.get((bi, h // G))

    # ---- forward
    q0 = torch.zeros((b, N, Hq, d), dtype=torch.bfloat16, device=dev)
    k0 = torch.zeros((b, N, Hkv, d), dtype=torch.bfloat16, device=dev)
    v1 = _onehot_rows(b, N, Hkv, d, kv_chunk, dev)
    o, lse = bd.attn_fwd(prob, q0, k0, v1)
    fwd_bits = _bits(o, G, b, N, Hkv, d, chunks, "q")
    assert torch.equal(fwd_bits, ref), ("fwd", torch.nonzero(fwd_bits != ref)[:5].tolist())
    counts = ref.sum(dim=1).double()
    got_counts = torch.exp(lse.double())
    assert torch.equal(torch.round(got_counts), counts.expand_as(got_counts)), "fwd LSE != ln(visible keys)"
    del o, lse, v1

    # ---- bwd A: dQ (row view) and dK (key view)
    q1 = _onehot_rows(b, N, Hq, d, q_chunk, dev)
    k1 = _onehot_rows(b, N, Hkv, d, kv_chunk, dev)
    e0q = torch.zeros((b, N, Hq, d), dtype=torch.bfloat16, device=dev)
    e0q[..., 0] = 1.0
    e0k = torch.zeros((b, N, Hkv, d), dtype=torch.bfloat16, device=dev)
    e0k[..., 0] = 1.0
    o0 = torch.zeros_like(q0)
    lse0 = torch.zeros((b, Hq, N), dtype=torch.float32, device=dev)
    dq, dk, _ = bd.attn_bwd(prob, q1, k1, e0k, o0, lse0, e0q)
    dq_bits = _bits(dq, G, b, N, Hkv, d, chunks, "q")
    assert torch.equal(dq_bits, ref), ("dQ", torch.nonzero(dq_bits != ref)[:5].tolist())
    dk_bits = _bits(dk, G, b, N, Hkv, d, chunks, "kv")  # [key j, row c d + col]
    assert torch.equal(dk_bits, ref.t()), ("dK", torch.nonzero(dk_bits != ref.t())[:5].tolist())
    del q1, k1, e0q, e0k, dq, dk

    # ---- bwd B: dV (key view)
    do1 = _onehot_rows(b, N, Hq, d, q_chunk, dev)
    _, _, dv = bd.attn_bwd(prob, q0, k0, k0, o0, lse0, do1)
    dv_bits = _bits(dv, G, b, N, Hkv, d, chunks, "kv")
    assert torch.equal(dv_bits, ref.t()), ("dV", torch.nonzero(dv_bits != ref.t())[:5].tolist())
    return int(ref.sum().item())


GRID = [
    # P, R, B, repeat_prompt, S
    (2, 6, 2, 1, 1), (2, 6, 2, 0, 1),          # Fig. 4 shape, both modes
    (32, 64, 4, 1, 1),                          # tiny
    (36, 264, 12, 1, 1), (42, 258, 12, 0, 1),   # B = 12: blocks straddle tile edges; P % B != 0
    (42, 214, 8, 0, 1), (42, 214, 8, 1, 1),     # P = 42, B = 8
    (48, 336, 48, 1, 1), (50, 334, 48, 0, 1),   # B = 48
    (96, 288, 96, 1, 1), (100, 284, 96, 0, 1),  # B = 96
    (0, 600, 200, 1, 1), (130, 470, 200, 0, 1),  # B = 200 > 128
    (7, 121, 128, 1, 1), (64, 448, 256, 1, 1),
    (0, 96, 1, 1, 1), (5, 355, 5, 1, 1),
    (36, 264, 12, 1, 3), (42, 258, 12, 0, 2),   # trace copies with non-power-of-two B
    (24, 216, 24, 1, 4),
]


@pytest.mark.parametrize("P,R,B,rp,S", GRID)
def test_mask_probe_grid(cuda_ok, P, R, B, rp, S):
    _probe(P, R, B, rp, S, Hkv=4, G=2)


@pytest.mark.parametrize("G,d", [(1, 128), (2, 64), (3, 64)])
def test_mask_probe_other_instantiations(cuda_ok, G, d):
    """NQ = 1 forward (odd group) and d = 64 kernels."""
    _probe(42, 258, 12, 0, 1, Hkv=4, G=G, d=d)


def test_mask_probe_sdar_1_7b(cuda_ok):
    """SDAR-1.7B heads (Hq 16 / Hkv 8, d 128), P 512 + R 2,048, B 4: all rows x all keys."""
    assert _probe(512, 2048, 4, 1, 1, Hkv=8, G=2) == 2560 * (2560 + 4)


def test_mask_probe_sdar_8b(cuda_ok):
    """SDAR-8B heads (Hq 32 / Hkv 8, d 128), P 1,024 + R 8,192, B 4: all
    18,432 x 18,432 elements of every kernel's mask."""
    assert _probe(1024, 8192, 4, 1, 1, Hkv=8, G=4) == 9216 * (9216 + 4)


def test_mask_probe_varlen(cuda_ok):
    """Varlen batch: each sequence's kernels apply that sequence's own mask;
    padding rows / keys (poisoned inputs) never become visible."""
    dev = torch.device("cuda")
    P, R, B, d, Hkv, G = 36, 264, 12, 128, 8, 2
    Ps, Rs = (36, 24, 0, 12), (264, 120, 96, 36)
    prob = bd.Problem(4, P, R, B, Hkv * G, Hkv, d, seq_prompt_lens=Ps, seq_response_lens=Rs)
    N = prob.ntot  # 600 -> 5 chunks <= Hkv
    chunks = {(bi, g): g for bi in range(4) for g in range(Hkv) if g * d < N}
    Ns = [prob.seq_packed_len(i) for i in range(4)]
    q0 = torch.zeros((4, N, Hkv * G, d), dtype=torch.bfloat16, device=dev)
    k0 = torch.zeros((4, N, Hkv, d), dtype=torch.bfloat16, device=dev)
    v1 = _onehot_rows(4, N, Hkv, d, lambda bi, g: chunks.get((bi, g)), dev)
    for bi, n in enumerate(Ns):  # padding rows: poison (a leaked padding key adds 64 P to every column)
        for t in (q0, k0, v1):
            t[bi, n:] = 64.0
    o, lse = bd.attn_fwd(prob, q0, k0, v1)
    for bi, n in enumerate(Ns):
        ref = _oracle_mask(Ps[bi], Rs[bi], B, 1, 1, dev)
        blk = o[bi, :n, ::G] != 0  # [n, Hkv, d]: chunk g = kv head g
        bits = blk.reshape(n, Hkv * d)[:, :N]
        assert torch.equal(bits[:, :n], ref), bi
        assert not bits[:, n:].any(), bi
        assert torch.isfinite(o[bi, :n].float()).all()
