"""Pins for oracle/decode.py (CPU only).

decode_attention is pinned to the (separately pinned) training oracle: the
active block's rows equal the noisy-copy rows of that block in the training
mask (S:201-205 inference mask == xt -> x0 blocks < k plus own xt block,
P:71-75), to torch fp64 SDPA, and to invariances.  select_tokens is pinned by
hand-constructed cases of P:312's threshold rule and torch.softmax."""

import math

import numpy as np
import pytest
import torch

from oracle import Problem, attention, decode


def _rand(shape, g):
    return torch.randn(shape, generator=g, dtype=torch.float64)


@pytest.mark.parametrize("P,R,B,Hq,Hkv", [(8, 16, 4, 4, 2), (0, 12, 3, 2, 2), (6, 18, 2, 6, 2)])
def test_equals_training_mask_noisy_rows(P, R, B, Hq, Hkv):
    """Block k of the training layout [x0 | xt] (DiRL mode): its xt rows see x0
    positions [0, kB) and its own xt block.  Put exactly those keys into the
    cache (clean prefix, then the noisy block) and decode: same O and LSE."""
    L, d = P + R, 8
    prob = Problem(1, P, R, B, Hq, Hkv, d, 1)
    g = torch.Generator().manual_seed(L + B)
    N = prob.ntot
    q, k, v = _rand((1, N, Hq, d), g), _rand((1, N, Hkv, d), g), _rand((1, N, Hkv, d), g)
    O, LSE = attention.forward(prob, q, k, v)
    for blk in range(L // B):
        c = blk * B
        xt = slice(L + c, L + c + B)
        kc = torch.cat([k[:, :c], k[:, xt]], 1)
        vc = torch.cat([v[:, :c], v[:, xt]], 1)
        o2, lse2 = decode.decode_attention(q[:, xt], kc, vc, [c + B])
        np.testing.assert_allclose(o2, O[:, xt], atol=1e-12)
        np.testing.assert_allclose(lse2, LSE[:, :, xt], atol=1e-12)


def test_vs_torch_sdpa_gqa_and_lengths():
    g = torch.Generator().manual_seed(1)
    b, B, Hq, Hkv, d, cap = 3, 4, 6, 2, 16, 40
    q, k, v = _rand((b, B, Hq, d), g), _rand((b, cap, Hkv, d), g), _rand((b, cap, Hkv, d), g)
    lens = [4, 17, 40]
    O, LSE = decode.decode_attention(q, k, v, lens)
    for s, n in enumerate(lens):
        for h in range(Hq):
            kk, vv = k[s, :n, h // 3], v[s, :n, h // 3]
            ref = torch.nn.functional.scaled_dot_product_attention(q[s, :, h][None], kk[None], vv[None])[0]
            np.testing.assert_allclose(O[s, :, h], ref.numpy(), atol=1e-12)
            lse = torch.logsumexp(q[s, :, h] @ kk.T / math.sqrt(d), -1)
            np.testing.assert_allclose(LSE[s, h], lse.numpy(), atol=1e-12)


def test_keys_past_kv_len_are_ignored():
    g = torch.Generator().manual_seed(2)
    q, k, v = _rand((1, 2, 2, 8), g), _rand((1, 10, 1, 8), g), _rand((1, 10, 1, 8), g)
    O, LSE = decode.decode_attention(q, k, v, [6])
    k2, v2 = k.clone(), v.clone()
    k2[:, 6:] = float("nan")
    v2[:, 6:] = float("nan")
    O2, LSE2 = decode.decode_attention(q, k2, v2, [6])
    np.testing.assert_array_equal(O, O2)
    np.testing.assert_array_equal(LSE, LSE2)


def test_single_key_and_errors():
    """kv_len = B = 1: the output is that key's value, LSE = its score."""
    q = torch.tensor([[[[1.0, 2.0]]]], dtype=torch.float64)
    k = torch.tensor([[[[0.5, -1.0]], [[9.0, 9.0]]]], dtype=torch.float64)
    v = torch.tensor([[[[3.0, 4.0]], [[0.0, 0.0]]]], dtype=torch.float64)
    O, LSE = decode.decode_attention(q, k, v, [1])
    np.testing.assert_allclose(O[0, 0, 0], [3.0, 4.0])
    np.testing.assert_allclose(LSE[0, 0, 0], (0.5 - 2.0) / math.sqrt(2))
    with pytest.raises(ValueError):
        decode.decode_attention(q, k, v, [3])
    with pytest.raises(ValueError):
        decode.decode_attention(torch.zeros(1, 2, 1, 2), k, v, [1])  # kv_len < B


def test_select_threshold_rule():
    V = 50
    z = np.zeros((2, 4, V))
    z[0, 1, 7] = 20.0          # confident
    z[0, 2, 3] = 20.0          # confident but not masked
    z[0, 3, 9] = 1.0           # not confident
    masked = np.array([[True, True, False, True], [True, True, True, True]])
    z[1, 2, 5] = 2.0           # sequence 1: nobody above 0.9 -> most confident (pos 2) only
    z[1, 0, 6] = 1.0
    tok, conf, com = decode.select_tokens(z, masked, 0.9)
    assert tok[0, 1] == 7 and tok[0, 2] == 3 and tok[0, 3] == 9 and tok[1, 2] == 5
    np.testing.assert_allclose(conf[0, 1], 1 / (1 + (V - 1) * math.exp(-20)))
    np.testing.assert_allclose(conf[0, 0], 1 / V)        # uniform row
    assert com.tolist() == [[False, True, False, False], [False, False, True, False]]


def test_select_ties_and_static_mode():
    V = 8
    z = np.zeros((1, 3, V))
    z[0, :, 2] = z[0, :, 5] = 4.0  # argmax tie -> lowest index; equal conf -> lowest position
    tok, conf, com = decode.select_tokens(z, np.ones((1, 3), bool), 1.0)
    assert (tok == 2).all()
    assert com.tolist() == [[True, False, False]]
    _, _, com2 = decode.select_tokens(z, np.array([[False, False, False]]), 0.0)
    assert not com2.any()


def test_select_conf_vs_torch_softmax():
    g = np.random.default_rng(3)
    z = g.standard_normal((3, 5, 101)) * 3
    tok, conf, _ = decode.select_tokens(z, np.ones((3, 5), bool), 0.9)
    p = torch.softmax(torch.from_numpy(z), -1)
    np.testing.assert_allclose(conf, p.max(-1).values.numpy(), atol=1e-14)
    np.testing.assert_array_equal(tok, p.argmax(-1).numpy())
