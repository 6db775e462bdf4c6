"""The device tile-map builder (run inside every bd_attn_fwd / bd_attn_bwd call,
map at workspace offset 0) writes exactly the host builder's image
(bd_tilemap_host_image, itself bit-exact against the oracle's dense-mask
classification in tests/test_tilemap_abi.py): header, both CSRs, both LPT
orders and the column-to-row-entry index, word for word (unused capacity words
excluded)."""

import pytest
import torch

import paper_2512_22234_b200 as bd
from paper_2512_22234_b200 import ops

pytestmark = pytest.mark.gpu

HDR = 16


def _meaningful(img, NT, cap):
    n = img[6]  # entries
    rp = HDR
    re = rp + NT + 1
    cp = re + cap
    ce = cp + NT + 1
    fo = ce + cap
    bo = fo + NT
    cr = bo + NT
    return (img[:9], img[rp:rp + NT + 1], img[re:re + n], img[cp:cp + NT + 1], img[ce:ce + n],
            img[fo:fo + NT], img[bo:bo + NT], img[cr:cr + n])


@pytest.mark.parametrize("P,R,B,rp,S", [
    (1024, 8192, 4, 1, 1),    # SDAR-8B
    (512, 2048, 4, 1, 1),     # SDAR-1.7B
    (1024, 4096, 32, 1, 1),   # block-size sweep
    (1024, 8192, 4, 1, 4),    # trace replay, 4 noisy copies
    (100, 300, 4, 0, 1),      # response-only, ragged
    (32, 64, 4, 1, 1),        # tiny, L < 128
    (7, 121, 128, 1, 1),      # B = 128, P % B != 0
    (4096, 28672, 4, 1, 1),   # L = 32k (NT = 512)
    # blocks not aligned to tiles: B not dividing 128, xb % B != 0 (a q-tile's
    # own-copy tiles exceeded the staged per-tile stride before the fix)
    (50, 334, 48, 0, 1), (36, 264, 12, 1, 3), (100, 284, 96, 0, 1), (130, 470, 200, 0, 1),
    (42, 214, 8, 0, 2), (5, 355, 5, 1, 1),
])
def test_device_map_equals_host_image(cuda_ok, P, R, B, rp, S):
    prob = bd.Problem(1, P, R, B, 1, 1, 64, repeat_prompt=rp, n_copies=S)
    host = ops.tilemap_host_image(prob)
    N = bd.packed_len(prob)
    q = torch.zeros((1, N, 1, 64), dtype=torch.bfloat16, device="cuda")
    ws = torch.full((bd.workspace_bytes(prob, False),), 0xFF, dtype=torch.uint8, device="cuda")
    ops.attn_fwd(prob, q, q, q, ws=ws)
    torch.cuda.synchronize()
    dev = ws[:4 * len(host)].view(torch.int32).cpu().tolist()
    NT, T0 = host[4], host[5]
    cap = (len(host) - HDR - 2 * (NT + 1) - 2 * NT) // 3
    for a, b in zip(_meaningful(dev, NT, cap), _meaningful(host, NT, cap)):
        assert a == b
