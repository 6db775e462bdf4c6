"""CPU tests of the argument validation of the LM-head, decode and logprob
entry points (include/bd_attn.h): every error is reported through the return
code before any device work is enqueued, so these run without a GPU."""

import ctypes

from paper_2512_22234_b200 import _lib

OK, INVALID, LAYOUT, UNSUPPORTED, ALIGN, WORKSPACE = 0, 1, 2, 3, 4, 5
P = 4096  # a 16-byte aligned fake device address (never dereferenced on these paths)


def L():
    return _lib.lib()


def test_lmhead_workspace_and_validation():
    lib = L()
    assert lib.bd_lmhead_workspace_bytes(0, 4096, 151936, 0, 0) == 0
    assert lib.bd_lmhead_workspace_bytes(16, 4100, 151936, 0, 0) == 0  # hidden % 8
    fwd = lib.bd_lmhead_workspace_bytes(131072, 4096, 151936, 0, 0)
    assert fwd >= 131072 * 8 * 8  # per-chunk (max, sum) partials
    # backward: one bf16 dz chunk of min(chunk, n) rows
    assert lib.bd_lmhead_workspace_bytes(1000, 512, 4104, 1, 384) >= 384 * 4104 * 2
    assert lib.bd_lmhead_workspace_bytes(1000, 512, 4104, 1, 0) >= 1000 * 4104 * 2
    assert lib.bd_lmhead_workspace_bytes(100, 512, 4104, 1, 5000) == lib.bd_lmhead_workspace_bytes(100, 512, 4104, 1, 0)
    rc = lib.bd_lmhead_logprob(16, 256, 1000, None, P, P, P, P, P, 1 << 30, None)
    assert rc == INVALID
    rc = lib.bd_lmhead_logprob(16, 250, 1000, P, P, P, P, P, P, 1 << 30, None)
    assert rc == UNSUPPORTED and b"multiples of 8" in lib.bd_last_error()
    rc = lib.bd_lmhead_logprob(16, 256, 1000, P + 8, P, P, P, P, P, 1 << 30, None)
    assert rc == ALIGN
    rc = lib.bd_lmhead_logprob(16, 256, 1000, P, P, P, P, P, P, 16, None)
    assert rc == WORKSPACE
    rc = lib.bd_lmhead_logprob(-1, 256, 1000, P, P, P, P, P, P, 1 << 30, None)
    assert rc == INVALID
    rc = lib.bd_lmhead_logprob_bwd(16, 256, 1000, P, P, P, P, None, P, P, 0, P, 1 << 30, None)
    assert rc == INVALID
    rc = lib.bd_lmhead_logprob_bwd(16, 256, 1000, P, P, P, P, P, P, P, 8, P, 64, None)
    assert rc == WORKSPACE


def test_decode_workspace_and_validation():
    lib = L()
    ws = lib.bd_decode_workspace_bytes(128, 4, 32, 8, 128, 9216)
    assert ws > 0
    assert lib.bd_decode_workspace_bytes(2, 4, 4, 2, 64, 300) == 0      # d != 128
    assert lib.bd_decode_workspace_bytes(2, 4, 6, 4, 128, 300) == 0     # Hq % Hkv
    assert lib.bd_decode_workspace_bytes(2, 64, 4, 2, 128, 300) == 0    # B > 32
    assert lib.bd_decode_workspace_bytes(2, 8, 4, 2, 128, 4) == 0       # cap < B
    args = lambda d=128, B=4, q=P, ws_bytes=1 << 30: (2, B, 4, 2, d, 300, 0.0, q, P, P, P, P, P, P, ws_bytes, None)
    assert lib.bd_decode_attn(*args(d=64)) == UNSUPPORTED
    assert lib.bd_decode_attn(*args(B=40)) == UNSUPPORTED
    assert lib.bd_decode_attn(*args(q=None)) == INVALID
    assert lib.bd_decode_attn(*args(q=P + 4)) == ALIGN
    assert lib.bd_decode_attn(*args(ws_bytes=8)) == WORKSPACE
    assert lib.bd_decode_attn(2, 4, 6, 4, 128, 300, 0.0, P, P, P, P, P, P, P, 1 << 30, None) == INVALID
    assert lib.bd_decode_select(0, 4, 100, P, P, 0.9, P, P, P, None) == INVALID
    assert lib.bd_decode_select(2, 4, 100, None, P, 0.9, P, P, P, None) == INVALID


def test_logprob_validation():
    lib = L()
    # row stride shorter than the vocabulary
    assert lib.bd_logprob(4, 100, P, 50, P, P, P, None, None, 0, None) == INVALID
    # gradient requested without an output
    assert lib.bd_logprob(4, 100, P, 100, P, P, P, P, None, 0, None) == INVALID
    # in place with different strides
    assert lib.bd_logprob(4, 100, P, 100, P, P, P, P, P, 128, None) == INVALID
    # zero rows is a no-op
    assert lib.bd_logprob(0, 100, None, 100, None, None, None, None, None, 0, None) == OK
    assert lib.bd_logprob_bwd(4, 100, P, 100, P, None, P, P, 100, None) == INVALID


def test_dipo_validation_names():
    lib = L()
    for code, name in ((OK, b"BD_OK"), (INVALID, b"BD_ERR_INVALID_ARG"), (LAYOUT, b"BD_ERR_LAYOUT"),
                       (UNSUPPORTED, b"BD_ERR_UNSUPPORTED"), (ALIGN, b"BD_ERR_ALIGNMENT"), (6, b"BD_ERR_CUDA")):
        assert lib.bd_error_string(code) == name
    assert lib.bd_error_string(99) == b"BD_ERR_UNKNOWN"


def test_binding_rejects_host_tensors():
    """The binding never passes host pointers to the device path (no CPU fallback)."""
    import pytest
    import torch
    import paper_2512_22234_b200 as bd
    from paper_2512_22234_b200._lib import BdError
    prob = bd.Problem(1, 32, 64, 4, 2, 2, 64)
    q = torch.zeros((1, prob.ntot, 2, 64), dtype=torch.bfloat16)
    with pytest.raises(BdError, match="CUDA"):
        bd.attn_fwd(prob, q, q, q)
    with pytest.raises(BdError, match="CUDA"):
        bd.ops.logprob(torch.zeros((2, 8), dtype=torch.bfloat16), torch.zeros(2, dtype=torch.int32))
    with pytest.raises(BdError, match="outside"):
        prob.head_shard(1, 2)
