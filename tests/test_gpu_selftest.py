"""GPU: hardware self-test of the UMMA / TMEM / TMA conventions (sm100.cuh)."""

import pytest
import torch

from paper_2512_22234_b200 import _lib


@pytest.mark.gpu
def test_selftest_mma(cuda_ok):
    L = _lib.lib()
    g = torch.Generator(device="cpu").manual_seed(0)
    a = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    b = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    outs = [torch.full((128, 128), float("nan"), device="cuda") for _ in range(4)]
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(L.bd_selftest_mma(a.data_ptr(), b.data_ptr(), v.data_ptr(), *[o.data_ptr() for o in outs], st),
               "selftest")
    torch.cuda.synchronize()
    c, o_ts, o_ss, o_mn = [o.cpu() for o in outs]
    c_ref = a.float().cpu() @ b.float().cpu().T
    err_c = (c - c_ref).abs().max().item()
    p = c.to(torch.bfloat16).float()
    o_ref = p @ v.float().cpu()
    errs = {name: (o - o_ref).abs().max().item() for name, o in (("ts", o_ts), ("ss", o_ss), ("mn", o_mn))}
    print("C err", err_c, "O errs", errs)
    assert err_c < 1e-2
    for name, e in errs.items():
        assert e < 5e-2, (name, e)
