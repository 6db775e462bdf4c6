"""Complete (sequence, kv-group) slices at BASELINE.json's full sizes (SURVEY
§8(c) "Parity procedure"): every one of the Ntot rows of every q-head of the
group -- O, LSE, dQ -- and that kv head's dK, dV, against the fp64 oracle's
backward_slice (oracle/attention.py, the plain dense definition), per tensor
and per segment (x0 rows, noisy-prompt rows, noisy-response rows).  A slice is
independent of the rest of the batch (dK/dV of kv head g depend only on the
q-heads of g in that sequence), so the check is exact for that slice.  The GPU
side is the full-batch launch bench.py times.  Exactness is the paper's claim
for this path ("exact" / "unbiased" logits)."""

import numpy as np
import pytest
import torch

import paper_2512_22234_b200 as bd
from oracle import Problem as OProblem, attention
from parity import FWD_MAX_ABS, FWD_REL_L2, GRAD_REL_L2, metrics, t2np
from workloads import CONFIGS, attn_inputs

pytestmark = pytest.mark.gpu


def _segments(cfg):
    """(name, row slice) of the packed axis: x0, noisy prompt, noisy response."""
    L, xb, P = cfg.L, cfg.xb, cfg.prompt_len
    segs = [("x0", slice(0, L))]
    Lx = L - xb
    for c in range(cfg.n_copies):
        base = L + c * Lx
        if P - xb > 0:
            segs.append((f"xt{c}_prompt", slice(base, base + P - xb)))
        segs.append((f"xt{c}_resp", slice(base + P - xb, base + Lx)))
    return segs


def _check_slice(cfg, q, k, v, do, o, lse, dq, dk, dv, b, g):
    G = cfg.n_q_heads // cfg.n_kv_heads
    one = OProblem(1, cfg.prompt_len, cfg.response_len, cfg.block_size, G, 1, cfg.head_dim, cfg.repeat_prompt,
                   n_copies=cfg.n_copies)
    hs = slice(g * G, (g + 1) * G)
    qs = q[b:b + 1, :, hs].float().cpu()
    dos = do[b:b + 1, :, hs].float().cpu()
    ks = k[b:b + 1, :, g:g + 1].float().cpu()
    vs = v[b:b + 1, :, g:g + 1].float().cpu()
    r_dq, r_dk, r_dv, r_o, r_lse = attention.backward_slice(one, qs, ks, vs, dos, 0, 0)
    got = {"o": t2np(o[b, :, hs]), "lse": t2np(lse[b, hs]).T, "dq": t2np(dq[b, :, hs]),
           "dk": t2np(dk[b, :, g]), "dv": t2np(dv[b, :, g])}
    ref = {"o": r_o, "lse": r_lse.T, "dq": r_dq, "dk": r_dk, "dv": r_dv}
    out = {}
    for name in got:
        fwd = name in ("o", "lse")
        for seg, sl in [("all", slice(None))] + _segments(cfg):
            a, r = got[name][sl], ref[name][sl]
            if np.linalg.norm(r) == 0:
                continue
            m = metrics(a, r)
            out[f"{name}/{seg}"] = m
            assert m["finite"], (b, g, name, seg, m)
            if fwd:
                assert m["max_abs"] <= FWD_MAX_ABS and m["rel_l2"] <= FWD_REL_L2, (b, g, name, seg, m)
            else:
                assert m["rel_l2"] <= GRAD_REL_L2, (b, g, name, seg, m)
    return out


def _run(name, slices):
    cfg = CONFIGS[name]
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, do = attn_inputs(cfg, device="cuda")
    o, lse = bd.attn_fwd(prob, q, k, v)
    dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    todo = []
    for s in slices:
        if s == "first":
            todo.append((0, 0))
        elif s == "last":
            todo.append((cfg.batch - 1, cfg.n_kv_heads - 1))
        else:
            todo.append((int(rng.integers(cfg.batch)), int(rng.integers(cfg.n_kv_heads))))
    for b, g in todo:
        m = _check_slice(cfg, q, k, v, do, o, lse, dq, dk, dv, b, g)
        print(name, (b, g), {key: (round(x["max_abs"], 5), round(x["rel_l2"], 6)) for key, x in m.items()
                             if key.endswith("/all")})


def test_full_slices_sdar_1_7b(cuda_ok):
    """SDAR-1.7B shape: four complete slices -- (0, 0), (b-1, Hkv-1), two seeded-random."""
    _run("sdar_1_7b", ["first", "last", "random", "random"])


def test_full_slices_sdar_8b(cuda_ok):
    """SDAR-8B shape (Ntot 18,432, GQA 4): (0, 0) and (b-1, Hkv-1), all rows."""
    _run("sdar_8b", ["first", "last"])


@pytest.mark.parametrize("name", ["sweep_b4", "sweep_b8", "sweep_b16", "sweep_b32"])
def test_full_slice_sweep(cuda_ok, name):
    """Block-size sweep (L = 5,120, B = 4 / 8 / 16 / 32): one seeded-random slice each."""
    _run(name, ["random"])


def test_full_slices_varlen(cuda_ok):
    """sdar_8b_varlen (16 rollouts, R_i ~ U[512, 8192]): a complete slice of the
    shortest and of a median-length sequence, against the oracle run on that
    sequence alone (its own P_i, R_i), in the batch launch bench.py times."""
    cfg = CONFIGS["sdar_8b_varlen"]
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, do = attn_inputs(cfg, device="cuda")
    o, lse = bd.attn_fwd(prob, q, k, v)
    dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
    torch.cuda.synchronize()
    order = sorted(range(cfg.batch), key=lambda i: cfg.resp_lens[i])
    for bi, g in ((order[0], 3), (order[len(order) // 2], 6)):
        one = cfg.with_(batch=1, response_len=cfg.resp_lens[bi], resp_lens=None)
        n = one.ntot
        sl = lambda t: t[bi:bi + 1, :n]  # noqa: E731
        m = _check_slice(one, sl(q), sl(k), sl(v), sl(do), sl(o), lse[bi:bi + 1, :, :n], sl(dq), sl(dk), sl(dv), 0, g)
        print("varlen", bi, cfg.resp_lens[bi], {key: (round(x["max_abs"], 5), round(x["rel_l2"], 6))
                                                for key, x in m.items() if key.endswith("/all")})
