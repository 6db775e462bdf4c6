"""Multi-rank equivalence on the real kernels (S:621-622
"W-rank loss == 1-rank loss"): two ranks (gloo, both on cuda:0 -- NCCL refuses
two ranks on one GPU) each run their (sequence, kv-head group) units of a job
through the library -- bd_attn_fwd / bd_attn_bwd on head slices of the
full-width tensors where a sequence's heads are split, bd_logprob on their
share of the response rows, bd_dipo_group_stats / bd_dipo_token_loss with the
straddling-group all-reduce -- and every output they own must be BITWISE equal
to a 1-rank run of the whole job (the kernels are deterministic and a unit's
result does not depend on which other units share the launch); the reduced
loss equals the 1-rank loss."""

import os
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

P, R, B, HQ, HKV, D, NSEQ, G, V = 64, 320, 4, 8, 4, 128, 3, 3, 1000


def _inputs():
    import paper_2512_22234_b200 as bd
    from workloads import AttnConfig, attn_inputs, logits_inputs
    cfg = AttnConfig("dist", NSEQ, HQ, HKV, D, P, R, B, seed=9)
    q, k, v, do = [x.cuda() for x in attn_inputs(cfg)]
    z, t = logits_inputs(NSEQ * R, V, seed=10)
    rewards = torch.tensor([1.0, 0.0, 1.0], device="cuda")
    return cfg, bd.Problem.from_cfg(cfg), q, k, v, do, z.cuda(), t.cuda(), rewards


def _dipo_full(ops, rewards, traj_of_token, n_groups):
    gid = torch.zeros(NSEQ, dtype=torch.int32, device="cuda")
    tlen = torch.full((NSEQ,), R, dtype=torch.int32, device="cuda")
    stats = ops.dipo_group_stats(rewards, gid, tlen, n_groups)
    return ops.dipo_token_loss(None, None, traj_of_token, rewards, gid, stats, n_groups)


def _reference():
    import paper_2512_22234_b200 as bd
    from paper_2512_22234_b200 import ops
    cfg, prob, q, k, v, do, z, t, rewards = _inputs()
    o, lse = bd.attn_fwd(prob, q, k, v)
    dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
    tok = torch.arange(NSEQ, dtype=torch.int32, device="cuda").repeat_interleave(R)
    dlogp, parts = _dipo_full(ops, rewards, tok, 1)
    logp, _, dz = ops.logprob(z, t, dlogp=dlogp)
    torch.cuda.synchronize()
    return {n: x.cpu() for n, x in dict(o=o, lse=lse, dq=dq, dk=dk, dv=dv, logp=logp, dlogp=dlogp, dz=dz,
                                          loss=parts).items()}


def _worker(rank, world, path, out_dir):
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    import paper_2512_22234_b200 as bd
    from paper_2512_22234_b200 import ops, shard, dipo
    cfg, prob, q, k, v, do, z, t, rewards = _inputs()
    o = torch.zeros_like(q)
    dq, dk, dv = torch.zeros_like(q), torch.zeros_like(k), torch.zeros_like(v)
    lse = torch.zeros((NSEQ, HQ, prob.ntot), device="cuda")
    pieces = shard.plan(NSEQ, HKV, world, rank)
    straddle = shard.groups_straddle(NSEQ, G, world, HKV)
    assert straddle
    own = shard.owners(NSEQ, HKV, world)[rank]
    gid = torch.zeros(NSEQ, dtype=torch.int32, device="cuda")
    tlen = torch.full((NSEQ,), R, dtype=torch.int32, device="cuda")
    own_t = torch.tensor(own, dtype=torch.long, device="cuda")
    stats = ops.dipo_group_stats(rewards[own_t].contiguous(), gid[own_t].contiguous(), tlen[own_t].contiguous(), 1)
    dipo.reduce_stats(stats, straddle)
    rows, tok = [], []
    for p in pieces:
        for s in range(p.seq0, p.seq1):
            a, b = shard.row_range(p.kv0, p.kv1, HKV, R)
            rows.append(torch.arange(s * R + a, s * R + b))
            tok.append(torch.full((b - a,), s, dtype=torch.int32))
    rows = torch.cat(rows).cuda()
    tok = torch.cat(tok).cuda()
    dlogp, parts = ops.dipo_token_loss(None, None, tok, rewards, gid, stats, 1)
    dipo.reduce_partials(parts)
    logp, _, dz = ops.logprob(z[rows].contiguous(), t[rows].contiguous(), dlogp=dlogp)
    for p in pieces:
        sl = slice(p.seq0, p.seq1)
        pp = prob.with_(batch=p.n_seq)
        qs, ks, vs, dos, os_, dqs, dks, dvs = q[sl], k[sl], v[sl], do[sl], o[sl], dq[sl], dk[sl], dv[sl]
        if p.n_kv != HKV:
            pp = pp.head_shard(p.kv0, p.n_kv)
            qs, dos, os_, dqs = (pp.head_slice_q(x) for x in (qs, dos, os_, dqs))
            ks, vs, dks, dvs = (pp.head_slice_kv(x) for x in (ks, vs, dks, dvs))
            assert not qs.is_contiguous()  # strided head slices go through the ABI without copies
        ls = torch.empty((p.n_seq, pp.n_q_heads, pp.ntot), device="cuda")
        bd.attn_fwd(pp, qs, ks, vs, os_, ls)
        bd.attn_bwd(pp, qs, ks, vs, os_, ls, dos, dqs, dks, dvs)
        lse[sl, p.kv0 * (HQ // HKV):p.kv1 * (HQ // HKV)] = ls
    torch.cuda.synchronize()
    torch.save({"pieces": [(p.seq0, p.seq1, p.kv0, p.kv1) for p in pieces], "rows": rows.cpu(),
                "o": o.cpu(), "lse": lse.cpu(), "dq": dq.cpu(), "dk": dk.cpu(), "dv": dv.cpu(),
                "logp": logp.cpu(), "dlogp": dlogp.cpu(), "dz": dz.cpu(), "loss": parts.cpu()},
               os.path.join(out_dir, f"rank{rank}.pt"))
    dist.destroy_process_group()


def test_two_rank_units_bitwise_equal_one_rank(cuda_ok):
    ref = _reference()
    world = 2
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        procs = [ctx.Process(target=_worker, args=(r, world, os.path.join(d, "pg"), d)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=600)
            assert p.exitcode == 0
        outs = [torch.load(os.path.join(d, f"rank{r}.pt")) for r in range(world)]
    split_heads = 0
    rows_seen = torch.zeros(NSEQ * R, dtype=torch.int32)
    Gq = HQ // HKV
    for out in outs:
        for s0, s1, kv0, kv1 in out["pieces"]:
            split_heads += kv1 - kv0 != HKV
            qh = slice(kv0 * Gq, kv1 * Gq)
            for name, hs in (("o", qh), ("dq", qh), ("dk", slice(kv0, kv1)), ("dv", slice(kv0, kv1))):
                assert torch.equal(out[name][s0:s1, :, hs], ref[name][s0:s1, :, hs]), (name, s0, kv0)
            assert torch.equal(out["lse"][s0:s1, qh], ref["lse"][s0:s1, qh])
        rows = out["rows"]
        rows_seen[rows] += 1
        assert torch.equal(out["logp"], ref["logp"][rows])
        assert torch.equal(out["dlogp"], ref["dlogp"][rows])
        assert torch.equal(out["dz"], ref["dz"][rows])
        assert abs(float(out["loss"][0]) - float(ref["loss"][0])) <= 1e-12 * max(1.0, abs(float(ref["loss"][0])))
        assert float(out["loss"][1]) == NSEQ * R
    assert split_heads >= 2  # the middle sequence's kv heads are split between the ranks
    assert bool((rows_seen == 1).all())


def test_head_shard_varlen_copies_d64_bitwise(cuda_ok):
    """Head sharding composes with varlen batches, trace-replay copies and
    d = 64: every kv-head slice run on its own (strided, no copies) is bitwise
    equal to the same heads of the unsharded launch."""
    import paper_2512_22234_b200 as bd
    from workloads import AttnConfig, attn_inputs
    cfg = AttnConfig("hs", 3, 8, 4, 64, 36, 264, 12, n_copies=2, resp_lens=(264, 120, 36))
    prob = bd.Problem.from_cfg(cfg)
    q, k, v, do = attn_inputs(cfg, device="cuda")
    o, lse = bd.attn_fwd(prob, q, k, v)
    dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
    G = 2
    for kv0, n in ((0, 1), (1, 2), (3, 1)):
        sh = prob.head_shard(kv0, n)
        qs, dos = sh.head_slice_q(q), sh.head_slice_q(do)
        ks, vs = sh.head_slice_kv(k), sh.head_slice_kv(v)
        o2, l2 = bd.attn_fwd(sh, qs, ks, vs)
        dq2, dk2, dv2 = bd.attn_bwd(sh, qs, ks, vs, o2, l2, dos)
        torch.cuda.synchronize()
        hq = slice(kv0 * G, (kv0 + n) * G)
        for bi in range(cfg.batch):
            nb = prob.seq_packed_len(bi)
            assert torch.equal(o2[bi, :nb], o[bi, :nb, hq]) and torch.equal(l2[bi, :, :nb], lse[bi, hq, :nb])
            assert torch.equal(dq2[bi, :nb], dq[bi, :nb, hq])
            assert torch.equal(dk2[bi, :nb], dk[bi, :nb, kv0:kv0 + n])
            assert torch.equal(dv2[bi, :nb], dv[bi, :nb, kv0:kv0 + n])
