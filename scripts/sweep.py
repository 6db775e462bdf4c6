"""Block-size sweep (BASELINE configs[3]) and the other BJ shapes:
per config tile-skip / partial fractions from the tile map and fwd / bwd /
fwd+bwd useful TFLOP/s and tokens/s (CUDA events on the current stream,
median of 5 repeats x 4 calls after warm-up; inputs >> L2).  Dev/evidence
helper -- bench.py is the contract.

    python scripts/sweep.py [out.json] [config ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_22234_b200 as bd  # noqa: E402
from paper_2512_22234_b200 import ops  # noqa: E402
from workloads import CONFIGS, attn_inputs, total_pairs, total_tokens, useful_flops  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep.json"
names = sys.argv[2:] or ["sweep_b4", "sweep_b8", "sweep_b16", "sweep_b32", "sdar_1_7b", "sdar_8b", "trace_s4",
                         "sdar_8b_varlen"]


def timeit(fn, n=4, reps=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(n):
            fn()
        en.record()
        torch.cuda.synchronize()
        out.append(st.elapsed_time(en) / n)
    return statistics.median(out)


res = []
for name in names:
    cfg = CONFIGS[name]
    prob = bd.Problem.from_cfg(cfg)
    st = ops.tilemap_stats(prob)
    q, k, v, do = attn_inputs(cfg, device="cuda")
    o, lse = bd.attn_fwd(prob, q, k, v)
    dq, dk, dv = bd.attn_bwd(prob, q, k, v, o, lse, do)
    f, fb = useful_flops(cfg)
    tf = timeit(lambda: bd.attn_fwd(prob, q, k, v, o, lse))
    tb = timeit(lambda: bd.attn_bwd(prob, q, k, v, o, lse, do, dq, dk, dv))
    pairs = total_pairs(cfg) / cfg.batch
    tiles_all, nonempty, partial = st["tiles"] ** 2, st["nonempty"], st["partial"]
    if cfg.resp_lens is not None:  # varlen: each sequence's own map, averaged
        sts = [ops.tilemap_stats(bd.Problem.from_cfg(cfg.with_(batch=1, response_len=r, resp_lens=None)))
               for r in cfg.resp_lens]
        tiles_all = sum(x["tiles"] ** 2 for x in sts) / len(sts)
        nonempty = sum(x["nonempty"] for x in sts) / len(sts)
        partial = sum(x["partial"] for x in sts) / len(sts)
    computed = nonempty * 128 * 128  # per (sequence, head), ragged tiles counted whole
    r = {"config": name, "block_size": cfg.block_size, "L": cfg.L, "batch": cfg.batch,
         "tiles": tiles_all, "nonempty": nonempty, "partial": partial,
         "tile_skip_frac": round(1 - nonempty / tiles_all, 4),
         "partial_frac": round(partial / nonempty, 4),
         "useful_over_computed": round(pairs / computed, 4),
         "fwd_ms": round(tf, 3), "bwd_ms": round(tb, 3),
         "fwd_tflops": round(f / tf / 1e9, 1), "bwd_tflops": round(fb / tb / 1e9, 1),
         "fwdbwd_tflops": round((f + fb) / (tf + tb) / 1e9, 1),
         "tokens_per_s": round(total_tokens(cfg) / ((tf + tb) / 1e3), 0)}
    print(json.dumps(r), flush=True)
    res.append(r)
    del q, k, v, do, o, lse, dq, dk, dv
    torch.cuda.empty_cache()
os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
json.dump({"what": "fwd/bwd per BJ config, one B200, CUDA events median", "results": res},
          open(out_path, "w"), indent=1)
