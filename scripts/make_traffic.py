"""profiles/ncu_traffic.json from an ncu --set full summary captured at the
bench shape (scripts/profile_step.py sdar_8b 16): per-launch DRAM bytes
(read + write) of each ABI call's kernels, as bench.py reports them."""
import json, sys
src = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_ncu_full_b16.json"
ks = json.load(open(src))["kernels"]
def tot(pred):
    return sum(k.get("traffic_bytes", 0) for k in ks if pred(k["kernel"]))
maps = [k for k in ks if k["kernel"].startswith("build_map")]
m1 = maps[0].get("traffic_bytes", 0) if maps else 0
out = {
    "source": src,
    "shape": "sdar_8b, batch 16 (bench shape); logprob kernels at 2048 x 151936 rows (ratio to algorithmic given)",
    "attn_fwd_kernel": tot(lambda n: n.startswith("attn_fwd")) + m1,
    "attn_bwd": tot(lambda n: n.startswith(("attn_bwd", "bwd_pre", "zero"))) + m1,
    "attn_bwd_dkdv_kernel": tot(lambda n: n.startswith("attn_bwd_dkdv")),
    "attn_bwd_dq_kernel": tot(lambda n: n.startswith("attn_bwd_dq")),
    "logprob_ratio": tot(lambda n: n == "logprob_kernel") / (2048 * 151936 * 2),
    "logprob_bwd_ratio": tot(lambda n: n == "logprob_bwd_kernel") / (2 * 2048 * 151936 * 2),
    "logprob_fused_ratio": tot(lambda n: n.startswith("logprob_fused")) / (2 * 2048 * 151936 * 2),
}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(out)
