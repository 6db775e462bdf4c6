"""Per-instruction table of one kernel from an ncu report (dev helper):
executed count, stall samples and the dominant stall reasons, in address order.
  python scripts/ncu_src_table.py REPORT.ncu-rep KERNEL_REGEX [min_share_pct]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
col = {k: i for i, k in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[col["Address"]].startswith("0x")]
seen, uniq = set(), []
for r in data:
    if r[col["Address"]] not in seen:
        seen.add(r[col["Address"]])
        uniq.append(r)
f = lambda r, k: float(r[col[k]] or 0)
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in uniq)
tot_i = sum(f(r, "Instructions Executed") for r in uniq)
stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
agg = {k: sum(f(r, k) for r in uniq) for k in stalls}
print({k[6:]: round(v / tot_s * 100, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]})
for r in uniq:
    s = f(r, "Warp Stall Sampling (All Samples)")
    ie = f(r, "Instructions Executed")
    if s / tot_s * 100 >= thr or ie / tot_i * 100 >= 1.0:
        top = sorted(((f(r, k), k[6:]) for k in stalls), reverse=True)[:2]
        print(f"{r[col['Address']][-5:]} {s / tot_s * 100:5.1f}% ie{ie / tot_i * 100:5.1f}% "
              f"{r[col['Source']].strip()[:58]:58s} {' '.join(f'{n}:{v / max(s, 1) * 100:.0f}' for v, n in top)}")
