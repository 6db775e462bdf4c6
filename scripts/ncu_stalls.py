"""Stall-sample breakdown of one kernel: top instructions with the barrier they wait on."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ia, isrc, iw = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
seen, data = set(), []
for r in rows[2:]:
    if len(r) == len(hdr) and r[ia].startswith("0x") and r[ia] not in seen:
        seen.add(r[ia])
        data.append(r)
tot = sum(float(r[iw] or 0) for r in data)
for i in sorted(range(len(data)), key=lambda i: -float(data[i][iw] or 0))[:n]:
    r = data[i]
    ctx = [data[j][isrc].strip()[:70] for j in range(max(0, i - 12), i) if "SYNCS" in data[j][isrc]]
    print(f"{float(r[iw]) / tot * 100:5.1f}% {r[ia][-5:]} {r[isrc].strip()[:60]:60s} {ctx[-1:] }")
cats = {}
for r in data:
    s = r[isrc].strip()
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    op = op.split(".")[0]
    cats[op] = cats.get(op, 0) + float(r[iw] or 0)
print({k: round(v / tot * 100, 1) for k, v in sorted(cats.items(), key=lambda x: -x[1])[:14]})
