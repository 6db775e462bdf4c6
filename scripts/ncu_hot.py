"""Top stall instructions of one kernel from an ncu report (source page, SASS)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[hdr.index("Address")].startswith("0x")]
ia, isrc, iw = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iw] or 0) for r in data)
idx = {r[ia]: i for i, r in enumerate(data)}
for r in sorted(data, key=lambda r: -float(r[iw] or 0))[:n]:
    print(f"{float(r[iw]) / tot * 100:5.1f}%  {r[ia][-5:]}  {r[isrc][:100]}")
