"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per
kernel launches, total time and share of OUR kernels (at:: kernels are torch's
input generation and are excluded from the share)."""
import csv, collections, sys

src, cmd = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    name = r[ki].replace("void ", "").split("(")[0][:60]
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
ours = sum(v for k, v in tot.items() if not k.startswith(("at::", "cuda::", "<unnamed>")))
print(f"ncu --metrics gpu__time_duration.sum --clock-control none -c 400: {cmd}")
print("(cold-cache, serialised launches: compare shares, not absolutes; at:: kernels are input generation)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    own = not k.startswith(("at::", "cuda::", "<unnamed>"))
    print(f"{cnt[k]:4d} launches {v:10.3f} ms {100 * v / ours if own else 0:6.1f}% of ours  {k}")
