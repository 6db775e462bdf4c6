"""Summarise an ncu --set full report: per-kernel key metrics (+ optional json out)."""
import csv, json, subprocess, sys, io

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
res = []
for d in data:
    e = {"kernel": d[hdr.index("Kernel Name")].split("(")[0][-60:]}
    for k in KEYS:
        if k in hdr:
            e[k] = d[hdr.index(k)]
    res.append(e)
for e in res:
    print(e["kernel"])
    for k in KEYS:
        if k in e:
            print(f"   {k:70s} {e[k]}")
if out:
    json.dump({"report": rep, "kernels": res}, open(out, "w"), indent=1)
