"""Summarise an ncu --set full report: per-kernel key metrics with units
normalised (bytes, ms, %); optional json out."""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1,
         "second": 1e3}
res = []
for d in data:
    e = {"kernel": d[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")}
    for k in KEYS:
        if k not in hdr:
            continue
        i = hdr.index(k)
        try:
            v = float(d[i].replace(",", ""))
        except ValueError:
            continue
        u = units[i]
        if u in SCALE:
            v *= SCALE[u]
            u = "bytes" if "byte" in units[i] else "ms"
        e[k] = v
        e[k + ".unit"] = u
    if "dram__bytes_read.sum" in e:
        e["traffic_bytes"] = e["dram__bytes_read.sum"] + e.get("dram__bytes_write.sum", 0)
    res.append(e)
for e in res:
    print(e["kernel"])
    for k in KEYS + ["traffic_bytes"]:
        if k in e:
            print(f"   {k:66s} {e[k]:.6g} {e.get(k + '.unit', '')}")
if out:
    json.dump({"report": rep, "kernels": res}, open(out, "w"), indent=1)
