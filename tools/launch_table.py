"""Per-kernel totals from an ncu launch-list CSV (gpu__time_duration + dram bytes)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # launches to drop (warm-up)
hdr = None
per = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if int(d["ID"]) < skip:
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    try:
        v = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], 1.0)
    e = per.setdefault(name, {"launches": set(), "ms": 0.0, "rd": 0.0, "wr": 0.0})
    e["launches"].add(d["ID"])
    m = d["Metric Name"]
    if m == "gpu__time_duration.sum":
        e["ms"] += v * scale
    elif m == "dram__bytes_read.sum":
        e["rd"] += v * scale
    elif m == "dram__bytes_write.sum":
        e["wr"] += v * scale
tot = sum(e["ms"] for e in per.values()) or 1.0
print("| kernel | launches | total ms | share | DRAM read GB | DRAM write GB | DRAM bytes / launch (MB) |")
print("|---|---|---|---|---|---|---|")
for k, e in sorted(per.items(), key=lambda kv: -kv[1]["ms"]):
    n = len(e["launches"])
    print(f"| {k} | {n} | {e['ms']:.2f} | {100 * e['ms'] / tot:.1f}% | {e['rd'] / 1e9:.2f} | {e['wr'] / 1e9:.2f} | "
          f"{(e['rd'] + e['wr']) / max(n, 1) / 1e6:.1f} |")
