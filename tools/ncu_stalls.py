"""Summary of one ncu report: key throughput metrics, stall reasons, and the top
source lines for a stall reason.  python tools/ncu_stalls.py rep.ncu-rep [reason] [n]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 12
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
# the longest captured launch
dur = {}
for r in rows[1:]:
    d0 = dict(zip(rows[0], r))
    if d0.get("Metric Name") == "Duration":
        v = float(d0["Metric Value"].replace(",", ""))
        dur[d0["ID"]] = v * (1000.0 if d0["Metric Unit"] == "ms" else (1e-3 if d0["Metric Unit"] == "ns" else 1.0))
LID = max(dur, key=dur.get) if dur else "0"
print("launch", LID, "of", len(dur))
rows = [rows[0]] + [r for r in rows[1:] if dict(zip(rows[0], r)).get("ID") == LID]
want = ["Duration", "DRAM Throughput", "L2 Cache Throughput", "Issue Slots Busy", "Executed Instructions", "L2 Hit Rate",
        "No Eligible", "Elapsed Cycles", "Achieved Active Warps Per SM", "Registers Per Thread"]
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:<30} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
idx = [i for i, r in enumerate(rr) if i >= 2 and dict(zip(rr[0], r)).get("ID") == LID] or [2 if len(rr) > 2 else 1]
d = dict(zip(rr[0], rr[idx[0]]))
st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0)) for k, v in d.items()
      if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
tot = sum(v for _, v in st) or 1
print("stalls:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(st, key=lambda kv: -kv[1])[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--launch-skip", LID, "--launch-count", "1"] if False else
                     ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
fname, hdr = None, None
agg, txt, allagg = collections.Counter(), {}, collections.Counter()
for r in csv.reader(io.StringIO(src)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 10 and r[0].isdigit():
        try:
            agg[(fname, r[0])] += int(r[hdr.index(reason)])
            allagg[(fname, r[0])] += int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        txt[(fname, r[0])] = r[1].strip()[:90]
t = sum(agg.values()) or 1
ta = sum(allagg.values()) or 1
print(f"top lines by {reason}:")
for k, v in agg.most_common(ntop):
    print(f"  {v / t * 100:5.1f}% ({allagg[k] / ta * 100:4.1f}% of all) {k[0]}:{k[1]}  {txt[k]}")
print("top lines by all samples:")
for k, v in allagg.most_common(ntop):
    print(f"  {v / ta * 100:5.1f}% {k[0]}:{k[1]}  {txt[k]}")
