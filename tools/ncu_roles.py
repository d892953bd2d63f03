"""Executed instructions and stall samples of one ncu report, grouped by source-line
ranges (kernel roles): python tools/ncu_roles.py rep name:lo-hi ..."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ranges = []
for a in sys.argv[2:]:
    n, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((n, int(lo), int(hi)))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
fname, hdr = None, None
inst, samp, sel = collections.Counter(), collections.Counter(), collections.Counter()
for r in csv.reader(io.StringIO(src)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 10 and r[0].isdigit():
        ln = int(r[0])
        role = "other:" + fname
        if fname == "sweep_tc.cu":
            for n, lo, hi in ranges:
                if lo <= ln <= hi:
                    role = n
        try:
            inst[role] += int(r[hdr.index("Instructions Executed")] or 0)
            samp[role] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            sel[role] += int(r[hdr.index("stall_selected")] or 0)
        except ValueError:
            pass
ti, ts = sum(inst.values()), sum(samp.values())
for k in sorted(inst, key=lambda k: -inst[k]):
    print(f"{k:<28} inst {inst[k] / ti * 100:5.1f}%  samples {samp[k] / ts * 100:5.1f}%  selected {sel[k]}")
