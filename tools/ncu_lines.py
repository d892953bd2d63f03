"""Aggregate ncu source-page warp-stall samples per CUDA source line."""
import csv, sys, subprocess, io, collections
rep = sys.argv[1]
kfilt = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
if kfilt:
    cmd[3:3] = ["-k", f"regex:{kfilt}", "-c", "1"]
out = subprocess.run(cmd,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
agg = collections.Counter()
inst = collections.Counter()
text = {}
hdr = None
total = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 4 and r[0] not in ("",) and r[0].isdigit():
        try:
            s = int(r[4])
        except ValueError:
            continue
        key = f"{fname}:{r[0]}"
        agg[key] += s
        try:
            inst[key] += int(r[7])
        except (ValueError, IndexError):
            pass
        text[key] = r[1].strip()[:110]
        total += s
itot = sum(inst.values()) or 1
print(f"total samples {total}  total warp-instructions {itot}")
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{100.0*v/total:5.1f}% stall {100.0*inst[k]/itot:5.1f}% inst  {k:28s} {text[k]}")
