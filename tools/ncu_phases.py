"""Group ncu source-page instruction counts and stall samples by source range."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
inst, samp = collections.Counter(), collections.Counter()
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0].isdigit():
        try:
            inst[(fname, int(r[0]))] += int(r[7])
            samp[(fname, int(r[0]))] += int(r[4])
        except ValueError:
            pass
# phase map: file -> list of (lo, hi, name); first match wins, else file name
phases = {}
for spec in sys.argv[2:]:
    f, rng, name = spec.split(":")
    lo, hi = map(int, rng.split("-"))
    phases.setdefault(f, []).append((lo, hi, name))
gi, gs = collections.Counter(), collections.Counter()
for (f, ln), v in inst.items():
    name = f
    for lo, hi, nm in phases.get(f, []):
        if lo <= ln <= hi:
            name = nm
            break
    gi[name] += v
    gs[name] += samp[(f, ln)]
ti, ts = sum(gi.values()) or 1, sum(gs.values()) or 1
for name in sorted(gi, key=lambda k: -gs[k]):
    print(f"{name:24s} inst {100*gi[name]/ti:5.1f}%  stall {100*gs[name]/ts:5.1f}%")
