"""Summarise an ncu report (+ optional launch-list CSV) into a markdown file."""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 else None
WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Size", "Grid Size"]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
lines = [f"# ncu summary: `{rep.split('/')[-1]}`", ""]
kn = hdr.index("Kernel Name")
mn, mu, mv = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
seen = set()
lines.append("| kernel | metric | value |")
lines.append("|---|---|---|")
for r in rows[1:]:
    if len(r) <= mv:
        continue
    if r[mn] in WANT and (r[kn], r[mn]) not in seen:
        seen.add((r[kn], r[mn]))
        lines.append(f"| {r[kn][:60]} | {r[mn]} | {r[mv]} {r[mu]} |")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) >= 3:
    h, v = rr[0], rr[2]
    lines += ["", "| raw metric | value |", "|---|---|"]
    for i, name in enumerate(h):
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
                    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                    "smsp__inst_executed.sum"):
            lines.append(f"| {name} | {v[i]} |")
if launches:
    lr = list(csv.reader(open(launches)))
    hi = next(i for i, r in enumerate(lr) if "Kernel Name" in r)
    h = lr[hi]
    k, val = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in lr[hi + 1:]:
        if len(r) > val:
            name = r[k].split("(")[0].replace("void ", "")
            c, t = agg.get(name, (0, 0.0))
            agg[name] = (c + 1, t + float(r[val].replace(",", "")))
    tot = sum(t for _, t in agg.values())
    ours = {n: v for n, v in agg.items() if "cals::" in n}
    tot_ours = sum(t for _, t in ours.values())
    lines += ["", f"## launch list (`{launches.split('/')[-1]}`, cold-cache serialised ncu timing)", "",
              "| kernel | launches | total ns | share of our kernels |", "|---|---|---|---|"]
    for n, (c, t) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {n} | {c} | {t:.0f} | {100 * t / max(tot_ours, 1):.1f}% |")
    lines.append(f"\n(all kernels incl. torch data generation: {tot:.0f} ns; ours: {tot_ours:.0f} ns)")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:60]))
