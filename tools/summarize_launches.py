"""Launch-list tables (mean us per kernel, launches) from the ncu --csv launch lists of
tools/profile_round.sh, in the launch order of the first step:

    python tools/summarize_launches.py gpurun_out/prof_r02 > table.md"""
import csv
import glob
import os
import sys


def table(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(r for r in rows if "Kernel Name" in r)
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    order, acc = [], {}
    for r in rows[rows.index(h) + 1:]:
        if len(r) != len(h) or r[iM] != "gpu__time_duration.sum":
            continue
        name = r[iK].split("(")[0]
        if name not in acc:
            order.append(name)
            acc[name] = []
        acc[name].append(float(r[iV].replace(",", "")))
    out = ["| kernel | launches | mean us |", "|---|---:|---:|"]
    for k in order:
        v = acc[k]
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1000:.1f} |")
    return "\n".join(out)


d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof_r02"
for f in sorted(glob.glob(os.path.join(d, "launches_*.csv"))):
    print(f"### {os.path.basename(f)[9:-4]}\n\n{table(f)}\n")
