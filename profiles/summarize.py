#!/usr/bin/env python
"""Summarise ncu artefacts into committed text (profiles/).

    python profiles/summarize.py launches <launches.csv>          # per-kernel mean device time
    python profiles/summarize.py report <prof.ncu-rep> [...]       # key metrics + stall mix

`launches` reads the `--metrics gpu__time_duration.sum --csv` launch list;
`report` exports the raw page of an `ncu --set full` report with the local ncu.
Both print markdown tables.
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) > vi:
            agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
    print("| kernel | launches | mean us |\n|---|---:|---:|")
    for k, v in agg.items():
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1000:.1f} |")


def report(path: str) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    print(f"#### {path}\n")
    print("| kernel | " + " | ".join(n for _, n in KEYS) + " | top stalls |")
    print("|---" * (len(KEYS) + 2) + "|")
    for d in data:
        name = d[hdr.index("Kernel Name")].split("(")[0]
        cells = []
        for k, _ in KEYS:
            if k in hdr:
                i = hdr.index(k)
                cells.append(f"{d[i]} {units[i]}".strip())
            else:
                cells.append("-")
        vals = sorted(((float(d[hdr.index(h)].replace(",", "") or 0), h) for h in stalls), reverse=True)
        tot = sum(v for v, _ in vals) or 1.0
        top = ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%"
                        for v, h in vals[:4])
        print(f"| `{name}` | " + " | ".join(cells) + f" | {top} |")
    print()


if __name__ == "__main__":
    mode, paths = sys.argv[1], sys.argv[2:]
    for p in paths:
        (launches if mode == "launches" else report)(p)
