#!/usr/bin/env python
"""Summarise ncu evidence for profiles/: per-kernel share of a frame from a
`--metrics gpu__time_duration.sum` launch list, and key counters / stall
reasons / hottest source lines from `--set full` reports.

  python scripts/ncu_summary.py --launches gpurun_out/launches2.csv \
      --reports gpurun_out/prof_k_march.ncu-rep ... > profiles/rNN_ncu_summary.md
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.per_cycle_active", "warps active/SM"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/instr"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem throughput %"),
]


def ncu_csv(path, *args):
    out = subprocess.run(["ncu", "-i", path, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def launches_table(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        name = name.split("<")[0] + ("<...>" if "<" in name else "")
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {100 * v / T:.1f}% |")
    return "\n".join(lines)


def report_summary(path, top=12, launch=None):
    sel = [] if launch is None else ["--launch-skip", str(launch), "--launch-count", "1"]
    rows = ncu_csv(path, "--page", "raw", *sel)
    h, units, d = rows[0], rows[1], rows[2]
    tag = "" if launch is None else f" (launch {launch} of the capture)"
    out = [f"### `{path.split('/')[-1]}`{tag} — `{d[h.index('Kernel Name')][:90]}`", "", "| counter | value |", "|---|---|"]
    for k, label in KEYS:
        if k in h:
            out.append(f"| {label} (`{k}`) | {d[h.index(k)]} {units[h.index(k)]} |")
    st = [(h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), d[i]) for i, c in enumerate(h)
          if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued")]

    def f(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0

    st = sorted(st, key=lambda x: -f(x[1]))[:6]
    out += ["", "stall samples: " + ", ".join(f"{k} {v}" for k, v in st), ""]
    src = ncu_csv(path, "--page", "source", "--print-source", "cuda,sass", *sel)
    agg, text, cur = collections.defaultdict(lambda: [0, 0]), {}, None
    for r in src:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) < 10 or r[0] in ("Line No", ""):
            continue
        try:
            ie, smp = int(r[7]), int(r[4])
        except ValueError:
            continue
        agg[(cur, r[0])][0] += ie
        agg[(cur, r[0])][1] += smp
        text[(cur, r[0])] = r[1][:70].replace("|", "\\|")
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    out += ["| % instr | % stall samples | line | source |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        out.append(f"| {100 * v[0] / ti:.1f} | {100 * v[1] / ts:.1f} | {k[0]}:{k[1]} | `{text[k]}` |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--reports", nargs="*", default=[])
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--launch", type=int, default=None, help="which launch of a multi-launch capture")
    ap.add_argument("--top", type=int, default=12)
    a = ap.parse_args()
    print(f"# {a.title}\n")
    if a.launches:
        print("## Launch list (gpu__time_duration.sum, --clock-control none; cold, serialised: compare shares)\n")
        print(launches_table(a.launches))
        print()
    for r in a.reports:
        print(report_summary(r, a.top, a.launch))
        print()


if __name__ == "__main__":
    main()
