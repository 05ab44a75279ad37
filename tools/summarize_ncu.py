#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (tracked):

  summarize_ncu.py launches <launches.csv> <out.md>
      per-kernel totals/shares of the library's kernels from a
      `ncu --metrics gpu__time_duration.sum --csv` launch list
  summarize_ncu.py full <report.ncu-rep> <out.md> [pixel_pairs]
      key counters of a `ncu --set full` capture (one launch)
"""

from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys


def short(name: str) -> str:
    m = re.search(r"pba::[^:]*::(\w+)", name)
    if m:
        tmpl = re.search(r"<\(bool\)(\d)(?:, (\d))?>", name)
        return m.group(1) + (f"<{tmpl.group(1)},{tmpl.group(2)}>" if tmpl and tmpl.group(2) else
                             (f"<{tmpl.group(1)}>" if tmpl else ""))
    return name.split("(")[0][:60]


def launches(path: str, out: str) -> None:
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if "pba::" not in name:
            continue
        k = short(name)
        tot[k] += float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else
                                              (1.0 if r["Metric Unit"] == "us" else 1e3))
        cnt[k] += 1
    all_us = sum(tot.values())
    lines = [f"# ncu launch list summary ({path})", "",
             "Library kernels only (torch setup kernels excluded); times are ncu's serialised,",
             "cold-cache per-launch durations, so compare SHARES with bench.py, not absolutes.", "",
             "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, t in tot.most_common():
        lines.append(f"| {k} | {cnt[k]} | {t:.1f} | {t / cnt[k]:.1f} | {100 * t / all_us:.1f}% |")
    lines.append(f"| **all** | {sum(cnt.values())} | {all_us:.1f} | | 100% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "  of which shared memory %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def full(path: str, out: str, pixel_pairs: float | None) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = csv.reader(io.StringIO(raw))
    h = next(r)
    units = next(r)
    vals = next(r)
    d = {k: (v, u) for k, u, v in zip(h, units, vals)}
    name = d.get("Kernel Name", ("?", ""))[0]
    lines = [f"# ncu --set full: {short(name)} ({path})", "", "| counter | value |", "|---|---|"]
    summary = {}
    for key, label in METRICS:
        if key in d:
            v, u = d[key]
            lines.append(f"| {label} (`{key}`) | {v} {u} |")
            summary[key] = (v, u)
    stalls = sorted(((k, float(v or 0)) for k, (v, u) in d.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")),
                    key=lambda kv: -kv[1])
    total = sum(v for _, v in stalls) or 1.0
    lines += ["", "| stall reason (PC samples) | share |", "|---|---|"]
    for k, v in stalls[:10]:
        lines.append(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {100 * v / total:.1f}% |")
    if pixel_pairs and "dram__bytes_read.sum" in d:
        def to_bytes(v, u):
            f = float(v)
            return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        rd = to_bytes(*d["dram__bytes_read.sum"])
        wr = to_bytes(*d["dram__bytes_write.sum"])
        lines += ["", f"DRAM bytes per pixel-pair: {(rd + wr) / pixel_pairs:.2f} "
                  f"(read {rd / pixel_pairs:.2f}, write {wr / pixel_pairs:.2f}) "
                  f"for {pixel_pairs:.0f} pixel-pairs; algorithmic = 80 B"]
        json.dump({"kernel": short(name), "pixel_pairs": pixel_pairs,
                   "dram_bytes_per_pixel_pair": (rd + wr) / pixel_pairs,
                   "dram_read_bytes": rd, "dram_write_bytes": wr, "source": path},
                  open(out.replace(".md", ".json"), "w"), indent=1)
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
