#!/usr/bin/env python
"""Per-phase instruction and stall-sample shares of K1 from an ncu capture.

  python tools/ncu_phases.py <report.ncu-rep> <mangled-name fragment> [out.md]
  e.g. fragment linearize_kernelILb1ELi128ELi3ELi0ELb1E (the lean default)

Joins the SASS source page of the capture (`ncu -i --page source --csv`,
per-instruction "Instructions Executed" and stall samples) with the
instruction-to-line map of the SAME build (csrc/linearize.cu recompiled
here with -lineinfo, `nvdisasm -g`), then buckets source lines into the
phases of the pixel loop.  The source must be unchanged since the capture.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CSRC = ROOT / "paper_2303_16878_b200" / "csrc"


SOURCE = Path(os.environ.get("PBA_PHASES_SRC", CSRC / "linearize.cu"))


def line_map(key):
    with tempfile.TemporaryDirectory() as tmp:
        cub = Path(tmp) / "lin.cubin"
        subprocess.run(["nvcc", "-gencode=arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                        "-std=c++17", "-I", str(ROOT / "include"), "-I", str(CSRC), "-cubin",
                        "-o", str(cub), str(SOURCE)], check=True,
                       capture_output=True)
        sass = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], check=True,
                              capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(sass)
             if l.startswith("_ZN") and key in l and l.rstrip().endswith(":")][0]
    out, cur = {}, None
    for l in sass[start + 1:]:
        if l.startswith("//---------") or l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            out[int(m.group(1), 16)] = cur
    return out


def phases(src_lines):
    """line -> phase, from the section comments of the pixel loop."""
    marks = [("---- source cue values and unprojection", "unproject + warp"),
             ("---- project into the destination", "project (+ table atan2)"),
             ("---- bilinear footprint", "dst gather + occlusion"),
             ("const bool normal_on", "normals"),
             ("---- per-cue Huber", "huber + cost"),
             ("const double wI = smI", "weights"),
             ("// Gradients of the four corners", "gradient gathers + accumulation"),
             ("---- fixed-order reduction", "reduce / epilogue")]
    loop = next(i for i, l in enumerate(src_lines) if "for (int idx = first" in l) + 1
    table, cur = {}, "prologue"
    for i, l in enumerate(src_lines, start=1):
        if i == loop:
            cur = "loop + source texel"
        for pat, name in marks:
            if pat in l:
                cur = name
        table[i] = cur
    return table


def main():
    rep, key = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else None
    csv_txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], check=True,
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(csv_txt)))
    hdr, data = rows[1], rows[2:]
    ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    lm = line_map(key)
    src = SOURCE.read_text().split("\n")
    ph = phases(src)
    helper = {"fastmath.cuh": "project (+ table atan2)"}
    base = int(data[0][ia], 16)
    agg = collections.defaultdict(lambda: [0, 0, 0])
    for r in data:
        f, ln = lm.get(int(r[ia], 16) - base, (None, None)) or (None, None)
        if f == SOURCE.name:
            name = ph.get(ln, "other")
            # inlined helpers defined above the kernel: charge to their phase
            text = src[ln - 1]
            if "ld.volatile.shared" in text or "__cvta_generic_to_shared" in text:
                name = "setup reads (volatile LDS)"
            elif "ld.global.nc.v2.f64" in text:
                name = "gradient gathers + accumulation"
            elif ln < len(src) and ("bil4" in text or "r.x = fma(w11" in text or "r.y = fma(w11" in text):
                name = "gradient gathers + accumulation"
            elif "return (1.0 - wy)" in text:
                name = "dst gather + occlusion"
            elif any(k in text for k in ("Q[upper_idx", "beta[k] = fma", "a[k] = ww", "c[0] = a[1]",
                                           "c[1] = a[2]", "c[2] = a[0]", "q[k] = -(g.x",
                                           "const double we = ww")):
                name = "gradient gathers + accumulation"
        else:
            name = helper.get(f, "library (ldg, math)")
        a = agg[name]
        a[0] += int(r[iex])
        a[1] += int(r[ist])
        op = r[hdr.index("Source")].split()[0] if r[hdr.index("Source")].split() else ""
        if re.match(r"(@!?U?P\w+\s+)?D(FMA|MUL|ADD)", r[hdr.index("Source")].strip()):
            a[2] += int(r[iex])
    te = sum(v[0] for v in agg.values())
    ts = sum(v[1] for v in agg.values())
    lines = [f"# K1 per-phase shares ({Path(rep).name})", "",
             "Warp instructions executed and warp-stall samples per phase of the pixel loop",
             "(ncu source page joined to nvdisasm -g line info of the same build; "
             "tools/ncu_phases.py).", "",
             "| phase | instructions | of which fp64 | stall samples |", "|---|---|---|---|"]
    for k, (e, s_, f) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| {k} | {100 * e / te:.1f}% | {100 * f / te:.1f}% | {100 * s_ / ts:.1f}% |")
    lines.append(f"| **total** | {te / 1e9:.2f} G | | {ts} |")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if out:
        Path(out).write_text(txt)


if __name__ == "__main__":
    main()
