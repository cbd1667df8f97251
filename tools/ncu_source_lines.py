#!/usr/bin/env python
"""Per-CUDA-source-line breakdown of one kernel from an `ncu --set full
--import-source on` report: warp instructions executed and warp-stall samples
per line (ncu --page source --print-source cuda,sass), sorted by instructions.

  python tools/ncu_source_lines.py report.ncu-rep [--top 40] [--kernel regex]
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--kernel", default=None)
    a = ap.parse_args()
    cmd = ["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if a.kernel:
        cmd += ["-k", f"regex:{a.kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    path, hdr = None, None
    agg = defaultdict(lambda: [0, 0, ""])
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0]:
            continue
        try:
            ins = int(r[hdr.index("Instructions Executed")])
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        k = (path, int(r[0]))
        agg[k][0] += ins
        agg[k][1] += smp
        agg[k][2] = r[1].strip()[:90]
    tot_i = sum(v[0] for v in agg.values()) or 1
    tot_s = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {tot_i}, stall samples {tot_s}")
    print(f"{'file:line':28s} {'warp inst':>11s} {'%inst':>6s} {'%stall':>6s}  source")
    for (f, ln), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: a.top]:
        print(f"{f + ':' + str(ln):28s} {i:11d} {100 * i / tot_i:6.2f} {100 * s / tot_s:6.2f}  {src}")


if __name__ == "__main__":
    main()
