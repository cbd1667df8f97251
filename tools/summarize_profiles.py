"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches csv) into profiles/."""
import csv, json, subprocess, sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "profiles"
W = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for w in W:
            if w in hdr:
                d[w] = f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip()
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.5:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 2)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        out.append(d)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr = rows[i]
            body = rows[i + 1:]
            break
    agg = defaultdict(list)
    for r in body:
        d = dict(zip(hdr, r))
        agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v) / 1000.0, "total_us": sum(v) / 1000.0}
            for k, v in agg.items()}


def main(tag, items):
    OUT.mkdir(exist_ok=True)
    summary = {}
    for name, path in items:
        p = Path(path)
        if not p.exists():
            continue
        summary[name] = launches(p) if p.suffix == ".csv" else raw(p)
    (OUT / f"{tag}.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    tag = sys.argv[1]
    main(tag, [a.split("=", 1) for a in sys.argv[2:]])
