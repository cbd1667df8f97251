"""Per-CUDA-line stall samples and instruction counts from an ncu report (cuda,sass view)."""
import csv, subprocess, sys
from collections import defaultdict
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
stall, inst, src = defaultdict(float), defaultdict(float), {}
cur_file = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    try:
        ws = float(r[4] or 0); ie = float(r[7] or 0)
    except ValueError:
        continue
    key = (cur_file, r[0])
    src[key] = r[1][:80]
    stall[key] += ws
    inst[key] += ie
ts, ti = sum(stall.values()) or 1, sum(inst.values()) or 1
for k in sorted(stall, key=lambda k: -stall[k])[:top]:
    print(f"{100*stall[k]/ts:5.1f}% stall {100*inst[k]/ti:5.1f}% inst  {k[0]}:{k[1]}  {src[k]}")
