#!/usr/bin/env python
"""SASS opcode mix (executed warp instructions) of one kernel from an ncu report."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
cnt = collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[ia])
    except (ValueError, IndexError):
        continue
    op = r[isrc].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1]
    cnt[op.split()[0]] += n
tot = sum(cnt.values())
print(f"total {tot}")
for op, n in cnt.most_common(top):
    print(f"{op:24s} {n:11d} {100 * n / tot:5.1f}")
