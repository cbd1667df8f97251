"""ICP per-iteration phase timers (SM cycles) inside a normal tracked frame (run with VF_ICP_TRACE=1)."""
import os
os.environ.setdefault("VF_ICP_TRACE", "1")
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import numpy as np
import vf_py
from helpers import frames
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
olib = vf_py.oracle_lib()
s, c = settings_from_config(cfg)
p = make_pipeline(s, c)
for pose, d, _ in frames(olib, cfg, 6):
    p.process_frame(None, d)
tr = p.icp_trace()
tot = tr[:, 44:48].sum(0)
print("rows", len(tr), "phase totals (cycles): pixel %d barrier %d sums %d controller %d" % tuple(tot), "=> us", tot.sum() / 1965.0)
for r in tr:
    print(f"L{int(r[0])} i{int(r[1])} rot{int(r[31])} n={int(r[30])} cyc={r[44:48].astype(int).tolist()}")
