"""ICP pixel-pass sub-phase timers (SM cycles, CTA 0 thread 0, first pixel pair):
needs a library built with -DVF_ICP_FINE_TIMERS -DVF_ICP_LEGACY_LOOP
-DVF_ICP_INFLIGHT=2 (VOXFUSE_B200_LIB=...): the sub-phases exist only in the
non-pipelined loop; tools/icp_timers.py gives the per-phase totals of the
default build."""
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
names = ["staging", "transforms", "taps", "terms", "warp_reduce", "cta_sum+part", "| barrier", "sums", "ctl"]
for lvl in sorted(set(tr[:, 0].astype(int)), reverse=True):
    rows = tr[tr[:, 0] == lvl]
    sub = np.concatenate([rows[:, 32:38], rows[:, 45:48]], axis=1).mean(0)
    print(f"L{lvl} n={len(rows)} pixel={rows[:, 44].mean():.0f} " + " ".join(f"{n}={v:.0f}" for n, v in zip(names, sub)))
