"""Diagnostic: per-frame pose deviation GPU vs oracle over a tracked sequence."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import numpy as np
import vf_py
from helpers import frames, rot_angle, centre_dist, allocated_blocks
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS
name, n = sys.argv[1], int(sys.argv[2])
cfg = CONFIGS[name]
olib = vf_py.oracle_lib()
s, c = settings_from_config(cfg)
p = make_pipeline(s, c); o = vf_py.Volume(olib, cfg, True)
for i, (pose, depth, _) in enumerate(frames(olib, cfg, n)):
    st = p.process_frame(None, depth); so = o.process(depth)
    pg, po = p.pose(), o.pose()
    bg = allocated_blocks(p.entries(), p.voxels(), 4); bo = allocated_blocks(o.entries(), o.voxels(), 4)
    print(f"f{i} it={st.tracking_iterations},{so.tracking_iterations} dpose={np.abs(pg-po).max():.3e} rot={rot_angle(pg,po):.3e} "
          f"gt_err={centre_dist(pg,pose):.2e} blocks={len(bg)},{len(bo)} symdiff={len(set(bg)^set(bo))} ms={st.ms_total:.3f}")
