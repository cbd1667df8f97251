"""Print differing voxels GPU vs oracle for the first known-pose frames (T320)."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import numpy as np
import vf_py
from helpers import frames, voxel_payload
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS

olib = vf_py.oracle_lib()
cfg = CONFIGS["T320"].with_(tracking=False)
s, c = settings_from_config(cfg)
p, o = make_pipeline(s, c), vf_py.Volume(olib, cfg, False)
for fi, (pose, depth, col) in enumerate(frames(olib, cfg, 5)):
    p.set_pose(pose)
    p.process_frame(None, depth)
    o.process(depth, None, pose)
    vg = p.voxels().reshape(-1, 4); vo = o.voxels().reshape(-1, 4)
    sg = vg[:, :2].copy().view(np.int16).ravel(); so = vo[:, :2].copy().view(np.int16).ravel()
    bad = np.nonzero((sg != so) | (vg[:, 2] != vo[:, 2]))[0]
    print("frame", fi, "differing voxels", len(bad))
    for b in bad[:12]:
        blk, loc = divmod(int(b), 512)
        print("  slot", blk, "local", loc % 8, (loc // 8) % 8, loc // 64, "gpu", sg[b], vg[b, 2], "oracle", so[b], vo[b, 2])
    if len(bad):
        break
