"""Per-iteration ICP H/g parity at identical evaluation poses (diagnostic)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import numpy as np
import test_gpu_parity as T
import vf_py
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import HashConfig
olib = vf_py.oracle_lib()
cfg, o, pts, nrm, render_pose, depth = T._icp_fixture(olib)
ok, iters, pose, tr = T._oracle_icp(olib, o, depth)
small = HashConfig(bucket_count=1 << 10, excess_count=1 << 8, block_count=1 << 8)
pipes = {}
for k, row in enumerate(tr):
    level, rot = int(row[0]), int(row[31])
    if (level, rot) not in pipes:
        s, c = settings_from_config(cfg.with_(hash=small, levels=level + 1, rotation_only_levels=rot, max_iterations=1))
        pipes[(level, rot)] = make_pipeline(s, c)
    p = pipes[(level, rot)]
    p.set_maps(pts, nrm, render_pose)
    c2w = np.concatenate([row[32:41], row[41:44]])
    p.icp_track(depth, initial=T._pose_inv(c2w))
    g = p.icp_trace()[0]
    gc2w = g[32:44]
    h_scale = np.abs(row[2:23]).max(); g_scale = np.sqrt(h_scale * row[29])
    eh = np.abs(g[2:23] - row[2:23]).max() / h_scale
    eg = np.abs(g[23:29] - row[23:29]) / g_scale
    print(f"row{k:2d} L{level} rot{rot} cnt {int(g[30])}/{int(row[30])} dpose={np.abs(gc2w-c2w).max():.2e} eH={eh:.2e} eg={eg.max():.2e} "
          f"ecost={abs(g[29]-row[29])/row[29]:.2e} g={np.abs(row[23:29]).max():.2e} gs={g_scale:.2e} cyc={g[44:48].astype(int).tolist()}")
