"""Diagnostic: per-frame poses of the GPU and reference pipelines for a tracker."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import numpy as np
import vf_py
from helpers import centre_dist, frames, rot_angle
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS

tracker, name, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
rgb = tracker == "color"
olib = vf_py.oracle_lib(); rlib = vf_py.ref_lib(); rlib.lib.vfr_set_threads(1)
cfg = CONFIGS[name].with_(tracking=True, tracker=tracker)
fr = frames(olib, cfg, n, rgb=rgb)
s, c = settings_from_config(cfg)
p = make_pipeline(s, c)
r = vf_py.Volume(rlib, cfg, tracking=True)
for i, (pose, depth, col) in enumerate(fr):
    st = p.process_frame(col, depth)
    sr = r.process(depth, col)
    gp, rp = p.pose(), r.pose()
    print(i, "gpu", st.tracking_ok, st.tracking_iterations, f"{rot_angle(gp, pose):.2e} {centre_dist(gp, pose):.2e}",
          "| ref", sr.tracking_ok, sr.tracking_iterations, f"{rot_angle(rp, pose):.2e} {centre_dist(rp, pose):.2e}",
          "| diff", f"{rot_angle(gp, rp):.2e} {centre_dist(gp, rp):.2e}")
